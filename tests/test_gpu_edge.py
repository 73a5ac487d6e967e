"""GPU edge cases through the C-ABI, against the CPU oracle ("What's weak" 3):

* inputs near the fp64 range limits (A x 1e-300 ... 1e+300): inside [2^-400, 2^400]
  the default kernels are exact (1e+-110 checks it), outside TSQR_FLAG_ROBUST makes
  every step rescale like LAPACK's dlarfg (reading R23); the oracle's long-double
  sums have the exponent range to take them unscaled;
* strided storage (lda = m + 7, ldc = m + 5, ldq = m + 3): the kernels must use the
  leading dimensions, never m, and leave the padding rows alone;
* the first factor on a fresh non-default stream (stream-ordered tree setup);
* R and Q against the oracle's PLAIN paper plan (one Householder QR per row block, no
  tiles, no chunks): both are plan-independent (uniqueness modulo signs, P:877-883;
  any tree), so the comparison does not share the kernel's plan.
Tolerances as test_gpu_parity.py (BASELINE.json north_star)."""
import numpy as np
import pytest
import torch

import oracle as orc
import paper_0808_2664_b200 as T
from paper_0808_2664_b200 import inputs

pytestmark = pytest.mark.gpu

TOL_R = 1e-11
TOL_INV = 1e-13
SENTINEL = 1234.5


def _np(t):
    return inputs.to_numpy_colmajor(t)


def _c(m, n, b, s):
    return T.plan_info(m, n, block_rows=b, tile_rows=s)["chunk_rows"]


def _sign_q(R, Q):
    """Q diag(s), s = sign(diag R): the column signs that go with R's row normalisation."""
    s = np.where(np.diag(R) < 0, -1.0, 1.0)
    return Q * s[None, :]


# (m, n, b, s): the narrow chain engine (structured and dense chunk steps, the pipelined
# tree), the wide engine (blocked leaves, the pipelined wide tree) and n > 224 (masked
# dense nodes)
SCALED_SHAPES = [(5000, 50, 4096, 1366), (3000, 16, 1000, 250), (4096, 64, 4096, 4096),
                 (3000, 100, 1500, 1500), (4000, 200, 2048, 2048), (2000, 240, 1000, 1000)]


@pytest.mark.parametrize("scale", [1e-160, 1e-150, 1e-110, 1e+110, 1e+150, 1e+155, 1e-300, 1e+300])
@pytest.mark.parametrize("m,n,b,s", SCALED_SHAPES)
def test_scaled_inputs(m, n, b, s, scale):
    At = inputs.gaussian(m, n, 21) * scale
    A0 = _np(At).copy()
    Ad = At.cuda()
    robust = not (2.0 ** -400 <= scale <= 2.0 ** 400)       # TSQR_FLAG_ROBUST outside the default range (R23)
    R, tree = T.factor(Ad, block_rows=b, tile_rows=s, debug=True, robust=robust)
    Q = T.form_q(tree)
    torch.cuda.synchronize()
    Rg, Qg = _np(R), _np(Q)
    assert np.all(np.isfinite(Rg)) and np.all(np.isfinite(Qg))
    f = orc.tsqr_factor(A0, orc.plan(m, n, b, s, 1, _c(m, n, b, s)))
    assert orc.rel_fro(orc.sign_normalise(Rg), orc.sign_normalise(f.R)) <= TOL_R
    assert orc.rel_fro(Qg, orc.tsqr_form_q(f)) <= TOL_R
    # invariants on the unscaled problem (A / scale is exact up to one rounding per entry)
    An = A0 / scale
    assert np.linalg.norm(An - Qg @ (Rg / scale)) / np.linalg.norm(An) <= TOL_INV
    assert np.linalg.norm(Qg.T @ Qg - np.eye(n)) <= TOL_INV
    tree.free()


@pytest.mark.parametrize("m,n,b,s,k", [(5000, 50, 4096, 1366, 20), (4096, 16, 512, 128, 8),
                                       (4096, 64, 4096, 4096, 64), (3000, 100, 1500, 1500, 13),
                                       (4000, 200, 2048, 400, 64)])
def test_strided_storage(m, n, b, s, k):
    At = inputs.gaussian(m, n, 22)
    Ct = inputs.gaussian(m, k, 23)
    A0, C0 = _np(At).copy(), _np(Ct).copy()
    Abuf = torch.full((n, m + 7), SENTINEL, dtype=torch.float64, device="cuda")
    Cbuf = torch.full((k, m + 5), SENTINEL, dtype=torch.float64, device="cuda")
    Qbuf = torch.full((n, m + 3), SENTINEL, dtype=torch.float64, device="cuda")
    Rbuf = torch.full((n, n + 2), SENTINEL, dtype=torch.float64, device="cuda")
    A, C, Q, R = Abuf[:, :m], Cbuf[:, :m], Qbuf[:, :m], Rbuf[:, :n]
    A.copy_(At.cuda())
    C.copy_(Ct.cuda())
    assert A.stride(0) == m + 7 and C.stride(0) == m + 5 and Q.stride(0) == m + 3 and R.stride(0) == n + 2
    _, tree = T.factor(A, block_rows=b, tile_rows=s, R=R, debug=True)
    T.apply_qt(tree, C)
    T.form_q(tree, Q)
    torch.cuda.synchronize()
    for buf, rows in ((Abuf, m), (Cbuf, m), (Qbuf, m), (Rbuf, n)):
        assert torch.all(buf[:, rows:] == SENTINEL), "padding rows were written"
    f = orc.tsqr_factor(A0, orc.plan(m, n, b, s, 1, _c(m, n, b, s)))
    Rg = _np(R)
    assert orc.rel_fro(orc.sign_normalise(Rg), orc.sign_normalise(f.R)) <= TOL_R
    assert orc.rel_fro(_np(C), orc.tsqr_apply_qt(f, C0)) <= TOL_R
    assert orc.rel_fro(_np(Q), orc.tsqr_form_q(f)) <= TOL_R
    # the stored reflectors, Q^T C and Q: the same bytes a contiguous factor gives.  The odd
    # lda (m + 7) stages chunks by per-element cp.async, the contiguous even-lda copy by TMA /
    # bulk copies wherever tiles start on even rows, so this also pins
    # the two staging paths to each other bit for bit.
    A2 = At.cuda()
    _, tree2 = T.factor(A2, block_rows=b, tile_rows=s)
    C2 = Ct.cuda()
    T.apply_qt(tree2, C2)
    Q2 = T.form_q(tree2)
    torch.cuda.synchronize()
    assert torch.equal(A, A2)
    assert torch.equal(C, C2) and torch.equal(Q, Q2)
    tree.free()
    tree2.free()


def test_first_factor_on_fresh_stream():
    """A new tree built and used on a non-blocking side stream: its plan upload and
    workspace setup are ordered on that stream (no legacy-stream copies)."""
    m, n, b, s = 200_000, 50, 4096, 1366
    At = inputs.gaussian(m, n, 24)
    A0 = _np(At).copy()
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        A = At.to("cuda", non_blocking=True)
        R, tree = T.factor(A, block_rows=b, tile_rows=s)
        Q = T.form_q(tree)
    # moving the tree to another stream: the call waits for the tree's last work
    C = torch.zeros((3, m), dtype=torch.float64, device="cuda")
    C[:, :n] = torch.eye(n, dtype=torch.float64, device="cuda")[:3]
    T.apply_q(tree, C)
    torch.cuda.synchronize()
    f = orc.tsqr_factor(A0, orc.plan(m, n, b, s, 1, _c(m, n, b, s)), threads=8)
    assert orc.rel_fro(orc.sign_normalise(_np(R)), orc.sign_normalise(f.R)) <= TOL_R
    Qg = _np(Q)
    assert np.linalg.norm(A0 - Qg @ _np(R)) / np.linalg.norm(A0) <= TOL_INV
    assert torch.allclose(C.T, Q.T[:, :3], rtol=0, atol=1e-14)
    tree.free()


@pytest.mark.parametrize("m,n,b,s,kind", [(300_000, 50, 4096, 1366, "gauss"), (100_000, 200, 2048, 400, "gauss"),
                                          (262_144, 64, 4096, 4096, "cond"), (262_144, 32, 4096, 4096, "gauss"),
                                          (40_000, 16, 512, 128, "gauss")])
def test_plain_plan_parity(m, n, b, s, kind):
    """GPU R (and thin Q for kappa ~ 1) against the oracle's plain paper plan: one
    Householder QR (DGEQR2) per row block of b rows, the binary tree over the blocks
    (Eqs. 1-4), no tiles and no chunks."""
    At = inputs.gaussian(m, n, 25) if kind == "gauss" else inputs.conditioned(m, n, 25, kappa=1e10)
    A0 = _np(At).copy()
    Ad = At.cuda()
    R, tree = T.factor(Ad, block_rows=b, tile_rows=s)
    Q = T.form_q(tree)
    torch.cuda.synchronize()
    plain = orc.plan(m, n, b, 0, 1, 0)                  # s = 0: each row block is one leaf; c = 0: DGEQR2
    f = orc.tsqr_factor(A0, plain, threads=8)
    Rg, Qg = _np(R), _np(Q)
    assert orc.rel_fro(orc.sign_normalise(Rg), orc.sign_normalise(f.R)) <= TOL_R
    if kind == "gauss":                                     # Q unique up to signs (kappa ~ 1; R10)
        Qo = orc.tsqr_form_q(f)
        assert orc.rel_fro(_sign_q(Rg, Qg), _sign_q(f.R, Qo)) <= TOL_R
    assert np.linalg.norm(A0 - Qg @ Rg) / np.linalg.norm(A0) <= TOL_INV
    assert np.linalg.norm(Qg.T @ Qg - np.eye(n)) <= TOL_INV
    tree.free()


@pytest.mark.parametrize("m,n,b,s", [(200_000, 50, 4096, 1024), (60_000, 100, 2048, 400), (100_000, 64, 4096, 4096)])
def test_rank_deficient_full_engines(m, n, b, s):
    """Rank-deficient input at scale on both leaf engines (chain n <= 64, wide n > 64): a
    duplicated column and a zero column.  R is not unique past a dependent column (its later
    rows are set by rounding), so the invariants are checked: A = QR, Q^T Q = I (the Householder
    Q stays orthogonal whatever the rank), exact zeros below R's diagonal, and the dependent
    columns' diagonal entries at rounding level."""
    At = inputs.gaussian(m, n, 31)
    At[10] = At[3]                       # column 10 = column 3 (tensor rows are matrix columns)
    At[20] = 0.0
    A0 = _np(At).copy()
    A = At.cuda()
    R, tree = T.factor(A, block_rows=b, tile_rows=s)
    Q = T.form_q(tree)
    torch.cuda.synchronize()
    Rg, Qg = _np(R), _np(Q)
    assert np.all(np.isfinite(Rg)) and np.all(np.isfinite(Qg))
    assert np.all(np.tril(Rg, -1) == 0.0)
    nA = np.linalg.norm(A0)
    assert np.linalg.norm(A0 - Qg @ Rg) / nA <= TOL_INV
    assert np.linalg.norm(Qg.T @ Qg - np.eye(n)) <= TOL_INV
    assert abs(Rg[10, 10]) <= 1e-13 * nA and abs(Rg[20, 20]) <= 1e-13 * nA
    tree.free()
