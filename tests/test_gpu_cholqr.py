"""CholeskyQR on the GPU (tsqr_cholqr / tsqr_ctx_cholqr): SURVEY 8(f) row 4, the comparison
method -- Alg. CholeskyQR ([TR] P:1410-1419).

Parity: R and Q against the oracle's orc_cholqr on well-conditioned inputs (kappa ~ 1,
where CholeskyQR is accurate: R within 1e-12 of the oracle, Q within 1e-12), ragged and
strided shapes, n up to TSQR_MAX_N; the breakdown index on a zero column equals the
oracle's.  Stability: on the C4 recipe CholeskyQR's
orthogonality degrades as kappa^2 and it breaks down (or loses all orthogonality) at
kappa = 1e10, while TSQR's Q stays orthogonal to 1e-13 at every kappa.  Multi-rank:
the loopback transport (one GPU, each rank's kernels never wait on another's) gives R
bitwise replicated across ranks and equal to the oracle on the global A.
CPU: the argument checks (no device work)."""
import ctypes
import threading

import numpy as np
import pytest
import torch

import oracle as orc
import paper_0808_2664_b200 as T
from paper_0808_2664_b200 import _lib, inputs


def test_cholqr_validation_without_gpu():
    L = _lib.lib()
    fake = ctypes.c_void_p(0x1000)
    assert L.tsqr_cholqr(100, 10, None, 100, fake, 10, None, 0, fake, None) == 1        # A null
    assert L.tsqr_cholqr(100, 10, fake, 100, fake, 10, None, 0, None, None) == 1        # info null
    assert L.tsqr_cholqr(5, 10, fake, 100, fake, 10, None, 0, fake, None) == 2          # m < n
    assert L.tsqr_cholqr(1000, 300, fake, 1000, fake, 300, None, 0, fake, None) == 3    # n > TSQR_MAX_N
    assert L.tsqr_cholqr(100, 10, fake, 99, fake, 10, None, 0, fake, None) == 1         # lda < m
    assert L.tsqr_cholqr(100, 10, fake, 100, fake, 10, fake, 50, fake, None) == 1       # ldq < m
    assert L.tsqr_ctx_cholqr(None, 100, 10, fake, 100, fake, 10, None, 0, fake, None) == 1


def _gauss(m, n, seed=0):
    return inputs.gaussian(m, n, seed)


@pytest.mark.gpu
@pytest.mark.parametrize("m,n", [(1000, 8), (5001, 16), (20000, 50), (3000, 64), (4099, 33), (6000, 100),
                                 (5000, 200), (2000, 256), (777, 1)])
def test_cholqr_parity(m, n):
    A = _gauss(m, n)
    info_o, Ro, Qo = orc.cholqr(inputs.to_numpy_colmajor(A))
    assert info_o == 0
    Ad = A.cuda()
    R, Q, info = T.cholqr(Ad)
    torch.cuda.synchronize()
    assert int(info.item()) == 0
    R, Q = inputs.to_numpy_colmajor(R), inputs.to_numpy_colmajor(Q)
    assert np.all(np.tril(R, -1) == 0.0) and np.all(np.diag(R) > 0)
    assert orc.rel_fro(R, Ro) <= 1e-12
    assert orc.rel_fro(Q, Qo) <= 1e-12
    assert torch.equal(Ad.cpu(), A)                              # A is read only


@pytest.mark.gpu
def test_cholqr_strided_and_r_only():
    m, n, pad = 3000, 24, 7
    A = _gauss(m, n, 3)
    big = torch.zeros((n, m + pad), dtype=torch.float64)
    big[:, :m] = A
    Ad = big.cuda()[:, :m]                                       # lda = m + 7
    Qbig = torch.full((n, m + 5), 7.0, dtype=torch.float64, device="cuda")
    R, Q, info = T.cholqr(Ad, Q=Qbig[:, :m])
    R2, Q2, info2 = T.cholqr(A.cuda(), want_q=False)
    torch.cuda.synchronize()
    assert int(info.item()) == 0 and int(info2.item()) == 0 and Q2 is None
    _, Ro, Qo = orc.cholqr(inputs.to_numpy_colmajor(A))
    assert orc.rel_fro(inputs.to_numpy_colmajor(R), Ro) <= 1e-12
    assert orc.rel_fro(inputs.to_numpy_colmajor(Q), Qo) <= 1e-12
    assert torch.all(Qbig[:, m:] == 7.0)                         # nothing past ldq's rows written
    assert torch.equal(R, R2)


@pytest.mark.gpu
def test_cholqr_breakdown_index():
    A = _gauss(2000, 12, 4)
    A[5, :] = 0.0                                                # column 5 (row 5 of the (n, m) tensor)
    info_o, _, _ = orc.cholqr(inputs.to_numpy_colmajor(A))
    _, _, info = T.cholqr(A.cuda())
    torch.cuda.synchronize()
    assert info_o == 6 and int(info.item()) == 6


@pytest.mark.gpu
def test_cholqr_vs_tsqr_stability_split():
    """P:1347-1354 / P:1399-1402 on the C4 recipe (reading R15) at m = 2^18, n = 64."""
    m, n = 1 << 18, 64
    errs = {}
    for kappa in (1e1, 1e3, 1e5, 1e10):
        A = inputs.conditioned(m, n, seed=0, kappa=kappa).cuda()
        R, Q, info = T.cholqr(A)
        Af = A.clone()
        Rt, tree = T.factor(Af, 4096, 4096)
        Qt = T.form_q(tree)
        torch.cuda.synchronize()
        I = torch.eye(n, dtype=torch.float64, device="cuda")
        orth_t = torch.linalg.norm(Qt @ Qt.T - I).item()
        assert orth_t <= 1e-13                                   # TSQR: orthogonal at every kappa
        assert (torch.linalg.norm(A - Rt @ Qt) / torch.linalg.norm(A)).item() <= 1e-13     # tensors hold R^T, Q^T
        if int(info.item()) == 0:
            errs[kappa] = torch.linalg.norm(Q @ Q.T - I).item()
        else:
            errs[kappa] = float("inf")                           # Cholesky of A^T A broke down
        tree.free()
    eps = np.finfo(np.float64).eps
    assert errs[1e1] <= 1e-13
    assert errs[1e3] <= 100 * 1e6 * eps
    assert errs[1e5] >= 1e3 * errs[1e3]                          # grows like kappa^2 (1e4 here)
    assert errs[1e10] > 1e-2                                     # lost (or broke down): kappa^2 eps >> 1


@pytest.mark.gpu
@pytest.mark.parametrize("G,m,n", [(2, 20000, 50), (4, 40001, 32), (8, 30000, 64)])
def test_ctx_cholqr_loopback(G, m, n):
    hub = T.Loopback(G)
    rows = [T.slab(m, n, 4096, G, r) for r in range(G)]
    out, errs = {}, []

    def rank_main(r):
        try:
            torch.cuda.set_device(0)
            st = torch.cuda.Stream()
            ctx = T.Ctx(0).set_loopback(hub, r)
            row0, ml = rows[r]
            with torch.cuda.stream(st):
                A = inputs.gaussian_rows(row0, ml, n, 0).cuda()
            R, Q, info = ctx.cholqr(A, stream=st)
            st.synchronize()
            out[r] = (inputs.to_numpy_colmajor(R).copy(), inputs.to_numpy_colmajor(Q).copy(), int(info.item()))
            ctx.free()
        except Exception as e:                                   # noqa: BLE001 -- reported below
            errs.append((r, repr(e)))

    th = [threading.Thread(target=rank_main, args=(r,)) for r in range(G)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    assert not errs, errs
    _, Ro, Qo = orc.cholqr(inputs.to_numpy_colmajor(_gauss(m, n)))
    for r, (row0, ml) in enumerate(rows):
        R, Q, info = out[r]
        assert info == 0
        assert np.array_equal(R, out[0][0])                      # W all-reduced in rank order: R bitwise replicated
        assert orc.rel_fro(R, Ro) <= 1e-12
        assert orc.rel_fro(Q, Qo[row0:row0 + ml]) <= 1e-12
