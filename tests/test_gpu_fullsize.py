"""GPU parity at BASELINE.json's full sizes, in the launch configuration bench.py
times (its block rows b and tile rows s).  C2 and C3 are compared with the CPU
oracle element by element (the oracle finishes them in seconds).  C4 and C5
(8.6 GB each): R against the oracle run on every host core (leaves in parallel,
orc_tsqr_factor_mt), both in the kernel's plan and in the paper's plain plan (one
DGEQR2 per 4096-row block), plus properties that hold at any size, computed
with plain PyTorch fp64 on the GPU from the untouched input:
  R^T R = A^T A (Cor. 1 identity), ||A - QR||/||A||, ||Q^T Q - I||,
  column norms of Q^T C equal those of C (Q orthogonal), and the thin part
  Q_thin^T C = R^-T (A^T C) (Q_thin = A R^-1 with the product's own R).
Tolerances as in test_gpu_parity.py (BASELINE.json north_star)."""
import os
import sys

import numpy as np
import pytest
import torch

import oracle as orc
import paper_0808_2664_b200 as T
from paper_0808_2664_b200 import inputs

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402  (only its CONFIGS table: the bench's launch configuration)

pytestmark = pytest.mark.gpu

TOL_R = 1e-11
TOL_INV = 1e-13
TOL_REFL = 1e-13


def _np(t):
    return inputs.to_numpy_colmajor(t)


def _cfg(name):
    c = bench.CONFIGS[name]
    return c["m"], c["n"], c["b"], c["s"], c["k"]


def _c(m, n, b, s):
    return T.plan_info(m, n, block_rows=b, tile_rows=s)["chunk_rows"]


THREADS = max(1, os.cpu_count() or 1)


def _oracle_r_full(A_dev, p):
    """R of the oracle's TSQR over plan p, on a host copy of A_dev (column-major (n, m)),
    leaves in parallel on every host core; the copy is factored in place."""
    Ah = A_dev.cpu().numpy().T                    # Fortran-ordered m x n view of the copy
    f = orc.tsqr_factor(Ah, p, threads=THREADS, overwrite=True, keep_y1=False)
    del Ah
    return f.R


def _sign_q(R, Q):
    s = np.where(np.diag(R) < 0, -1.0, 1.0)
    return Q * s[None, :]


def _check_reflectors(F, tree, p, f, n):
    """Leaf reflector tails (every tile row below its diagonal), node Y1 (the
    right subtree's head, upper triangle) and all taus against the oracle."""
    local = np.arange(F.shape[0]) - np.repeat(p.tile_row0, p.tile_rows)     # row index inside its tile
    below = local[:, None] > np.arange(n)[None, :]
    assert orc.rel_fro(np.where(below, F, 0.0), np.where(below, f.A, 0.0)) <= TOL_REFL
    tt, tn = tree.export_tau()
    assert orc.rel_fro(tt, f.tau_tile) <= TOL_REFL
    for q in range(p.nnodes):
        bt = p.node_b[q]
        assert orc.rel_fro(np.triu(F[p.tile_row0[bt]:p.tile_row0[bt] + n]), orc.node_y1(f, q)) <= TOL_REFL
        assert orc.rel_fro(tn[bt], f.tau_node[q]) <= TOL_REFL


def test_full_c2_factor_and_form_q():
    m, n, b, s, _ = _cfg("c2")
    At = inputs.gaussian(m, n, 0)
    A0 = _np(At).copy()
    Ad = At.cuda()
    R, tree = T.factor(Ad, b, s)
    Q = T.form_q(tree)
    torch.cuda.synchronize()
    p = orc.plan(m, n, b, s, 1, _c(m, n, b, s))
    f = orc.tsqr_factor(A0, p)
    Rg = _np(R)
    assert orc.rel_fro(orc.sign_normalise(Rg), orc.sign_normalise(f.R)) <= TOL_R
    _check_reflectors(_np(Ad), tree, p, f, n)
    Qo = orc.tsqr_form_q(f)
    assert orc.rel_fro(_np(Q), Qo) <= TOL_R
    Qt, Rt = Q.T, R.T                             # (m, n) and (n, n) views of the matrices
    assert torch.linalg.norm(At.cuda().T - Qt @ Rt) / torch.linalg.norm(At) <= TOL_INV
    assert torch.linalg.norm(Qt.T @ Qt - torch.eye(n, dtype=torch.float64, device="cuda")) <= TOL_INV
    tree.free()


@pytest.mark.parametrize("s", [2048, None])
def test_full_c3_factor_and_apply(s):
    m, n, b, s_bench, k = _cfg("c3")
    s = s_bench if s is None else s
    At = inputs.gaussian(m, n, 0)
    A0 = _np(At).copy()
    Ad = At.cuda()
    R, tree = T.factor(Ad, b, s)
    Ct = inputs.gaussian(m, k, 1)
    C0 = _np(Ct).copy()
    Cd = Ct.cuda()
    T.apply_qt(tree, Cd)
    torch.cuda.synchronize()
    p = orc.plan(m, n, b, s, 1, _c(m, n, b, s))
    f = orc.tsqr_factor(A0, p)
    Rg = _np(R)
    assert orc.rel_fro(orc.sign_normalise(Rg), orc.sign_normalise(f.R)) <= TOL_R
    assert np.linalg.norm(Rg.T @ Rg - A0.T @ A0) / np.linalg.norm(A0) ** 2 <= 1e-14
    _check_reflectors(_np(Ad), tree, p, f, n)
    assert orc.rel_fro(_np(Cd), orc.tsqr_apply_qt(f, C0)) <= TOL_R
    tree.free()


def _gram_check(A, R):
    """||R^T R - A^T A||_F / ||A||_F^2 with A (n, m) column-major and R (n, n) column-major."""
    G = A @ A.T                                   # A^T A of the m x n matrix
    Rm = R.T                                      # the matrix R
    return (torch.linalg.norm(Rm.T @ Rm - G) / torch.linalg.norm(A) ** 2).item()


def test_full_c2_plain_plan():
    """C2 R and Q against the oracle's plain paper plan (one DGEQR2 per 4096-row block,
    the binary tree over the 245 blocks): plan-independent."""
    m, n, b, s, _ = _cfg("c2")
    At = inputs.gaussian(m, n, 0)
    A0 = _np(At).copy()
    Ad = At.cuda()
    R, tree = T.factor(Ad, b, s)
    Q = T.form_q(tree)
    torch.cuda.synchronize()
    f = orc.tsqr_factor(A0, orc.plan(m, n, b, 0, 1, 0), threads=THREADS)
    Rg, Qg = _np(R), _np(Q)
    assert orc.rel_fro(orc.sign_normalise(Rg), orc.sign_normalise(f.R)) <= TOL_R
    assert orc.rel_fro(_sign_q(Rg, Qg), _sign_q(f.R, orc.tsqr_form_q(f))) <= TOL_R
    tree.free()


@pytest.mark.parametrize("cfg", ["c4", "c5"])
def test_full_r_parity_oracle(cfg):
    """north_star: GPU R within 1e-11 (relative Frobenius, rows sign-normalised) of the
    oracle's R at the full C4 (kappa = 1e10) and C5 sizes, in the kernel's plan and in
    the plain plan."""
    m, n, b, s, _ = _cfg(cfg)
    if cfg == "c4":
        A = inputs.conditioned_rows(0, m, n, 0, 1e10, 2, "cuda")
    else:
        A = inputs.gaussian_rows(0, m, n, 0, "cuda")
    Ad = A.clone()
    R, tree = T.factor(Ad, b, s)
    torch.cuda.synchronize()
    Rg = orc.sign_normalise(_np(R))
    tree.free()
    del Ad
    torch.cuda.empty_cache()
    for p in (orc.plan(m, n, b, s, 1, _c(m, n, b, s)), orc.plan(m, n, b, 0, 1, 0)):
        Ro = _oracle_r_full(A, p)
        err = orc.rel_fro(Rg, orc.sign_normalise(Ro))
        print(f"{cfg} R vs oracle (c={p.c}, {p.ntiles} leaves): {err:.3e}")
        assert err <= TOL_R


def test_full_c4_invariants():
    m, n, b, s, _ = _cfg("c4")
    A = inputs.conditioned_rows(0, m, n, 0, 1e10, 2, "cuda")    # G diag(sigma) V^T, kappa = 1e10
    Ad = A.clone()
    R, tree = T.factor(Ad, b, s)
    Q = T.form_q(tree)
    torch.cuda.synchronize()
    Rm = R.T
    assert torch.all(torch.tril(Rm, -1) == 0)
    assert _gram_check(A, R) <= 1e-13
    Qt = Q.T
    assert (torch.linalg.norm(A.T - Qt @ Rm) / torch.linalg.norm(A)).item() <= TOL_INV
    assert torch.linalg.norm(Qt.T @ Qt - torch.eye(n, dtype=torch.float64, device="cuda")).item() <= TOL_INV
    tree.free()


def test_full_c5_apply_invariants():
    m, n, b, s, k = _cfg("c5")
    A = inputs.gaussian_rows(0, m, n, 0, "cuda")
    Ad = A.clone()
    R, tree = T.factor(Ad, b, s)
    C = inputs.gaussian_rows(0, m, k, 1, "cuda")
    Cd = C.clone()
    T.apply_qt(tree, Cd)
    torch.cuda.synchronize()
    assert _gram_check(A, R) <= 1e-13
    # Q orthogonal: every column of C keeps its norm
    nc, nq = torch.linalg.norm(C, dim=1), torch.linalg.norm(Cd, dim=1)
    assert (torch.max(torch.abs(nq - nc) / nc)).item() <= 1e-13
    # thin part (rows 0..n-1 of the tree-order result) = Q_thin^T C = R^-T (A^T C)
    AtC = A @ C.T                                 # (n, k) = A^T C
    Rm = R.T
    thin = torch.linalg.solve_triangular(Rm.T, AtC, upper=False)
    got = Cd[:, :n].T                             # rows 0..n-1 of the result, (n, k)
    assert (torch.linalg.norm(got - thin) / torch.linalg.norm(thin)).item() <= TOL_R
    tree.free()
