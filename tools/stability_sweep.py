"""SURVEY 8(f) row 4 (tools only, not the product): TSQR against CholeskyQR (Alg. CholeskyQR,
P:1408-1419: W = A^T A, W = L L^T, Q = A L^-T) over a condition-number grid on the C4 recipe
(A = G diag(sigma) V^T, sigma log-spaced 1 .. 1/kappa; reading R15), both on the GPU.  TSQR is
libtsqr.so (factor + form Q); CholeskyQR uses cuBLAS/cuSOLVER through torch (DGEMM for A^T A,
potrf, trsm) -- a comparison algorithm, timed as a library baseline.  Reports ||Q^T Q - I||_F,
||A - QR||_F / ||A||_F and device times (CUDA events, median of 3).
usage: python tools/stability_sweep.py [m] [n]"""
import sys

import torch

import paper_0808_2664_b200 as T
from paper_0808_2664_b200 import inputs

m = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 20
n = int(sys.argv[2]) if len(sys.argv) > 2 else 64
b, s = 4096, 4096 if n > 32 else 4096
I = torch.eye(n, dtype=torch.float64, device="cuda")


def timed(fn, reps=3):
    ts, out = [], None
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        out = fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return sorted(ts)[len(ts) // 2], out


def metrics(A, Qt, Rm):
    """A: (n, m) = A^T storage; Qt: (n, m) = Q^T; Rm: the n x n R as a matrix."""
    orth = torch.linalg.norm(Qt @ Qt.T - I).item()
    res = (torch.linalg.norm(A.T - Qt.T @ Rm) / torch.linalg.norm(A)).item()
    return orth, res


print(f"m={m} n={n}: kappa | TSQR orth  resid  ms | CholeskyQR orth  resid  ms | CholeskyQR2 orth ms")
for e in range(0, 16, 2):
    kappa = 10.0 ** e
    A = inputs.conditioned_rows(0, m, n, 0, kappa, 2, "cuda")
    R = torch.empty((n, n), dtype=torch.float64, device="cuda")
    Q = torch.empty((n, m), dtype=torch.float64, device="cuda")
    W = A.clone()
    hold = {"tree": None}

    def tsqr():
        W.copy_(A)
        _, hold["tree"] = T.factor(W, b, s, R=R, tree=hold["tree"])
        T.form_q(hold["tree"], Q)
        return Q

    t_ts, _ = timed(tsqr)
    o_ts, r_ts = metrics(A, Q, R.T)

    def chol(X):
        G = X @ X.T                                    # A^T A (n x n), DGEMM
        L, info = torch.linalg.cholesky_ex(G)
        if info.item() != 0:
            return None, None
        Qt = torch.linalg.solve_triangular(L, X, upper=False)   # Q^T = L^-1 A^T
        return Qt, L.T

    t_ch, (Qc, Rc) = timed(lambda: chol(A))
    if Qc is None:
        cq = "   breakdown (Cholesky of A^T A failed)"
    else:
        o_ch, r_ch = metrics(A, Qc, Rc)
        cq = f"  {o_ch:9.2e} {r_ch:9.2e} {t_ch:7.3f}"

    def chol2():
        Q1, R1 = chol(A)
        if Q1 is None:
            return None, None
        Q2, R2 = chol(Q1)
        return (None, None) if Q2 is None else (Q2, R2 @ R1)

    t_c2, (Q2, R2) = timed(chol2)
    c2 = "   breakdown" if Q2 is None else f"  {metrics(A, Q2, R2)[0]:9.2e} {t_c2:7.3f}"
    print(f"{kappa:8.0e} | {o_ts:9.2e} {r_ts:9.2e} {t_ts:7.3f} |{cq} |{c2}")
    hold["tree"].free()
