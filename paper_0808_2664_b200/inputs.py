"""Seeded synthetic inputs.  Holds none of the TSQR
arithmetic; shared by the product tests, the bench and the oracle checks.

Matrices are returned column-major as torch tensors of shape (ncols, nrows)
(row i, column j of the m x n matrix is t[j, i]), the layout of include/tsqr.h.

N(0,1) entries are generated in chunks of CHUNK rows; chunk c of a matrix with
seed s uses a generator seeded with s*1_000_003 + c (reading R13), so any row
range -- in particular one rank's slab -- can be generated independently and
the bytes do not depend on how the rows are sharded.
"""
from __future__ import annotations

import math

import torch

CHUNK = 65536


def _gen(device, seed: int) -> torch.Generator:
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    return g


def gaussian_rows(row0: int, rows: int, ncols: int, seed: int, device="cpu") -> torch.Tensor:
    """Rows [row0, row0+rows) of an (unbounded) N(0,1) matrix with ncols columns."""
    out = torch.empty((ncols, rows), dtype=torch.float64, device=device)
    c0, c1 = row0 // CHUNK, (row0 + rows - 1) // CHUNK if rows > 0 else row0 // CHUNK - 1
    for c in range(c0, c1 + 1):
        g = _gen(device, seed * 1_000_003 + c)
        chunk = torch.randn((ncols, CHUNK), dtype=torch.float64, device=device, generator=g)
        lo = max(row0, c * CHUNK)
        hi = min(row0 + rows, (c + 1) * CHUNK)
        out[:, lo - row0:hi - row0] = chunk[:, lo - c * CHUNK:hi - c * CHUNK]
    return out


def gaussian(m: int, n: int, seed: int = 0, device="cpu") -> torch.Tensor:
    return gaussian_rows(0, m, n, seed, device)


def conditioned_factors(n: int, kappa: float = 1e10, vseed: int = 2):
    """sigma_i = kappa^(-i/(n-1)) (log-spaced 1 .. 1/kappa) and V orthogonal from the QR of a
    seeded N(0,1) n x n matrix (BASELINE.json config 4; reading R15).  CPU float64."""
    sig = torch.tensor([kappa ** (-(i / (n - 1))) if n > 1 else 1.0 for i in range(n)], dtype=torch.float64)
    g = _gen("cpu", vseed)
    V, _ = torch.linalg.qr(torch.randn((n, n), dtype=torch.float64, generator=g))
    return sig, V


def conditioned_rows(row0: int, rows: int, n: int, seed: int = 0, kappa: float = 1e10, vseed: int = 2,
                     device="cpu") -> torch.Tensor:
    """Rows of A = G diag(sigma) V^T with G = gaussian(seed): column-major (n, rows)."""
    sig, V = conditioned_factors(n, kappa, vseed)
    G = gaussian_rows(row0, rows, n, seed, device)          # (n, rows) = G^T
    M = (V * sig[None, :]).to(device)                        # V diag(sigma)
    return M @ G                                             # (A^T) = V diag(sigma) G^T


def conditioned(m: int, n: int, seed: int = 0, kappa: float = 1e10, vseed: int = 2, device="cpu") -> torch.Tensor:
    return conditioned_rows(0, m, n, seed, kappa, vseed, device)


def to_numpy_colmajor(t: torch.Tensor):
    """(ncols, nrows) column-major torch tensor -> numpy (nrows, ncols) Fortran-ordered array."""
    return t.detach().cpu().numpy().T


def from_numpy(a) -> torch.Tensor:
    import numpy as np
    return torch.from_numpy(np.ascontiguousarray(np.asarray(a, dtype=np.float64).T))


def flops_factor(m: int, n: int) -> float:
    """The metric's model numerator 2 m n^2 (BASELINE.json; Table 1)."""
    return 2.0 * m * n * n


def log2i(x: int) -> int:
    return int(math.log2(x))
