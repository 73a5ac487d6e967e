"""oracle -- TEST INFRASTRUCTURE ONLY.

ctypes/numpy front end of the plain C oracle in ``oracle.c`` (see ``oracle.h`` for
the paper passages each function follows).  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py`` (its ``cpu_baseline`` leg and its
``--impl reference`` arm) may import this package.  It shares no code with the
CUDA product path in ``paper_0808_2664_b200/``.

All matrices are numpy float64 arrays in Fortran (column-major) order.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_HDR = os.path.join(_HERE, "oracle.h")
_LIB = os.path.join(_HERE, "liboracle.so")
CFLAGS = ["-O2", "-fno-fast-math", "-ffp-contract=off", "-fPIC", "-shared", "-std=c11"]


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (plain C11, no BLAS)."""
    newest = max(os.path.getmtime(_SRC), os.path.getmtime(_HDR))
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < newest:
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.run(["gcc", *CFLAGS, "-pthread", "-o", tmp, _SRC, "-lm"], check=True)
        os.replace(tmp, _LIB)
    return _LIB


_lib = None
_i64 = ctypes.c_int64
_pd = ctypes.POINTER(ctypes.c_double)
_pi = ctypes.POINTER(ctypes.c_int64)


def lib():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        _lib.orc_plan_count.restype = ctypes.c_int
        _lib.orc_plan_fill.restype = ctypes.c_int
        _lib.orc_cholqr.restype = ctypes.c_int
    return _lib


def _d(a: np.ndarray):
    assert a.dtype == np.float64
    return a.ctypes.data_as(_pd)


def _i(a: np.ndarray):
    assert a.dtype == np.int64
    return a.ctypes.data_as(_pi)


def _fortran(a) -> np.ndarray:
    return np.asfortranarray(np.array(a, dtype=np.float64, copy=True))


def _ld(a: np.ndarray) -> int:
    assert a.flags.f_contiguous
    return max(1, a.shape[0])


# ----------------------------------------------------------------- kernels
def house(x):
    """Returns (v, tau, beta) with v[0] = 1 (LAPACK dlarfg convention)."""
    x = np.array(x, dtype=np.float64, copy=True)
    tau = ctypes.c_double()
    beta = ctypes.c_double()
    lib().orc_house(_i64(len(x)), _d(x), ctypes.byref(tau), ctypes.byref(beta))
    v = x.copy()
    v[0] = 1.0
    return v, tau.value, beta.value


def hqr(A):
    """Unblocked Householder QR. Returns (F, tau): F upper = R, strictly lower = v's."""
    F = _fortran(A)
    m, n = F.shape
    tau = np.zeros(n)
    lib().orc_hqr(_i64(m), _i64(n), _d(F), _i64(_ld(F)), _d(tau))
    return F, tau


def chain_qr(A, c: int = 0):
    """Flat-chain QR of one tile over c-row chunks (orc_chain_qr).
    Returns (F, tau): F upper (first n rows) = R, below the diagonal = reflector
    tails; tau (nchunks x n)."""
    F = _fortran(A)
    m, n = F.shape
    nch = 1 if c <= 0 else -(-m // c)
    tau = np.zeros((nch, n))
    lib().orc_chain_qr(_i64(m), _i64(n), _d(F), _i64(_ld(F)), _i64(c), _d(tau))
    return F, tau


def combine(Ra, Rb):
    """Structured QR of [Ra; Rb]. Returns (R, Y1, tau, flops)."""
    a = _fortran(Ra)
    b = _fortran(Rb)
    n = a.shape[0]
    tau = np.zeros(n)
    fl = ctypes.c_double()
    lib().orc_combine(_i64(n), _d(a), _i64(n), _d(b), _i64(n), _d(tau), ctypes.byref(fl))
    return np.triu(a), np.triu(b), tau, fl.value


def combine_q(Rs):
    """Alg. QR:qnxn ([TR] P:1957-1979): structured Householder QR of q stacked n x n upper
    triangles [R_1; ...; R_q], column by column: I_j = {j} U {rows 0..j of R_2} U ... U
    {rows 0..j of R_q}; w = A(I_j, j); [tau_j, v] = House(w) (v(1) = 1); A(I_j, j+1:n) :=
    (I - tau_j v v^T) A(I_j, j+1:n); v(2:end) scattered back into A(I_j minus {j}, j).
    Returns (R, [Y_2, ..., Y_q] (upper triangles holding the v parts), tau); (2/3)(q-1)n^3 flops."""
    q = len(Rs)
    n = Rs[0].shape[0]
    A = np.vstack([np.triu(np.asarray(R, dtype=np.float64)) for R in Rs])
    tau = np.zeros(n)
    for j in range(n):
        I = [j] + [i * n + r for i in range(1, q) for r in range(j + 1)]
        v, t, beta = house(A[I, j])
        X = A[np.ix_(I, range(j + 1, n))]
        A[np.ix_(I, range(j + 1, n))] = X - t * np.outer(v, v @ X)
        A[I[1:], j] = v[1:]
        A[j, j] = beta
        tau[j] = t
    return np.triu(A[:n]), [np.triu(A[i * n:(i + 1) * n]) for i in range(1, q)], tau


def build_t(Y, tau):
    """T (k x k) with H_0...H_{k-1} = I - Y T Y^T, Y unit lower trapezoidal."""
    Y = _fortran(Y)
    rows, k = Y.shape
    T = np.zeros((k, k), order="F")
    tau = np.ascontiguousarray(tau, dtype=np.float64)
    lib().orc_build_t(_i64(rows), _i64(k), _d(Y), _i64(_ld(Y)), _d(tau), _d(T), _i64(k))
    return T


def build_t_node(Y1, tau):
    Y1 = _fortran(Y1)
    n = Y1.shape[0]
    T = np.zeros((n, n), order="F")
    tau = np.ascontiguousarray(tau, dtype=np.float64)
    lib().orc_build_t_node(_i64(n), _d(Y1), _i64(n), _d(tau), _d(T), _i64(n))
    return T


def mgs_ld(A):
    A = _fortran(A)
    m, n = A.shape
    Q = np.zeros((m, n), order="F")
    R = np.zeros((n, n), order="F")
    lib().orc_mgs_ld(_i64(m), _i64(n), _d(A), _i64(m), _d(Q), _i64(m), _d(R), _i64(n))
    return Q, R


def cholqr(A, want_q: bool = True):
    """Alg. CholeskyQR (the comparison method, orc_cholqr).  Returns (info, R, Q or None)."""
    A = _fortran(A)
    m, n = A.shape
    R = np.zeros((n, n), order="F")
    Q = np.zeros((m, n), order="F") if want_q else None
    info = lib().orc_cholqr(_i64(m), _i64(n), _d(A), _i64(m), _d(R), _i64(n),
                            _d(Q) if want_q else None, _i64(m))
    return int(info), R, Q


# ------------------------------------------------------------------- plan
@dataclass
class Plan:
    m: int
    n: int
    b: int
    s: int
    G: int
    tile_row0: np.ndarray
    tile_rows: np.ndarray
    tile_rank: np.ndarray
    node_a: np.ndarray
    node_b: np.ndarray
    node_stage: np.ndarray
    node_level: np.ndarray
    c: int = 0                 # chunk rows of the tiles' flat chains (0: one chunk per tile)

    @property
    def ntiles(self) -> int:
        return len(self.tile_row0)

    @property
    def tile_chunk0(self) -> np.ndarray:
        """First chunk of every tile (+ the total), the row index into tau_tile."""
        k = np.ones_like(self.tile_rows) if self.c <= 0 else -(-self.tile_rows // self.c)
        return np.concatenate([[0], np.cumsum(k)]).astype(np.int64)

    @property
    def nnodes(self) -> int:
        return len(self.node_a)


def plan(m: int, n: int, b: int, s: int | None = None, G: int = 1, c: int = 0) -> Plan:
    s = 0 if s is None else s
    nt, nn = _i64(), _i64()
    rc = lib().orc_plan_count(_i64(m), _i64(n), _i64(b), _i64(s), _i64(G),
                              ctypes.byref(nt), ctypes.byref(nn))
    if rc != 0:
        raise ValueError(f"invalid TSQR shape m={m} n={n} b={b} s={s} G={G}")
    arr = [np.zeros(nt.value, np.int64) for _ in range(3)] + \
          [np.zeros(nn.value, np.int64) for _ in range(4)]
    rc = lib().orc_plan_fill(_i64(m), _i64(n), _i64(b), _i64(s), _i64(G), *[_i(x) for x in arr])
    assert rc == 0
    return Plan(m, n, b, s, G, *arr, c=c)


# ------------------------------------------------------------------- TSQR
@dataclass
class Factor:
    plan: Plan
    A: np.ndarray          # overwritten A (tile reflectors below the tile diagonals)
    tau_tile: np.ndarray   # nchunks x n (plan.tile_chunk0 indexes the tiles)
    Y1: np.ndarray         # nnodes x n x n (each column-major n x n, upper)
    tau_node: np.ndarray   # nnodes x n
    R: np.ndarray          # n x n


def _plan_args(p: Plan):
    return (_i64(p.ntiles), _i(p.tile_row0), _i(p.tile_rows),
            _i64(p.nnodes), _i(p.node_a), _i(p.node_b))


def tsqr_factor(A, p: Plan, threads: int = 1, overwrite: bool = False, keep_y1: bool = True) -> Factor:
    """TSQR over the plan p.  threads > 1 runs the leaf QRs (Eq. 1, independent per
    leaf) on that many host threads (orc_tsqr_factor_mt, bitwise the same result);
    overwrite=True factors A itself (a Fortran-ordered float64 array) instead of a
    copy, keep_y1=False skips the node factors (nnodes x n^2 words) -- both for
    full-size checks whose matrices are GBs."""
    F = A if (overwrite and isinstance(A, np.ndarray) and A.dtype == np.float64 and A.flags.f_contiguous) \
        else _fortran(A)
    m, n = F.shape
    assert m == p.m and n == p.n
    tau_tile = np.zeros((int(p.tile_chunk0[-1]), n))
    Y1 = np.zeros((max(p.nnodes, 1), n * n)) if keep_y1 else None
    tau_node = np.zeros((max(p.nnodes, 1), n))
    R = np.zeros((n, n), order="F")
    lib().orc_tsqr_factor_mt(_i64(m), _i64(n), _d(F), _i64(_ld(F)), _i64(p.c), *_plan_args(p),
                             _d(tau_tile), _d(Y1) if keep_y1 else None, _d(tau_node), _d(R), _i64(n),
                             _i64(max(1, int(threads))))
    return Factor(p, F, tau_tile, Y1, tau_node, R)


def _factor_args(f: Factor):
    return (_d(f.A), _i64(_ld(f.A)), _i64(f.plan.c), *_plan_args(f.plan), _d(f.tau_tile), _d(f.Y1),
            _d(f.tau_node))


def tsqr_apply_qt(f: Factor, C) -> np.ndarray:
    C = _fortran(C)
    k = C.shape[1]
    lib().orc_tsqr_apply_qt(_i64(f.plan.m), _i64(f.plan.n), *_factor_args(f), _d(C), _i64(_ld(C)), _i64(k))
    return C


def tsqr_apply_q(f: Factor, C) -> np.ndarray:
    C = _fortran(C)
    k = C.shape[1]
    lib().orc_tsqr_apply_q(_i64(f.plan.m), _i64(f.plan.n), *_factor_args(f), _d(C), _i64(_ld(C)), _i64(k))
    return C


def tsqr_form_q(f: Factor) -> np.ndarray:
    Q = np.zeros((f.plan.m, f.plan.n), order="F")
    lib().orc_tsqr_form_q(_i64(f.plan.m), _i64(f.plan.n), *_factor_args(f), _d(Q), _i64(_ld(Q)))
    return Q


def node_y1(f: Factor, k: int) -> np.ndarray:
    n = f.plan.n
    return f.Y1[k].reshape(n, n, order="F")


# -------------------------------------------------- sequential (streamed) TSQR
def slab_ranges(m: int, n: int, slab_rows: int):
    """Row slabs of the streamed TSQR: slab_rows each from row 0; a remainder of fewer than n
    rows is merged into the last slab (the row-block rule of reading R6 at slab granularity)."""
    full, rem = divmod(m, slab_rows)
    if full == 0:
        return [(0, m)]
    out = [(k * slab_rows, slab_rows) for k in range(full)]
    if rem >= n:
        out.append((full * slab_rows, rem))
    elif rem:
        out[-1] = (out[-1][0], slab_rows + rem)
    return out


def sequential_tsqr_r(A, slab_rows: int, b: int, s: int | None = None, c: int = 0) -> np.ndarray:
    """R of A by sequential TSQR over row slabs (flat tree; [TR] Alg. sequential TSQR
    P:1725-1753, flat tree P:954-993): each slab's R by the (parallel) TSQR of its rows with
    the plan (b, s, c), then R <- structured QR of [R; R_slab] (Alg. QR:qnxn with q = 2)."""
    F = np.asarray(A, dtype=np.float64)
    m, n = F.shape
    R = None
    for r0, rows in slab_ranges(m, n, slab_rows):
        f = tsqr_factor(np.array(F[r0:r0 + rows], order="F"), plan(rows, n, b, s, 1, c))
        R = f.R if R is None else combine(R, f.R)[0]
    return R


# ------------------------------------------------------------------- CAQR
@dataclass
class CaqrFactor:
    m: int
    N: int
    panel: int
    panels: list           # (c0, Factor of the panel's TSQR over rows c0..m-1)
    R: np.ndarray          # N x N upper triangular


def caqr_factor(A, panel: int, b: int, s: int | None = None, chunk=lambda w: 0) -> CaqrFactor:
    """Right-looking CAQR with TSQR panels on one processor column: "CAQR simply implements
    the right-looking QR factorization using ... TSQR as the panel factorization" (Sec. 3,
    P:2944-2946); Alg. CAQR:j ([TR] P:3992-4048) with one process row: panel j (columns
    c0..c0+w-1, rows c0..m-1) is factored by TSQR (line 1), then Q_j^T is applied to the
    trailing columns (line 3 and the tree stages of lines 4-9, i.e. tsqr_apply_qt); rows
    c0..c0+w-1 of the updated trailing block are R's row block, rows c0+w.. (tree order)
    are the next panel's input.  chunk(w) gives the leaves' chunk height for a panel of
    width w (the plan parameter c of reading R20)."""
    W = np.array(A, dtype=np.float64, order="F", copy=True)
    m, N = W.shape
    R = np.zeros((N, N), order="F")
    panels = []
    for c0 in range(0, N, panel):
        w = min(panel, N - c0)
        f = tsqr_factor(np.array(W[c0:, c0:c0 + w], order="F"), plan(m - c0, w, b, s, 1, chunk(w)))
        R[c0:c0 + w, c0:c0 + w] = f.R
        if c0 + w < N:
            T = tsqr_apply_qt(f, np.array(W[c0:, c0 + w:], order="F"))
            W[c0:, c0 + w:] = T
            R[c0:c0 + w, c0 + w:] = T[:w]
        panels.append((c0, f))
    return CaqrFactor(m, N, panel, panels, R)


def caqr_apply_qt(cf: CaqrFactor, C) -> np.ndarray:
    """C <- Q^T C = Q_p^T ... Q_1^T C, Q_j acting on rows c0_j..m-1 (tree order)."""
    C = np.array(C, dtype=np.float64, order="F", copy=True)
    for c0, f in cf.panels:
        C[c0:] = tsqr_apply_qt(f, np.array(C[c0:], order="F"))
    return C


def caqr_apply_q(cf: CaqrFactor, C) -> np.ndarray:
    """C <- Q C = Q_1 ... Q_p C (the panels in reverse order)."""
    C = np.array(C, dtype=np.float64, order="F", copy=True)
    for c0, f in reversed(cf.panels):
        C[c0:] = tsqr_apply_q(f, np.array(C[c0:], order="F"))
    return C


def caqr_form_q(cf: CaqrFactor) -> np.ndarray:
    """Explicit thin Q = Q [I_N; 0] (m x N)."""
    E = np.zeros((cf.m, cf.N), order="F")
    E[:cf.N] = np.eye(cf.N)
    return caqr_apply_q(cf, E)


# --------------------------------------------------------------- checkers
def sign_normalise(R, Q=None):
    """R^ = diag(s) R, Q^ = Q diag(s), s = sign(diag R) (sign(0)=+1) -- reading R9."""
    s = np.where(np.diag(R) < 0, -1.0, 1.0)
    Rn = R * s[:, None]
    if Q is None:
        return Rn
    return Rn, Q * s[None, :]


def rel_fro(X, Y) -> float:
    """||X - Y||_F / ||Y||_F, both scaled by max|Y| first so that the squares neither
    overflow nor underflow (inputs near the fp64 range limits, reading R23)."""
    X, Y = np.asarray(X, dtype=np.float64), np.asarray(Y, dtype=np.float64)
    s = float(np.max(np.abs(Y))) if Y.size else 0.0
    if not np.isfinite(s) or s == 0.0:
        s = 1.0
    d = np.linalg.norm(X / s - Y / s)
    nrm = np.linalg.norm(Y / s)
    return float(d / nrm) if nrm > 0 else float(d)
