"""User-facing API of the B200 TSQR path (torch tensors in, torch tensors out).

Matrices are column-major: an m x n matrix is a float64 CUDA tensor of shape
(n, m) whose rows are the matrix columns (stride(1) == 1, lda = stride(0)).
Every call marshals pointers into libtsqr.so (include/tsqr.h); all arithmetic
runs in its sm_100a kernels.  Calls are asynchronous on the current stream.
"""
from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _lib
from ._lib import Opts, PlanInfo, check, lib


def _stream_ptr(stream=None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def _colmajor(t: torch.Tensor, name: str, host: bool = False):
    if t.dtype != torch.float64:
        raise TypeError(f"{name} must be float64")
    if host and t.is_cuda:
        raise TypeError(f"{name} must be a host (CPU) tensor")
    if not host and not t.is_cuda:
        raise TypeError(f"{name} must be a CUDA tensor (the product path has no CPU fallback)")
    if t.dim() != 2 or (t.shape[1] > 1 and t.stride(1) != 1):
        raise ValueError(f"{name} must be column-major: shape (ncols, nrows) with stride(1) == 1")
    ncols, nrows = t.shape
    ld = t.stride(0) if ncols > 1 else max(nrows, 1)
    return t.data_ptr(), nrows, ncols, ld


def opts(block_rows: int = 0, tile_rows: int = 0, nranks: int = 1, rank: int = 0, debug: bool = False,
         stage_timing: bool = False, robust: bool = False) -> Opts:
    """robust: TSQR_FLAG_ROBUST -- rescaled Householder steps for inputs outside [2^-400, 2^400]."""
    return Opts(block_rows, tile_rows, nranks, rank,
                (1 if debug else 0) | (2 if stage_timing else 0) | (4 if robust else 0), 0)


class Tree:
    """Implicit Q of one rank (the tree of Householder reflectors, Eq. 4).
    Borrows A (which holds the tile reflectors) until freed."""

    def __init__(self):
        self.handle = ctypes.c_void_p(None)
        self.A = None
        self.m_local = 0
        self.n = 0
        self.opts = None

    def free(self):
        if self.handle:
            lib().tsqr_tree_free(self.handle)
            self.handle = ctypes.c_void_p(None)
        self.A = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass

    def stage_ms(self):
        """(leaf_ms, tree_ms) of the last factor run with stage_timing=True (device events)."""
        a, b = ctypes.c_float(), ctypes.c_float()
        check(lib().tsqr_tree_stage_ms(self.handle, ctypes.byref(a), ctypes.byref(b)), "tsqr_tree_stage_ms")
        return a.value, b.value

    def export_tau(self):
        info = plan_info(self.m_local, self.n, self.opts)
        L, n = info["ntiles"], self.n
        tt = np.zeros((info["nchunks"], n))
        tn = np.zeros((L, n))
        check(lib().tsqr_tree_export_tau(self.handle, tt.ctypes.data_as(ctypes.c_void_p),
                                          tn.ctypes.data_as(ctypes.c_void_p)), "tsqr_tree_export_tau")
        return tt, tn


def factor(A: torch.Tensor, block_rows: int = 0, tile_rows: int = 0, R: torch.Tensor | None = None,
           nranks: int = 1, rank: int = 0, tree: Tree | None = None, stream=None, debug: bool = False,
           stage_timing: bool = False, robust: bool = False):
    """Factor A (column-major m_local x n) in place.  Returns (R, tree): R is n x n upper
    triangular as a column-major (n, n) tensor.  Pass `tree` back in to reuse its workspace.
    robust: rescaled steps for entries outside [2^-400, 2^400] (TSQR_FLAG_ROBUST)."""
    pa, m, n, lda = _colmajor(A, "A")
    if R is None:
        R = torch.empty((n, n), dtype=torch.float64, device=A.device)
    pr, _, _, ldr = _colmajor(R, "R")
    o = opts(block_rows, tile_rows, nranks, rank, debug, stage_timing, robust)
    t = tree if tree is not None else Tree()
    h = t.handle
    check(lib().tsqr_factor(m, n, pa, lda, pr, ldr, ctypes.byref(o), _stream_ptr(stream), ctypes.byref(h)),
          "tsqr_factor")
    t.handle = h
    t.A, t.m_local, t.n, t.opts = A, m, n, o
    return R, t


def apply_qt(tree: Tree, C: torch.Tensor, top: torch.Tensor | None = None, stream=None):
    """C <- Q^T C in tree order (in place).  Returns (C, top)."""
    pc, m, k, ldc = _colmajor(C, "C")
    if m != tree.m_local:
        raise ValueError("C must have m_local rows")
    ptop, ldtop = None, 0
    if top is not None:
        ptop, _, _, ldtop = _colmajor(top, "top")
    check(lib().tsqr_apply_qt(tree.handle, pc, ldc, k, ptop, ldtop, _stream_ptr(stream)), "tsqr_apply_qt")
    return C, top


def apply_q(tree: Tree, C: torch.Tensor, stream=None) -> torch.Tensor:
    """C <- Q C in place, C in tree order (the inverse of apply_qt; one-rank trees)."""
    pc, m, k, ldc = _colmajor(C, "C")
    if m != tree.m_local:
        raise ValueError("C must have m_local rows")
    check(lib().tsqr_apply_q(tree.handle, pc, ldc, k, _stream_ptr(stream)), "tsqr_apply_q")
    return C


def form_q(tree: Tree, Q: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    """Explicit thin Q rows of this rank (column-major m_local x n)."""
    if Q is None:
        Q = torch.empty((tree.n, tree.m_local), dtype=torch.float64, device=tree.A.device)
    pq, m, n, ldq = _colmajor(Q, "Q")
    check(lib().tsqr_form_q(tree.handle, pq, ldq, _stream_ptr(stream)), "tsqr_form_q")
    return Q


def pack_r(tree: Tree, packed: torch.Tensor, stream=None) -> torch.Tensor:
    check(lib().tsqr_pack_r(tree.handle, packed.data_ptr(), _stream_ptr(stream)), "tsqr_pack_r")
    return packed


def cross_factor(tree: Tree, rnd: int, partner_packed: torch.Tensor, R: torch.Tensor | None = None, stream=None):
    pr, ldr = None, 0
    if R is not None:
        pr, _, _, ldr = _colmajor(R, "R")
    check(lib().tsqr_cross_factor(tree.handle, rnd, partner_packed.data_ptr(), pr, ldr, _stream_ptr(stream)),
          "tsqr_cross_factor")
    return R


def cross_factor_gathered(tree: Tree, all_packed: torch.Tensor, R: torch.Tensor | None = None, stream=None):
    """Every butterfly round from the all-gathered packed leaf R's (rank i at i*n(n+1)/2)."""
    pr, ldr = None, 0
    if R is not None:
        pr, _, _, ldr = _colmajor(R, "R")
    check(lib().tsqr_cross_factor_gathered(tree.handle, all_packed.data_ptr(), pr, ldr, _stream_ptr(stream)),
          "tsqr_cross_factor_gathered")
    return R


def cross_apply_qt(tree: Tree, rnd: int, top: torch.Tensor, partner_top: torch.Tensor, C: torch.Tensor,
                   stream=None):
    ptop, _, k, ldtop = _colmajor(top, "top")
    pc, _, _, ldc = _colmajor(C, "C")
    check(lib().tsqr_cross_apply_qt(tree.handle, rnd, ptop, ldtop, partner_top.data_ptr(), pc, ldc, k,
                                    _stream_ptr(stream)), "tsqr_cross_apply_qt")
    return top


def cross_apply_q(tree: Tree, rnd: int, top: torch.Tensor, partner_top: torch.Tensor, C: torch.Tensor,
                  stream=None):
    """Butterfly round rnd of C <- Q C (group heads only): top <- this rank's half of
    Q_node [lower; upper], also written to C's head rows."""
    ptop, _, k, ldtop = _colmajor(top, "top")
    pc, _, _, ldc = _colmajor(C, "C")
    check(lib().tsqr_cross_apply_q(tree.handle, rnd, ptop, ldtop, partner_top.data_ptr(), pc, ldc, k,
                                   _stream_ptr(stream)), "tsqr_cross_apply_q")
    return top


def factor_streamed(A_host: torch.Tensor, slab_rows: int, block_rows: int = 0, tile_rows: int = 0,
                    R: torch.Tensor | None = None, Y_host: torch.Tensor | None = None, device=None,
                    stream=None) -> torch.Tensor:
    """R of a host-resident A (CPU tensor, column-major m x n; pin it for overlapped copies)
    streamed through the GPU in slabs of slab_rows (sequential TSQR).  Returns R on the device."""
    pa, m, n, lda = _colmajor(A_host, "A", host=True)
    if R is None:
        R = torch.empty((n, n), dtype=torch.float64, device=device or "cuda")
    pr, _, _, ldr = _colmajor(R, "R")
    py, ldy = None, 0
    if Y_host is not None:
        py, _, _, ldy = _colmajor(Y_host, "Y", host=True)
    o = opts(block_rows, tile_rows)
    check(lib().tsqr_factor_streamed(m, n, pa, lda, slab_rows, py, ldy, pr, ldr, ctypes.byref(o),
                                     _stream_ptr(stream)), "tsqr_factor_streamed")
    return R


class StreamTree:
    """Implicit Q of a streamed factor (tsqr_factor_streamed_q): slab trees' taus / T's and the
    flat-tree nodes in pinned host memory; borrows the host Y (the reflectors) until freed."""

    def __init__(self):
        self.handle = ctypes.c_void_p(None)
        self.Y = None
        self.m = self.n = 0

    def free(self):
        if self.handle:
            lib().tsqr_stream_tree_free(self.handle)
            self.handle = ctypes.c_void_p(None)
        self.Y = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


def factor_streamed_q(A_host: torch.Tensor, slab_rows: int, Y_host: torch.Tensor, block_rows: int = 0,
                      tile_rows: int = 0, R: torch.Tensor | None = None, device=None, stream=None):
    """Streamed factor keeping Q: returns (R on the device, StreamTree)."""
    pa, m, n, lda = _colmajor(A_host, "A", host=True)
    if R is None:
        R = torch.empty((n, n), dtype=torch.float64, device=device or "cuda")
    pr, _, _, ldr = _colmajor(R, "R")
    py, _, _, ldy = _colmajor(Y_host, "Y", host=True)
    o = opts(block_rows, tile_rows)
    st = StreamTree()
    h = st.handle
    check(lib().tsqr_factor_streamed_q(m, n, pa, lda, slab_rows, py, ldy, pr, ldr, ctypes.byref(o),
                                       _stream_ptr(stream), ctypes.byref(h)), "tsqr_factor_streamed_q")
    st.handle, st.Y, st.m, st.n = h, Y_host, m, n
    return R, st


def streamed_apply_qt(t: StreamTree, C_host: torch.Tensor, top: torch.Tensor | None = None, stream=None):
    pc, m, k, ldc = _colmajor(C_host, "C", host=True)
    ptop, ldtop = None, 0
    if top is not None:
        ptop, _, _, ldtop = _colmajor(top, "top", host=True)
    check(lib().tsqr_streamed_apply_qt(t.handle, pc, ldc, k, ptop, ldtop, _stream_ptr(stream)),
          "tsqr_streamed_apply_qt")
    return C_host


def streamed_apply_q(t: StreamTree, C_host: torch.Tensor, stream=None):
    pc, m, k, ldc = _colmajor(C_host, "C", host=True)
    check(lib().tsqr_streamed_apply_q(t.handle, pc, ldc, k, _stream_ptr(stream)), "tsqr_streamed_apply_q")
    return C_host


def streamed_form_q(t: StreamTree, Q_host: torch.Tensor | None = None, stream=None):
    if Q_host is None:
        Q_host = torch.empty((t.n, t.m), dtype=torch.float64).pin_memory()
    pq, _, _, ldq = _colmajor(Q_host, "Q", host=True)
    check(lib().tsqr_streamed_form_q(t.handle, pq, ldq, _stream_ptr(stream)), "tsqr_streamed_form_q")
    return Q_host


def combine_stacked(packed: torch.Tensor, q: int, n: int, tau: torch.Tensor | None = None, stream=None):
    """Alg. QR:qnxn on q packed triangles (device, q*n(n+1)/2, in place): slot 0 becomes R,
    slots 1.. the reflectors' v parts.  Returns tau (n)."""
    if not packed.is_cuda or packed.dtype != torch.float64 or packed.numel() != q * n * (n + 1) // 2:
        raise ValueError("packed must be a CUDA float64 tensor of q*n(n+1)/2 words")
    if tau is None:
        tau = torch.empty(n, dtype=torch.float64, device=packed.device)
    check(lib().tsqr_combine_stacked(q, n, packed.data_ptr(), tau.data_ptr(), _stream_ptr(stream)),
          "tsqr_combine_stacked")
    return tau


# ------------------------------------------------------------ communicator
class Ctx:
    """A libtsqr communicator context (one per process / GPU): the collective
    tsqr_ctx_* calls run every butterfly round inside the C library (NCCL grouped
    send/recv on the call's stream, or the in-process loopback of the tests)."""

    def __init__(self, device: int | None = None):
        self.handle = ctypes.c_void_p(None)
        self.device = torch.cuda.current_device() if device is None else device
        check(lib().tsqr_ctx_create(self.device, ctypes.byref(self.handle)), "tsqr_ctx_create")

    @staticmethod
    def unique_id() -> bytes:
        buf = ctypes.create_string_buffer(128)
        check(lib().tsqr_get_unique_id(buf), "tsqr_get_unique_id")
        return buf.raw

    def set_comm(self, uid: bytes, nranks: int, rank: int):
        if len(uid) != 128:
            raise ValueError("uid must be the 128 bytes of tsqr_get_unique_id")
        check(lib().tsqr_ctx_set_comm(self.handle, ctypes.create_string_buffer(uid, 128), nranks, rank),
              "tsqr_ctx_set_comm")
        return self

    def set_loopback(self, hub: "Loopback", rank: int):
        check(lib().tsqr_ctx_set_loopback(self.handle, hub.handle, rank), "tsqr_ctx_set_loopback")
        self._hub = hub                           # keep the hub alive
        return self

    def info(self):
        nr, rk = ctypes.c_int32(), ctypes.c_int32()
        check(lib().tsqr_ctx_info(self.handle, ctypes.byref(nr), ctypes.byref(rk)), "tsqr_ctx_info")
        return nr.value, rk.value

    def factor(self, A: torch.Tensor, block_rows: int = 0, tile_rows: int = 0, R: torch.Tensor | None = None,
               tree: Tree | None = None, stream=None, debug: bool = False, stage_timing: bool = False):
        """Collective factor of this rank's slab; R replicated.  Returns (R, tree)."""
        pa, m, n, lda = _colmajor(A, "A")
        if R is None:
            R = torch.empty((n, n), dtype=torch.float64, device=A.device)
        pr, _, _, ldr = _colmajor(R, "R")
        nr, rk = self.info()
        o = opts(block_rows, tile_rows, nr, rk, debug, stage_timing)
        t = tree if tree is not None else Tree()
        h = t.handle
        check(lib().tsqr_ctx_factor(self.handle, m, n, pa, lda, pr, ldr, ctypes.byref(o), _stream_ptr(stream),
                                    ctypes.byref(h)), "tsqr_ctx_factor")
        t.handle = h
        t.A, t.m_local, t.n, t.opts = A, m, n, o
        return R, t

    def apply_qt(self, tree: Tree, C: torch.Tensor, top: torch.Tensor | None = None, stream=None):
        pc, m, k, ldc = _colmajor(C, "C")
        ptop, ldtop = None, 0
        if top is not None:
            ptop, _, _, ldtop = _colmajor(top, "top")
        check(lib().tsqr_ctx_apply_qt(self.handle, tree.handle, pc, ldc, k, ptop, ldtop, _stream_ptr(stream)),
              "tsqr_ctx_apply_qt")
        return C, top

    def apply_q(self, tree: Tree, C: torch.Tensor, stream=None):
        pc, m, k, ldc = _colmajor(C, "C")
        check(lib().tsqr_ctx_apply_q(self.handle, tree.handle, pc, ldc, k, _stream_ptr(stream)), "tsqr_ctx_apply_q")
        return C

    def form_q(self, tree: Tree, Q: torch.Tensor | None = None, stream=None):
        if Q is None:
            Q = torch.empty((tree.n, tree.m_local), dtype=torch.float64, device=tree.A.device)
        pq, _, _, ldq = _colmajor(Q, "Q")
        check(lib().tsqr_ctx_form_q(self.handle, tree.handle, pq, ldq, _stream_ptr(stream)), "tsqr_ctx_form_q")
        return Q

    def cholqr(self, A: torch.Tensor, R: torch.Tensor | None = None, Q: torch.Tensor | None = None,
               want_q: bool = True, stream=None):
        """Collective CholeskyQR (tsqr_ctx_cholqr): R replicated, Q this rank's rows.
        Returns (R, Q or None, info) with info a device int32 tensor (0 = ok, j+1 = breakdown)."""
        return _cholqr(A, R, Q, want_q, stream, ctx=self)

    def free(self):
        if self.handle:
            lib().tsqr_ctx_destroy(self.handle)
            self.handle = ctypes.c_void_p(None)

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


class Loopback:
    """In-process exchange hub for G contexts of one process (tests): each rank's call
    synchronises its own stream before posting, so no kernel waits on another rank."""

    def __init__(self, nranks: int):
        self.handle = ctypes.c_void_p(None)
        check(lib().tsqr_loopback_create(nranks, ctypes.byref(self.handle)), "tsqr_loopback_create")

    def __del__(self):
        try:
            if self.handle:
                lib().tsqr_loopback_destroy(self.handle)
        except Exception:
            pass


def _cholqr(A, R, Q, want_q, stream, ctx=None):
    pa, m, n, lda = _colmajor(A, "A")
    if R is None:
        R = torch.empty((n, n), dtype=torch.float64, device=A.device)
    pr, _, _, ldr = _colmajor(R, "R")
    pq, ldq = None, 0
    if want_q:
        if Q is None:
            Q = torch.empty((n, m), dtype=torch.float64, device=A.device)
        pq, _, _, ldq = _colmajor(Q, "Q")
    info = torch.zeros(1, dtype=torch.int32, device=A.device)
    if ctx is None:
        check(lib().tsqr_cholqr(m, n, pa, lda, pr, ldr, pq, ldq, info.data_ptr(), _stream_ptr(stream)), "tsqr_cholqr")
    else:
        check(lib().tsqr_ctx_cholqr(ctx.handle, m, n, pa, lda, pr, ldr, pq, ldq, info.data_ptr(), _stream_ptr(stream)),
              "tsqr_ctx_cholqr")
    return R, (Q if want_q else None), info


def cholqr(A: torch.Tensor, R: torch.Tensor | None = None, Q: torch.Tensor | None = None, want_q: bool = True,
           stream=None):
    """CholeskyQR (tsqr_cholqr; Alg. CholeskyQR [TR] P:1410-1419) -- the comparison method
    of SURVEY 8(f) row 4, not TSQR.  A is read only.  Returns (R, Q or None, info) with
    info a device int32 tensor: 0, or j+1 when the Cholesky of A^T A broke down at j."""
    return _cholqr(A, R, Q, want_q, stream)


def measure_fp64_peak(stream=None):
    """(DMMA, DFMA) TFLOP/s of this GPU, measured now (tsqr_measure_fp64_peak)."""
    a, b = ctypes.c_double(), ctypes.c_double()
    check(lib().tsqr_measure_fp64_peak(ctypes.byref(a), ctypes.byref(b), _stream_ptr(stream)),
          "tsqr_measure_fp64_peak")
    return a.value, b.value


# ------------------------------------------------------------------- CAQR
class Caqr:
    """Right-looking CAQR with TSQR panels (tsqr_caqr_*): one panel tree per panel_cols
    columns.  Borrows A until freed."""

    def __init__(self):
        self.handle = ctypes.c_void_p(None)
        self.A = None
        self.m = self.N = self.panel = 0

    def free(self):
        if self.handle:
            lib().tsqr_caqr_free(self.handle)
            self.handle = ctypes.c_void_p(None)
        self.A = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


def caqr(A: torch.Tensor, panel_cols: int, block_rows: int = 0, tile_rows: int = 0, R: torch.Tensor | None = None,
         handle: Caqr | None = None, stream=None, debug: bool = False):
    """QR of A (column-major m x N) in place by CAQR.  Returns (R, handle)."""
    pa, m, N, lda = _colmajor(A, "A")
    if R is None:
        R = torch.empty((N, N), dtype=torch.float64, device=A.device)
    pr, _, _, ldr = _colmajor(R, "R")
    o = opts(block_rows, tile_rows, 1, 0, debug)
    c = handle if handle is not None else Caqr()
    h = c.handle
    check(lib().tsqr_caqr_factor(m, N, pa, lda, panel_cols, pr, ldr, ctypes.byref(o), _stream_ptr(stream),
                                 ctypes.byref(h)), "tsqr_caqr_factor")
    c.handle = h
    c.A, c.m, c.N, c.panel = A, m, N, panel_cols
    return R, c


def caqr_apply_qt(c: Caqr, C: torch.Tensor, stream=None) -> torch.Tensor:
    pc, m, k, ldc = _colmajor(C, "C")
    if m != c.m:
        raise ValueError("C must have m rows")
    check(lib().tsqr_caqr_apply_qt(c.handle, pc, ldc, k, _stream_ptr(stream)), "tsqr_caqr_apply_qt")
    return C


def caqr_apply_q(c: Caqr, C: torch.Tensor, stream=None) -> torch.Tensor:
    pc, m, k, ldc = _colmajor(C, "C")
    if m != c.m:
        raise ValueError("C must have m rows")
    check(lib().tsqr_caqr_apply_q(c.handle, pc, ldc, k, _stream_ptr(stream)), "tsqr_caqr_apply_q")
    return C


def caqr_form_q(c: Caqr, Q: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    if Q is None:
        Q = torch.empty((c.N, c.m), dtype=torch.float64, device=c.A.device)
    pq, _, _, ldq = _colmajor(Q, "Q")
    check(lib().tsqr_caqr_form_q(c.handle, pq, ldq, _stream_ptr(stream)), "tsqr_caqr_form_q")
    return Q


# ----------------------------------------------------------------- host-only
def plan_info(m_local: int, n: int, o: Opts | None = None, **kw) -> dict:
    o = o if o is not None else opts(**kw)
    info = PlanInfo()
    check(lib().tsqr_plan_info(m_local, n, ctypes.byref(o), ctypes.byref(info)), "tsqr_plan_info")
    return {f: getattr(info, f) for f, _ in PlanInfo._fields_}


def plan_export(m_local: int, n: int, **kw) -> dict:
    o = opts(**kw)
    info = plan_info(m_local, n, o)
    L, N = info["ntiles"], info["nnodes"]
    arrs = {k: np.zeros(L if k.startswith("tile") else max(N, 1), np.int64)
            for k in ("tile_row0", "tile_rows", "node_a", "node_b", "node_stage", "node_level")}
    ptr = lambda a: a.ctypes.data_as(_lib._pi64)  # noqa: E731
    check(lib().tsqr_plan_export(m_local, n, ctypes.byref(o), *[ptr(arrs[k]) for k in
                                 ("tile_row0", "tile_rows", "node_a", "node_b", "node_stage", "node_level")]),
          "tsqr_plan_export")
    for k in ("node_a", "node_b", "node_stage", "node_level"):
        arrs[k] = arrs[k][:N]
    return arrs


def slab(m: int, n: int, block_rows: int, nranks: int, rank: int):
    r0, ml = ctypes.c_int64(), ctypes.c_int64()
    check(lib().tsqr_slab(m, n, block_rows, nranks, rank, ctypes.byref(r0), ctypes.byref(ml)), "tsqr_slab")
    return r0.value, ml.value


def cross_partner(nranks: int, rank: int, rnd: int):
    p, lo, role = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32()
    check(lib().tsqr_cross_partner(nranks, rank, rnd, ctypes.byref(p), ctypes.byref(lo), ctypes.byref(role)),
          "tsqr_cross_partner")
    return p.value, bool(lo.value), role.value


# ----------------------------------------------------------------- end to end
class HostQR:
    """End-to-end QR of HOST matrices through one C call (tsqr_qr_host): copies in,
    factor, form Q / apply Q^T, copies out, on one GPU; the device workspace and tree
    are kept between calls of the same shape."""

    def __init__(self):
        self.ws = ctypes.c_void_p(None)

    def __call__(self, A_host: torch.Tensor, block_rows: int = 0, tile_rows: int = 0, R_host=None, Q_host=None,
                 C_host=None, want_q: bool = True, stream=None):
        pa, m, n, lda = _colmajor(A_host, "A", host=True)
        if R_host is None:
            R_host = torch.empty((n, n), dtype=torch.float64).pin_memory()
        pr, _, _, ldr = _colmajor(R_host, "R", host=True)
        pq, ldq = None, 0
        if want_q:
            if Q_host is None:
                Q_host = torch.empty((n, m), dtype=torch.float64).pin_memory()
            pq, _, _, ldq = _colmajor(Q_host, "Q", host=True)
        pc, ldc, k = None, 0, 0
        if C_host is not None:
            pc, _, k, ldc = _colmajor(C_host, "C", host=True)
        o = opts(block_rows, tile_rows)
        check(lib().tsqr_qr_host(ctypes.byref(self.ws), m, n, pa, lda, pr, ldr, pq, ldq, pc, ldc, k,
                                 ctypes.byref(o), _stream_ptr(stream)), "tsqr_qr_host")
        return R_host, Q_host, C_host

    def free(self):
        if self.ws:
            lib().tsqr_host_ws_free(self.ws)
            self.ws = ctypes.c_void_p(None)

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


def tsqr(A_host: torch.Tensor, block_rows: int = 0, tile_rows: int = 0, want_q: bool = True, stream=None):
    """End-to-end convenience call with HOST tensors (column-major (n, m), ideally pinned):
    returns (R, Q) in host memory (Q None unless want_q)."""
    h = HostQR()
    R, Q, _ = h(A_host, block_rows, tile_rows, want_q=want_q, stream=stream)
    h.free()
    return R, Q
