"""ctypes binding of libtsqr.so (include/tsqr.h).  Argument marshalling only:
every numeric step runs in the library's CUDA kernels.  There is no fallback:
if the library is missing or fails to load, this raises."""
from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# developer override (A/B builds of the same sources); the default is the in-tree build
LIB_PATH = os.environ.get("TSQR_LIBRARY", os.path.join(HERE, "libtsqr.so"))

TSQR_OK = 0
STATUS = {0: "TSQR_OK", 1: "TSQR_ERR_INVALID", 2: "TSQR_ERR_SHAPE", 3: "TSQR_ERR_UNSUPPORTED",
          4: "TSQR_ERR_ALLOC", 5: "TSQR_ERR_CUDA", 6: "TSQR_ERR_NCCL"}
MAX_N = 256

# every symbol include/tsqr.h declares
SYMBOLS = ["tsqr_status_string", "tsqr_last_error", "tsqr_slab", "tsqr_plan_info", "tsqr_plan_export",
           "tsqr_cross_partner", "tsqr_factor", "tsqr_pack_r", "tsqr_cross_factor", "tsqr_cross_factor_gathered", "tsqr_apply_qt",
           "tsqr_cross_apply_qt", "tsqr_apply_q", "tsqr_cross_apply_q", "tsqr_form_q", "tsqr_tree_free", "tsqr_tree_export_tau",
           "tsqr_tree_stage_ms", "tsqr_caqr_factor", "tsqr_caqr_apply_qt", "tsqr_caqr_apply_q",
           "tsqr_caqr_form_q", "tsqr_caqr_free", "tsqr_factor_streamed", "tsqr_combine_stacked",
           "tsqr_ctx_create", "tsqr_get_unique_id", "tsqr_ctx_set_comm", "tsqr_loopback_create",
           "tsqr_loopback_destroy", "tsqr_ctx_set_loopback", "tsqr_ctx_info", "tsqr_ctx_destroy", "tsqr_ctx_factor",
           "tsqr_ctx_apply_qt", "tsqr_ctx_apply_q", "tsqr_ctx_form_q", "tsqr_measure_fp64_peak",
           "tsqr_qr_host", "tsqr_host_ws_free", "tsqr_cholqr", "tsqr_ctx_cholqr",
           "tsqr_factor_streamed_q", "tsqr_streamed_apply_qt", "tsqr_streamed_apply_q", "tsqr_streamed_form_q",
           "tsqr_stream_tree_free"]


class TsqrError(RuntimeError):
    def __init__(self, status: int, where: str, detail: str = ""):
        self.status = status
        super().__init__(f"{where}: {STATUS.get(status, status)}" + (f" ({detail})" if detail else ""))


class Opts(ctypes.Structure):
    _fields_ = [("block_rows", ctypes.c_int64), ("tile_rows", ctypes.c_int64), ("nranks", ctypes.c_int32),
                ("rank", ctypes.c_int32), ("flags", ctypes.c_int32), ("reserved", ctypes.c_int32)]


class PlanInfo(ctypes.Structure):
    _fields_ = [(f, ctypes.c_int64) for f in
                ("m_local", "n", "block_rows", "tile_rows", "ntiles", "nnodes", "nblocks", "depth",
                 "cross_rounds", "max_tile_rows", "min_tile_rows", "tile_capacity", "chunk_rows", "nchunks")]


_lib = None
_i64 = ctypes.c_int64
_i32 = ctypes.c_int32
_vp = ctypes.c_void_p
_pi64 = ctypes.POINTER(ctypes.c_int64)
_pi32 = ctypes.POINTER(ctypes.c_int32)
_pd = ctypes.POINTER(ctypes.c_double)


def lib():
    """Load libtsqr.so (building it if this checkout has nvcc and no library yet)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        from . import _build
        _build.build()
    L = ctypes.CDLL(LIB_PATH)
    L.tsqr_status_string.restype = ctypes.c_char_p
    L.tsqr_status_string.argtypes = [ctypes.c_int]
    L.tsqr_last_error.restype = ctypes.c_char_p
    L.tsqr_last_error.argtypes = []
    sig = {
        "tsqr_slab": [_i64, _i64, _i64, _i32, _i32, _pi64, _pi64],
        "tsqr_plan_info": [_i64, _i64, ctypes.POINTER(Opts), ctypes.POINTER(PlanInfo)],
        "tsqr_plan_export": [_i64, _i64, ctypes.POINTER(Opts), _pi64, _pi64, _pi64, _pi64, _pi64, _pi64],
        "tsqr_cross_partner": [_i32, _i32, _i32, _pi32, _pi32, _pi32],
        "tsqr_factor": [_i64, _i64, _vp, _i64, _vp, _i64, ctypes.POINTER(Opts), _vp, ctypes.POINTER(_vp)],
        "tsqr_pack_r": [_vp, _vp, _vp],
        "tsqr_cross_factor": [_vp, _i32, _vp, _vp, _i64, _vp],
        "tsqr_cross_factor_gathered": [_vp, _vp, _vp, _i64, _vp],
        "tsqr_apply_qt": [_vp, _vp, _i64, _i64, _vp, _i64, _vp],
        "tsqr_cross_apply_qt": [_vp, _i32, _vp, _i64, _vp, _vp, _i64, _i64, _vp],
        "tsqr_apply_q": [_vp, _vp, _i64, _i64, _vp],
        "tsqr_cross_apply_q": [_vp, _i32, _vp, _i64, _vp, _vp, _i64, _i64, _vp],
        "tsqr_form_q": [_vp, _vp, _i64, _vp],
        "tsqr_tree_free": [_vp],
        "tsqr_tree_export_tau": [_vp, _vp, _vp],
        "tsqr_tree_stage_ms": [_vp, _vp, _vp],
        "tsqr_caqr_factor": [_i64, _i64, _vp, _i64, _i64, _vp, _i64, ctypes.POINTER(Opts), _vp, ctypes.POINTER(_vp)],
        "tsqr_caqr_apply_qt": [_vp, _vp, _i64, _i64, _vp],
        "tsqr_caqr_apply_q": [_vp, _vp, _i64, _i64, _vp],
        "tsqr_caqr_form_q": [_vp, _vp, _i64, _vp],
        "tsqr_caqr_free": [_vp],
        "tsqr_combine_stacked": [_i32, _i64, _vp, _vp, _vp],
        "tsqr_factor_streamed": [_i64, _i64, _vp, _i64, _i64, _vp, _i64, _vp, _i64, ctypes.POINTER(Opts), _vp],
        "tsqr_ctx_create": [ctypes.c_int, ctypes.POINTER(_vp)],
        "tsqr_get_unique_id": [_vp],
        "tsqr_ctx_set_comm": [_vp, _vp, _i32, _i32],
        "tsqr_loopback_create": [_i32, ctypes.POINTER(_vp)],
        "tsqr_loopback_destroy": [_vp],
        "tsqr_ctx_set_loopback": [_vp, _vp, _i32],
        "tsqr_ctx_info": [_vp, _pi32, _pi32],
        "tsqr_ctx_destroy": [_vp],
        "tsqr_ctx_factor": [_vp, _i64, _i64, _vp, _i64, _vp, _i64, ctypes.POINTER(Opts), _vp, ctypes.POINTER(_vp)],
        "tsqr_ctx_apply_qt": [_vp, _vp, _vp, _i64, _i64, _vp, _i64, _vp],
        "tsqr_ctx_apply_q": [_vp, _vp, _vp, _i64, _i64, _vp],
        "tsqr_ctx_form_q": [_vp, _vp, _vp, _i64, _vp],
        "tsqr_measure_fp64_peak": [_pd, _pd, _vp],
        "tsqr_qr_host": [ctypes.POINTER(_vp), _i64, _i64, _vp, _i64, _vp, _i64, _vp, _i64, _vp, _i64, _i64,
                         ctypes.POINTER(Opts), _vp],
        "tsqr_host_ws_free": [_vp],
        "tsqr_cholqr": [_i64, _i64, _vp, _i64, _vp, _i64, _vp, _i64, _vp, _vp],
        "tsqr_ctx_cholqr": [_vp, _i64, _i64, _vp, _i64, _vp, _i64, _vp, _i64, _vp, _vp],
        "tsqr_factor_streamed_q": [_i64, _i64, _vp, _i64, _i64, _vp, _i64, _vp, _i64, ctypes.POINTER(Opts), _vp,
                                   ctypes.POINTER(_vp)],
        "tsqr_streamed_apply_qt": [_vp, _vp, _i64, _i64, _vp, _i64, _vp],
        "tsqr_streamed_apply_q": [_vp, _vp, _i64, _i64, _vp],
        "tsqr_streamed_form_q": [_vp, _vp, _i64, _vp],
        "tsqr_stream_tree_free": [_vp],
    }
    for name, args in sig.items():
        if "TSQR_LIBRARY" in os.environ and not hasattr(L, name):
            continue                              # an older A/B build: its own symbols only
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = ctypes.c_int
    _lib = L
    return L


def check(status: int, where: str) -> None:
    if status != TSQR_OK:
        detail = lib().tsqr_last_error().decode() if status in (5, 6) else ""
        raise TsqrError(status, where, detail)
