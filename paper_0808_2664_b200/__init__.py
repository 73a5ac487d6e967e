"""paper_0808_2664_b200 -- B200-native (sm_100a) Tall-Skinny QR after arXiv 0808.2664.

The hot path lives in libtsqr.so (csrc/, C-ABI include/tsqr.h); this package is
the thin Python binding (api.py) plus the multi-GPU butterfly driver (dist.py)
and the seeded input recipe (inputs.py)."""
from .api import (Caqr, Ctx, cholqr, StreamTree, factor_streamed_q, streamed_apply_q, streamed_apply_qt, streamed_form_q, HostQR, Loopback, Tree, measure_fp64_peak, caqr, caqr_apply_q, caqr_apply_qt, caqr_form_q, combine_stacked, factor_streamed, apply_q, apply_qt, cross_apply_q, cross_apply_qt, cross_factor, cross_partner, factor, form_q, pack_r,
                  plan_export, plan_info, slab, tsqr)

__all__ = ["cholqr", "StreamTree", "factor_streamed_q", "streamed_apply_q", "streamed_apply_qt", "streamed_form_q", "HostQR", "Ctx", "Loopback", "measure_fp64_peak", "Tree", "Caqr", "caqr", "caqr_apply_qt", "caqr_apply_q", "caqr_form_q", "factor_streamed", "combine_stacked", "factor", "apply_qt", "apply_q", "form_q", "pack_r", "cross_factor", "cross_apply_qt", "cross_apply_q", "plan_info",
           "plan_export", "slab", "cross_partner", "tsqr"]
