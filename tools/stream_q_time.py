"""Streamed factor with Q kept (tsqr_factor_streamed_q) and the streamed Q / Q^T C (tools only):
wall times of the synchronous calls on pinned host matrices against the bare host<->device copies
of the bytes each must move.  usage: python tools/stream_q_time.py m n slab b s k"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_0808_2664_b200 as T  # noqa: E402
from paper_0808_2664_b200 import inputs  # noqa: E402

m, n, slab, b, s, k = (int(x) for x in sys.argv[1:7])
A = torch.cat([inputs.gaussian_rows(r, min(1 << 22, m - r), n, 0, "cuda").cpu() for r in range(0, m, 1 << 22)], 1).pin_memory()
Y = torch.empty_like(A).pin_memory()
Q = torch.empty_like(A).pin_memory()
C0 = torch.cat([inputs.gaussian_rows(r, min(1 << 22, m - r), k, 1, "cuda").cpu() for r in range(0, m, 1 << 22)], 1)
C = C0.clone().pin_memory()


def wall(fn, reps=3):
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    return sorted(ts)[len(ts) // 2]


st = None


def fac():
    global st
    if st is not None:
        st.free()
    st = T.factor_streamed_q(A, slab, Y, block_rows=b, tile_rows=s)[1]


tf = wall(fac)
tq = wall(lambda: T.streamed_form_q(st, Q))
ta = wall(lambda: (C.copy_(C0), T.streamed_apply_qt(st, C)))
tc = wall(lambda: C.copy_(C0), 3)
ta -= tc
D = torch.empty((n, m), dtype=torch.float64, device="cuda")
h2d = wall(lambda: D.copy_(A, non_blocking=True))
d2h = wall(lambda: Y.copy_(D, non_blocking=True))
gb = 8.0 * m * n / 1e9
print(f"m={m} n={n} slab={slab} b={b} s={s}: A = {gb:.2f} GB; bare copies H2D {h2d * 1e3:.1f} ms ({gb / h2d:.1f} GB/s), "
      f"D2H {d2h * 1e3:.1f} ms ({gb / d2h:.1f} GB/s)")
print(f"  factor_streamed_q (A in, Y out, state out) {tf * 1e3:.1f} ms = {tf / max(h2d, d2h):.2f} x max(H2D, D2H)")
print(f"  streamed_form_q   (Y in, Q out)            {tq * 1e3:.1f} ms = {tq / max(h2d, d2h):.2f} x max(H2D, D2H)")
print(f"  streamed_apply_qt (Y, C in, C out), k={k}    {ta * 1e3:.1f} ms")
