"""Per-panel phases of tile 0 in k_wide_leaves (variant build with -DTSQR_LEAF_PROBE).
usage: TSQR_LIBRARY=.../lprobe.so python tools/leaf_probe.py m n b s"""
import ctypes
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_0808_2664_b200 as T  # noqa: E402
from paper_0808_2664_b200 import _lib  # noqa: E402

m, n, b, s = (int(x) for x in sys.argv[1:5])
A = torch.randn((n, m), dtype=torch.float64, device="cuda")
for _ in range(2):
    T.factor(A.clone(), b, s)
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * 128)()
_lib.lib().tsqr_leaf_probe_dump(buf)
tot = [0.0] * 3
for p in range((n + 7) // 8):
    t = [buf[p * 4 + i] for i in range(4)]
    d = [(t[i + 1] - t[i]) / 1e3 for i in range(3)]
    tot = [a + x for a, x in zip(tot, d)]
    print(f"p={p:2d} steps {d[0]:6.2f}  writeback+T {d[1]:6.2f}  trailing {d[2]:6.2f} us")
print(f"total steps {tot[0]:.1f}  writeback+T {tot[1]:.1f}  trailing {tot[2]:.1f} us")
