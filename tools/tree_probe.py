"""Per-phase time of node 0's panels in k_wide_tree_pipe (variant build with -DTSQR_TREE_PROBE).
usage: TSQR_LIBRARY=.../tprobe.so python tools/tree_probe.py m n b s"""
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
buf = (ctypes.c_ulonglong * 256)()
_lib.lib().tsqr_tree_probe_dump(buf)
npan = (n + 7) // 8
names = ["wait+load", "steps+T", "trailing", "publish+fence"]
tot = [0.0] * 4
for P in range(npan):
    t = [buf[P * 8 + i] for i in range(5)]
    d = [(t[i + 1] - t[i]) / 1e3 for i in range(4)]
    for i in range(4):
        tot[i] += d[i]
    print(f"P={P:2d} " + "  ".join(f"{names[i]} {d[i]:6.2f}us" for i in range(4)))
print("total " + "  ".join(f"{names[i]} {tot[i]:7.1f}us" for i in range(4)))

print("P=20 steps 0..3 (us): dots, quad, house, update")
for jj in range(4):
    t = [buf[208 + jj * 8 + i] for i in range(5)]
    print(jj, " ".join(f"{(t[i + 1] - t[i]) / 1e3:6.3f}" for i in range(4)))
