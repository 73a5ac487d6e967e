"""Staging vs compute time of node 0 in each k_node_apply launch (variant build with -DTSQR_NA_PROBE).
usage: TSQR_LIBRARY=.../naprobe.so python tools/na_probe.py m n b s k"""
import ctypes
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_0808_2664_b200 as T  # noqa: E402
from paper_0808_2664_b200 import _lib  # noqa: E402

m, n, b, s, k = (int(x) for x in sys.argv[1:6])
A = torch.randn((n, m), dtype=torch.float64, device="cuda")
C = torch.randn((k, m), dtype=torch.float64, device="cuda")
_, tree = T.factor(A, b, s)
T.apply_qt(tree, C)
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * 256)()
cnt = ctypes.c_int()
_lib.lib().tsqr_na_probe_dump(buf, ctypes.byref(cnt))
for i in range(min(cnt.value, 64)):
    t = [buf[i * 4 + j] for j in range(4)]
    print(f"launch {i}: staging {(t[1] - t[0]) / 1e3:7.2f} us  compute {(t[3] - t[1]) / 1e3:7.2f} us")
