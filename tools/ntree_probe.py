"""Per-panel phases of the first leaf-level node and of the root in k_tree_pipe
(variant build with -DTSQR_NTREE_PROBE).  usage: TSQR_LIBRARY=... python tools/ntree_probe.py m n b s"""
import ctypes
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_0808_2664_b200 as T  # noqa: E402
from paper_0808_2664_b200 import _lib  # noqa: E402

m, n, b, s = (int(x) for x in sys.argv[1:5])
A = torch.randn((n, m), dtype=torch.float64, device="cuda")
R = torch.empty((n, n), dtype=torch.float64, device="cuda")
for _ in range(2):
    T.factor(A.clone(), b, s, R=R)
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * 128)()
_lib.lib().tsqr_ntree_probe_dump(buf)
npan = (n + 7) // 8
for name, base in (("leaf-level node", 0), ("root", 64)):
    t00 = buf[base]
    print(name)
    for P in range(npan):
        t = [buf[base + P * 8 + i] for i in range(5)]
        print(f"  P={P} start {(t[0] - t00) / 1e3:7.2f}us  wait {(t[1] - t[0]) / 1e3:6.2f}  load+steps {(t[2] - t[1]) / 1e3:6.2f}"
              f"  T+trail {(t[3] - t[2]) / 1e3:6.2f}  publish {(t[4] - t[3]) / 1e3:6.2f}")
