"""Run one workload op a few times (for ncu / quick timing).  Not a bench number.
usage: python tools/prof_one.py CONFIG OP [reps] [m_override]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_0808_2664_b200 as T  # noqa: E402

cfg = dict(bench.CONFIGS[sys.argv[1]])
op = sys.argv[2]
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
if len(sys.argv) > 4:
    cfg["m"] = int(sys.argv[4])
if len(sys.argv) > 5:
    cfg["s"] = int(sys.argv[5])
m, n, b, s = cfg["m"], cfg["n"], cfg["b"], cfg["s"]
A0 = bench.make_slab(cfg, 0, m, "cuda")
A = A0.clone()
tree = None
R = torch.empty((n, n), dtype=torch.float64, device="cuda")
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
for it in range(reps):
    A.copy_(A0)
    ev[0].record()
    _, tree = T.factor(A, b, s, R=R, tree=tree)
    ev[1].record()
    torch.cuda.synchronize()
    tf = ev[0].elapsed_time(ev[1])
    t2 = None
    if op == "form_q":
        ev[0].record()
        Q = T.form_q(tree)
        ev[1].record()
        torch.cuda.synchronize()
        t2 = ev[0].elapsed_time(ev[1])
    elif op == "apply_qt":
        C = bench.make_c_slab(cfg, 0, m, "cuda") if cfg["k"] else torch.randn((64, m), dtype=torch.float64, device="cuda")
        ev[0].record()
        T.apply_qt(tree, C)
        ev[1].record()
        torch.cuda.synchronize()
        t2 = ev[0].elapsed_time(ev[1])
    print(f"rep {it}: factor {tf:.3f} ms ({2*m*n*n/tf/1e6:.1f} GF/s)  second {t2}", flush=True)
