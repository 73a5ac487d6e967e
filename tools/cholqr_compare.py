"""CholeskyQR (the comparison method, tsqr_cholqr) vs TSQR (factor + form Q) on the C4 recipe:
orthogonality ||Q^T Q - I||_F, backward error ||A - QR|| / ||A|| and device time (CUDA events,
median of 5) over a kappa grid.  Tools only, not a bench line.
usage: python tools/cholqr_compare.py [m] [n]"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_0808_2664_b200 as T  # noqa: E402
from paper_0808_2664_b200 import inputs  # noqa: E402

m = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 20
n = int(sys.argv[2]) if len(sys.argv) > 2 else 64
print(f"m = {m}, n = {n}, C4 recipe A = G diag(sigma) V^T, sigma log-spaced 1 .. 1/kappa; times: median of 5 (ms)")
print(f"{'kappa':>8s} | {'CholQR orth':>12s} {'CholQR bwd':>11s} {'info':>5s} {'ms':>8s} | {'TSQR orth':>10s} {'TSQR bwd':>10s} {'ms':>8s}")
I = torch.eye(n, dtype=torch.float64, device="cuda")
ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
for kappa in (1e0, 1e2, 1e4, 1e6, 1e7, 1e8, 1e10, 1e12):
    A0 = torch.cat([inputs.conditioned_rows(r, min(1 << 20, m - r), n, 0, kappa).cuda() for r in range(0, m, 1 << 20)], 1)
    A = A0.clone()
    Qc = torch.empty_like(A0)
    Qt = torch.empty_like(A0)
    Rc = torch.empty((n, n), dtype=torch.float64, device="cuda")
    tree = None
    tc, tt = [], []
    for it in range(6):
        A.copy_(A0)
        ev[0].record()
        _, _, info = T.cholqr(A0, R=Rc, Q=Qc)
        ev[1].record()
        Rt, tree = T.factor(A, 4096, 4096, tree=tree)
        T.form_q(tree, Qt)
        ev[2].record()
        ev[2].synchronize()
        if it:
            tc.append(ev[0].elapsed_time(ev[1]))
            tt.append(ev[1].elapsed_time(ev[2]))
    nA = torch.linalg.norm(A0).item()
    ok = int(info.item()) == 0
    oc = torch.linalg.norm(Qc @ Qc.T - I).item() if ok else float("nan")
    bc = (torch.linalg.norm(A0 - Rc @ Qc) / nA).item() if ok else float("nan")
    ot = torch.linalg.norm(Qt @ Qt.T - I).item()
    bt = (torch.linalg.norm(A0 - Rt @ Qt) / nA).item()
    print(f"{kappa:8.0e} | {oc:12.2e} {bc:11.2e} {int(info.item()):5d} {statistics.median(tc):8.3f} | "
          f"{ot:10.2e} {bt:10.2e} {statistics.median(tt):8.3f}", flush=True)
    tree.free()
    del A0, A, Qc, Qt
    torch.cuda.empty_cache()
