"""Small shapes of every engine for compute-sanitizer (memcheck / racecheck / synccheck runs; tools
only).  Each shape: factor, form Q, Q^T C, Q C; checks A = QR and Q^T Q = I on the host.
usage: compute-sanitizer --tool racecheck python tools/sanitize_small.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_0808_2664_b200 as T  # noqa: E402
from paper_0808_2664_b200 import inputs  # noqa: E402

SHAPES = [(2048, 16, 512, 256), (4096, 32, 1024, 1024), (4096, 50, 2048, 1366), (4096, 64, 2048, 2048),
          (1200, 200, 600, 300)]
for m, n, b, s in SHAPES:
    A0 = inputs.gaussian(m, n, 0).cuda()
    A = A0.clone()
    R, tree = T.factor(A, block_rows=b, tile_rows=s)
    Q = T.form_q(tree)
    C = inputs.gaussian(m, 8, 1).cuda()
    C1 = C.clone()
    T.apply_qt(tree, C)
    T.apply_q(tree, C)
    torch.cuda.synchronize()
    res = (torch.linalg.norm(A0 - Q @ R) / torch.linalg.norm(A0)).item()
    orth = torch.linalg.norm(Q.T @ Q - torch.eye(n, dtype=Q.dtype, device=Q.device)).item()
    rt = (torch.linalg.norm(C - C1) / torch.linalg.norm(C1)).item()
    tree.free()
    print(f"{m}x{n} b={b} s={s}: ||A-QR||/||A|| {res:.1e}  ||Q^TQ-I|| {orth:.1e}  Q(Q^T C) {rt:.1e}", flush=True)
    assert res < 1e-13 and orth < 1e-13 and rt < 1e-13
