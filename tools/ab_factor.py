"""A/B timing of tsqr_factor (+ second op) for variant builds of libtsqr.so (not product code).
usage: TSQR_LIBRARY=build_ab/x.so python tools/ab_factor.py c4 c2 ..."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_0808_2664_b200 as T  # noqa: E402

lib = os.environ.get("TSQR_LIBRARY", "default")
for name in sys.argv[1:]:
    cfg = bench.CONFIGS[name]
    m, n, b, s, k = cfg["m"], cfg["n"], cfg["b"], int(os.environ.get("AB_S", cfg["s"])), cfg["k"]
    A0 = bench.make_slab(cfg, 0, m, "cuda")
    A = torch.empty_like(A0)
    Q = torch.empty_like(A0) if cfg["op"] == "form_q" else None
    C0 = bench.make_c_slab(cfg, 0, m, "cuda") if k else None
    C = torch.empty_like(C0) if k else None
    tree = None
    e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
    tf, ts, tl = [], [], []
    for it in range(13):
        A.copy_(A0)
        if C is not None:
            C.copy_(C0)
        e0.record()
        _, tree = T.factor(A, b, s, tree=tree, stage_timing=True)
        e1.record()
        if Q is not None:
            T.form_q(tree, Q)
        else:
            T.apply_qt(tree, C)
        e2.record()
        e2.synchronize()
        if it >= 3:
            tf.append(e0.elapsed_time(e1))
            ts.append(e1.elapsed_time(e2))
            tl.append(tree.stage_ms()[0])
    med = statistics.median
    print(f"{os.path.basename(lib):28s} {name} s={s}: factor {med(tf):8.3f} ms (leaf {med(tl):8.3f})  second op {med(ts):8.3f} ms",
          flush=True)
    tree.free()
    del A0, A, Q, C0, C
    torch.cuda.empty_cache()
