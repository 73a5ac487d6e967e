"""Streamed (out-of-HBM) TSQR timing (tools only): R of a pinned host matrix through
tsqr_factor_streamed, against the host->device copy of the same bytes alone (the bound of a
streamed factorization) and the in-HBM factor.  usage: python tools/stream_time.py m n slab b s"""
import sys
import time

import torch

import paper_0808_2664_b200 as T
from paper_0808_2664_b200 import inputs

m, n, slab, b, s = (int(x) for x in sys.argv[1:6])
A = inputs.gaussian_rows(0, m, n, 0, "cuda").cpu().pin_memory()
R = torch.empty((n, n), dtype=torch.float64, device="cuda")
T.factor_streamed(A, slab, b, s, R=R)                 # warm-up (allocations, module load)
ts = []
for _ in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    T.factor_streamed(A, slab, b, s, R=R)             # synchronous
    ts.append(time.perf_counter() - t0)
t = sorted(ts)[1]
D = torch.empty((n, m), dtype=torch.float64, device="cuda")
cs = []
for _ in range(3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    D.copy_(A, non_blocking=True)
    e1.record()
    torch.cuda.synchronize()
    cs.append(e0.elapsed_time(e1) / 1e3)
c = sorted(cs)[1]
fs = []
for _ in range(3):
    W = D.clone()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    T.factor(W, b, s)[1].free()
    e1.record()
    torch.cuda.synchronize()
    fs.append(e0.elapsed_time(e1) / 1e3)
f = sorted(fs)[1]
gb = 8.0 * m * n / 1e9
print(f"streamed m={m} n={n} slab={slab}: {t * 1e3:.2f} ms wall ({gb / t:.1f} GB/s of A, "
      f"{2 * m * n * n / t / 1e12:.2f} TF/s); H2D copy alone {c * 1e3:.2f} ms ({gb / c:.1f} GB/s); "
      f"in-HBM factor {f * 1e3:.2f} ms; streamed / copy = {t / c:.2f}")
