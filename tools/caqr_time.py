"""CAQR timing (tools only): factor of an m x N matrix with TSQR panels vs cuSOLVER's
geqrf (torch.geqrf) on the same matrix, CUDA events, inputs larger than L2."""
import sys
import torch
import paper_0808_2664_b200 as T
from paper_0808_2664_b200 import inputs

m, N, panel, b, s = (int(x) for x in sys.argv[1:6])
reps = 5
A0 = inputs.gaussian_rows(0, m, N, 0, "cuda")
flops = 2 * m * N * N - 2 * N ** 3 / 3
A = A0.clone()
R, h = T.caqr(A, panel, block_rows=b, tile_rows=s)
ts = []
for _ in range(reps):
    A.copy_(A0)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    T.caqr(A, panel, block_rows=b, tile_rows=s, R=R, handle=h)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
t = sorted(ts)[len(ts) // 2]
print(f"caqr m={m} N={N} panel={panel} b={b} s={s}: {t:.3f} ms  {flops / t / 1e9:.2f} TF/s")
Q = T.caqr_form_q(h)
torch.cuda.synchronize()
Am = A0.T
err = (torch.linalg.norm(Am - Q.T @ R.T) / torch.linalg.norm(Am)).item()
print(f"  ||A - QR||/||A|| = {err:.2e}")
At = A0.T.contiguous().T          # (m, N) column-major for cuSOLVER
ts = []
for _ in range(reps):
    X = At.clone()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    torch.geqrf(X)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
t2 = sorted(ts)[len(ts) // 2]
print(f"cusolver geqrf: {t2:.3f} ms  {flops / t2 / 1e9:.2f} TF/s")
