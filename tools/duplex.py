"""Host<->device copy bandwidth alone and concurrently (full duplex check; tools only)."""
import time
import torch

n = int(2 ** 30 * 2)  # 16 GiB total? no: elements of fp64 -> 8 * n bytes
n = 1 << 30           # 8 GiB of fp64
a = torch.empty(n, dtype=torch.float64).pin_memory()
b = torch.empty(n, dtype=torch.float64).pin_memory()
da = torch.empty(n, dtype=torch.float64, device="cuda")
db = torch.empty(n, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def run(h2d, d2h):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    if h2d:
        with torch.cuda.stream(s1):
            da.copy_(a, non_blocking=True)
    if d2h:
        with torch.cuda.stream(s2):
            b.copy_(db, non_blocking=True)
    torch.cuda.synchronize()
    return time.perf_counter() - t0


for _ in range(2):
    t1, t2, t3 = run(1, 0), run(0, 1), run(1, 1)
    gb = 8 * n / 1e9
    print(f"{gb:.1f} GB: H2D {t1*1e3:.0f} ms ({gb/t1:.1f} GB/s)  D2H {t2*1e3:.0f} ms ({gb/t2:.1f} GB/s)  both {t3*1e3:.0f} ms ({2*gb/t3:.1f} GB/s total)")
