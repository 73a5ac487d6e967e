"""Per-kernel device times (CUPTI via torch.profiler) of factor / apply_qt /
form_q at one configuration.  usage: python tools/kprof.py m n b s [k] [reps]"""
import collections
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from torch.profiler import profile, ProfilerActivity  # noqa: E402
import paper_0808_2664_b200 as T  # noqa: E402

m, n, b, s = (int(x) for x in sys.argv[1:5])
k = int(sys.argv[5]) if len(sys.argv) > 5 else n
reps = int(sys.argv[6]) if len(sys.argv) > 6 else 5
g = torch.Generator(device="cuda").manual_seed(0)
A0 = torch.randn((n, m), dtype=torch.float64, device="cuda", generator=g)
C0 = torch.randn((k, m), dtype=torch.float64, device="cuda", generator=g)
A, C = A0.clone(), C0.clone()
Q = torch.empty((n, m), dtype=torch.float64, device="cuda")
R = torch.empty((n, n), dtype=torch.float64, device="cuda")
_, tree = T.factor(A, b, s, R=R)


def step():
    T.factor(A, b, s, R=R, tree=tree)
    T.apply_qt(tree, C)
    T.form_q(tree, Q)


for _ in range(2):
    A.copy_(A0)
    C.copy_(C0)
    step()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(reps):
        step()
    torch.cuda.synchronize()
tot = collections.defaultdict(float)
cnt = collections.Counter()
for ev in prof.events():
    if ev.device_type == torch.autograd.DeviceType.CUDA:
        tot[ev.name] += ev.device_time_total if hasattr(ev, "device_time_total") else ev.cuda_time_total
        cnt[ev.name] += 1
print(f"m={m} n={n} b={b} s={s} k={k}: per-step kernel times (us)")
for name, t in sorted(tot.items(), key=lambda x: -x[1]):
    print(f"  {t / reps:9.1f}  x{cnt[name] / reps:4.1f}  {name[:110]}")
print(f"  total {sum(tot.values()) / reps:.1f} us")
