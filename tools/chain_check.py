"""Quick check of the factor path: R vs torch.linalg.qr's R (sign-normalised,
normwise) and device timing.  usage: python tools/chain_check.py m n b s [reps]"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_0808_2664_b200 as T  # noqa: E402

m, n, b, s = (int(x) for x in sys.argv[1:5])
reps = int(sys.argv[5]) if len(sys.argv) > 5 else 5
g = torch.Generator(device="cuda").manual_seed(0)
A0 = torch.randn((n, m), dtype=torch.float64, device="cuda", generator=g)
A = A0.clone()
R = torch.empty((n, n), dtype=torch.float64, device="cuda")
tree = None
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
ts = []
for it in range(reps):
    A.copy_(A0)
    ev[0].record()
    _, tree = T.factor(A, b, s, R=R, tree=tree)
    ev[1].record()
    torch.cuda.synchronize()
    ts.append(ev[0].elapsed_time(ev[1]))
Rr = torch.linalg.qr(A0.T, mode="r")[1]
R = R.T                                     # column-major (n, n) tensor -> the matrix
sg = lambda X: X * torch.sign(torch.diagonal(X)).unsqueeze(1)
err = (sg(R) - sg(Rr)).norm() / Rr.norm()
low = torch.tril(R, -1).abs().max().item()
tmin = min(ts[1:]) if reps > 1 else ts[0]
print(f"m={m} n={n} b={b} s={s}: R err {err:.2e} lower {low:.1e}  factor {tmin:.3f} ms "
      f"({2*m*n*n/tmin/1e6:.0f} GF/s, {2*m*n*n/tmin/1e6/37220*100:.1f}% of FP64 peak)  all {['%.3f'%t for t in ts]}")
