"""Repeat the factor (+ form Q / apply) of one configuration and compare every result bitwise
with the first run: a race in a hand-off would show up as run-to-run differences (tools only).
usage: python tools/determinism.py m n b s [reps]"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_0808_2664_b200 as T  # noqa: E402

m, n, b, s = (int(x) for x in sys.argv[1:5])
reps = int(sys.argv[5]) if len(sys.argv) > 5 else 10
g = torch.Generator(device="cuda").manual_seed(7)
A0 = torch.randn((n, m), dtype=torch.float64, device="cuda", generator=g)
C0 = torch.randn((min(n, 64), m), dtype=torch.float64, device="cuda", generator=g)
ref = None
tree = None
bad = 0
for it in range(reps):
    A = A0.clone()
    R, tree = T.factor(A, b, s, tree=tree)
    Q = T.form_q(tree)
    C = C0.clone()
    T.apply_qt(tree, C)
    torch.cuda.synchronize()
    out = (A, R, Q, C)
    if ref is None:
        ref = tuple(x.clone() for x in out)
    else:
        same = all(torch.equal(x, y) for x, y in zip(out, ref))
        bad += not same
print(f"m={m} n={n} b={b} s={s}: {reps} runs, {bad} differing from the first")
