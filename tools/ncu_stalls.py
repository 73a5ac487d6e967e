"""Summarise an ncu SASS source-page CSV: per-opcode and top instructions with
stall reasons (tools only).  usage: python tools/ncu_stalls.py file.csv [lo hi]"""
import csv
import collections
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
data = rows[2:]
ia, isrc = h.index("Address"), h.index("Source")
iss, iex = h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
reasons = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
ri = [h.index(c) for c in reasons]
f = lambda x: float(x or 0)  # noqa: E731
tot = sum(f(r[iss]) for r in data)
agg = collections.Counter()
for r in data:
    for c, i in zip(reasons, ri):
        agg[c] += f(r[i])
print("total samples", tot)
print("by reason:", ", ".join(f"{k[6:]} {100*v/tot:.1f}%" for k, v in agg.most_common(10)))
if len(sys.argv) > 3:
    lo, hi = int(sys.argv[2], 16), int(sys.argv[3], 16)
    for r in data:
        a = int(r[ia], 16) & 0xfffff
        if lo <= a <= hi:
            top = sorted(((f(r[i]), c[6:]) for c, i in zip(reasons, ri)), reverse=True)[:2]
            print(f"{a:05x} {f(r[iss]):6.0f} {f(r[iex]):9.0f} {r[isrc][:60]:60s} " +
                  " ".join(f"{c}:{v:.0f}" for v, c in top if v > 0))
else:
    top = sorted(data, key=lambda r: -f(r[iss]))[:30]
    for r in top:
        a = int(r[ia], 16) & 0xfffff
        t2 = sorted(((f(r[i]), c[6:]) for c, i in zip(reasons, ri)), reverse=True)[:2]
        print(f"{a:05x} {f(r[iss]):6.0f} {f(r[iex]):9.0f} {r[isrc][:60]:60s} " +
              " ".join(f"{c}:{v:.0f}" for v, c in t2 if v > 0))
