"""Summarise an ncu source page (SASS) CSV: stall reasons overall and per region
between barriers, top instructions.  usage: ncu_sass_summary.py file.csv"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, data = rows[1], rows[2:]
ix = {h: i for i, h in enumerate(hdr)}
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]


def val(r, h):
    v = r[ix[h]]
    try:
        return float(v)
    except ValueError:
        return 0.0


tot = collections.Counter()
for r in data:
    for h in stalls:
        tot[h] += val(r, h)
S = sum(tot.values())
print("total stall samples", S)
for h, v in tot.most_common(10):
    print(f"  {h:28s} {100 * v / S:5.1f}%")
# regions delimited by BAR.SYNC
reg, cur = [], {"start": 0, "samples": 0, "exec": 0, "first": "", "stalls": collections.Counter()}
for k, r in enumerate(data):
    src = r[ix["Source"]].strip()
    s = val(r, "Warp Stall Sampling (All Samples)")
    cur["samples"] += s
    cur["exec"] += val(r, "Instructions Executed")
    if not cur["first"]:
        cur["first"] = src[:50]
    for h in stalls:
        cur["stalls"][h] += val(r, h)
    if "BAR.SYNC" in src or k == len(data) - 1:
        cur["end"] = k
        reg.append(cur)
        cur = {"start": k + 1, "samples": 0, "exec": 0, "first": "", "stalls": collections.Counter()}
print("regions (between barriers) with >2% of samples:")
for g in reg:
    if g["samples"] > 0.02 * S:
        top = ", ".join(f"{h[6:]}={100 * v / g['samples']:.0f}%" for h, v in g["stalls"].most_common(3))
        print(f"  [{g['start']:5d}-{g['end']:5d}] {100 * g['samples'] / S:5.1f}%  exec={g['exec']:.0f}  {top}  | {g['first']}")
print("top instructions:")
for r in sorted(data, key=lambda r: -val(r, "Warp Stall Sampling (All Samples)"))[:int(sys.argv[2]) if len(sys.argv) > 2 else 15]:
    top = max(stalls, key=lambda h: val(r, h))
    print(f"  {val(r, 'Warp Stall Sampling (All Samples)'):6.0f} {top[6:]:14s} {r[ix['Source']].strip()[:70]}")
