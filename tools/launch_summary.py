"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list per kernel (tools only).
usage: python tools/launch_summary.py launches.csv [title]"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h, agg = None, collections.defaultdict(list)
scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "second": 1e6, "s": 1e6}
for r in rows:
    if "Kernel Name" in r:
        h = r
        continue
    if h and len(r) == len(h) and r[h.index("Metric Name")] == "gpu__time_duration.sum":
        name = r[h.index("Kernel Name")].replace("(anonymous namespace)::", "").replace("<unnamed>::", "").replace("void ", "")
        name = name.split("(")[0].split("<")[0].replace("tsqr::", "")
        agg[name].append(float(r[h.index("Metric Value")].replace(",", "")) * scale[r[h.index("Metric Unit")]])
tot = sum(sum(v) for v in agg.values())
if len(sys.argv) > 2:
    print(sys.argv[2])
print("per-launch times are cold-cache and serialised (ncu); compare the shares, not the absolutes")
for k, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
    print(f"{k:30s} launches {len(v):4d}  total {sum(v) / 1e3:9.3f} ms  mean {sum(v) / len(v):10.1f} us  share {100 * sum(v) / tot:5.1f}%")
