"""Warp-stall samples of an ncu report grouped by source-line ranges (tools only).
usage: python tools/ncu_groups.py report.ncu-rep"""
import collections
import csv
import io
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "sass,cuda"],
                     capture_output=True, text=True).stdout
GROUPS = [("chunk.cuh", 100, 145, "hand-off waits/publish"), ("chunk.cuh", 146, 188, "house_bf"),
          ("chunk.cuh", 218, 245, "build_t"), ("chunk.cuh", 246, 260, "quad_sums"),
          ("chunk.cuh", 300, 415, "structured steps"), ("chunk.cuh", 416, 490, "dense steps"),
          ("chunk.cuh", 491, 580, "trailing update"), ("chunk.cuh", 581, 700, "factor_panel glue"),
          ("tsqr_chain.cu", 0, 100000, "chunk prologue/epilogue + walk"), ("wy.cuh", 30, 45, "DMMA (all callers)")]
fname, hdr = None, None
agg = collections.Counter()
tot = 0.0
for r in csv.reader(io.StringIO(out)):
    if len(r) >= 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        iS = hdr.index("Warp Stall Sampling (All Samples)")
        continue
    if hdr is None or len(r) < len(hdr) or not r[0].isdigit():
        continue
    r = r[:2] + r[len(r) - (len(hdr) - 2):]
    v = float(r[iS]) if r[iS] not in ("-", "") else 0.0
    tot += v
    line = int(r[0])
    for f, lo, hi, name in GROUPS:
        if fname == f and lo <= line <= hi:
            agg[name] += v
            break
    else:
        agg[f"other ({fname})"] += v
for k, v in agg.most_common():
    print(f"{100 * v / tot:5.1f}%  {k}")
