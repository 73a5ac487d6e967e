"""Per-CUDA-source-line warp-stall samples from an ncu report (tools only).
usage: python tools/ncu_lines.py report.ncu-rep [top]"""
import collections
import csv
import io
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "sass,cuda"],
                     capture_output=True, text=True).stdout
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
fname, hdr = None, None
agg, ins, src = collections.Counter(), collections.Counter(), {}
for r in csv.reader(io.StringIO(out)):
    if len(r) >= 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        iS, iE = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
        continue
    if hdr is None or len(r) < len(hdr) or not r[0].isdigit():
        continue
    r = r[:2] + r[len(r) - (len(hdr) - 2):]          # source text with stray quotes: align from the end
    key = (fname, int(r[0]))
    src[key] = r[1][:70]
    agg[key] += float(r[iS]) if r[iS] not in ("-", "") else 0
    ins[key] += float(r[iE] or 0) if r[iE] not in ("-", "") else 0
tot = sum(agg.values())
print(f"total samples {tot:.0f}")
for k, v in agg.most_common(top):
    print(f"{100 * v / tot:5.1f}%  {k[0]}:{k[1]:<5d} inst {ins[k]:12.0f}  {src[k]}")
