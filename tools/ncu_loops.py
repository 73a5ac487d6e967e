"""Summarise an ncu SASS source-page CSV by loop (backward-branch ranges) and by
opcode class: stall samples and executed warp-instructions.  Tools only.
usage: ncu_loops.py file.csv"""
import collections
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, data = rows[1], rows[2:]
ix = {h: i for i, h in enumerate(hdr)}


def f(r, h):
    try:
        return float(r[ix[h]])
    except (ValueError, KeyError):
        return 0.0


ins = []
for r in data:
    addr = int(r[ix["Address"]], 16) if r[ix["Address"]].startswith("0x") else int(r[ix["Address"]])
    ins.append((addr, r[ix["Source"]], f(r, "Warp Stall Sampling (All Samples)"), f(r, "Instructions Executed"), r))
tot_s = sum(i[2] for i in ins) or 1
tot_e = sum(i[3] for i in ins) or 1
print(f"total samples {tot_s:.0f}  executed warp-instr {tot_e:.3e}")
cls = collections.Counter()
cle = collections.Counter()
for a, src, s, e, _ in ins:
    op = re.sub(r"^@!?U?P\w+\s+", "", src.strip()).split(" ")[0].split(".")[0]
    cls[op] += s
    cle[op] += e
print("by opcode (samples%, exec%):")
for op, s in cls.most_common(16):
    print(f"  {op:10s} {100*s/tot_s:5.1f}%  {100*cle[op]/tot_e:5.1f}%")
# loops: backward branches
loops = []
for a, src, s, e, _ in ins:
    m = re.search(r"BRA[^ ]* +(?:\w+, *)?(0x[0-9a-f]+)", src)
    if m:
        t = int(m.group(1), 16)
        if t <= a:
            loops.append((t, a))
print("loops (start-end: samples%, exec%, top stalls):")
stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
for t, a in sorted(set(loops)):
    sel = [i for i in ins if t <= i[0] <= a]
    s = sum(i[2] for i in sel)
    e = sum(i[3] for i in sel)
    if s / tot_s < 0.02:
        continue
    st = collections.Counter()
    for i in sel:
        for h in stall_cols:
            st[h] += f(i[4], h)
    tops = ", ".join(f"{h[6:]} {100*v/max(s,1):.0f}%" for h, v in st.most_common(4))
    nshfl = sum(1 for i in sel if "SHFL" in i[1])
    ndmma = sum(1 for i in sel if "DMMA" in i[1])
    print(f"  {t:#06x}-{a:#06x} ({len(sel)} instr, {nshfl} SHFL, {ndmma} DMMA): {100*s/tot_s:5.1f}% samples, {100*e/tot_e:5.1f}% exec; {tops}")
