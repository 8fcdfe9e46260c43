"""Stall samples along the program: buckets of consecutive SASS instructions of an
`ncu --page source --csv --print-source sass` export (first kernel), with each bucket's executed
instruction count, sample share, top stall reasons and opcode mix.
  python tools/ncu_sass_regions.py report.csv [bucket]"""
import csv, sys
from collections import Counter
rows = list(csv.reader(open(sys.argv[1])))
B = int(sys.argv[2]) if len(sys.argv) > 2 else 200
hdr = rows[1]
data = []
for r in rows[2:]:  # first kernel only: a report with several launches repeats the two header rows
    if r and r[0] == "Kernel Name":
        break
    if len(r) == len(hdr):
        data.append(r)
c = {h: i for i, h in enumerate(hdr)}
iE, iS = c["Instructions Executed"], c["Warp Stall Sampling (All Samples)"]
reasons = [h for h in hdr if h.startswith("stall_") and "Not" not in h]
ts = sum(int(r[iS]) for r in data)
print("instructions", len(data), "samples", ts)
for b0 in range(0, len(data), B):
    blk = data[b0:b0 + B]
    s = sum(int(r[iS]) for r in blk); e = sum(int(r[iE]) for r in blk)
    if s < ts * 0.002: continue
    ops = Counter(); st = Counter()
    for r in blk:
        o = [x for x in r[1].split() if not x.startswith("@")][0]
        ops[o.split(".")[0]] += int(r[iE])
        for h in reasons: st[h[6:]] += int(r[c[h]])
    top = ", ".join(f"{k} {100*v/max(s,1):.0f}" for k, v in st.most_common(4))
    mix = ", ".join(f"{k} {100*v/max(e,1):.0f}" for k, v in ops.most_common(4))
    print(f"[{b0:5d}] samples {100*s/ts:5.1f}%  exec/instr {e/len(blk):9.0f}  samples/exec {1e3*s/max(e,1):7.2f}e-3 | {top} | {mix}")
