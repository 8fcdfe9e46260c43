import csv, sys, subprocess
from collections import Counter
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
# may contain several kernels: split on "Kernel Name" rows
blocks=[]; cur=None
for r in rows:
    if r and r[0]=="Kernel Name":
        cur={"name":r[1],"rows":[]}; blocks.append(cur); continue
    if cur is not None: cur["rows"].append(r)
for b in blocks[:1]:
    hdr=b["rows"][0]; data=b["rows"][1:]
    cols={h:i for i,h in enumerate(hdr)}
    iE=cols["Instructions Executed"]; iS=cols["Warp Stall Sampling (All Samples)"]
    tot=sum(int(r[iE]) for r in data if len(r)>iE and r[iE].isdigit()); ts=sum(int(r[iS]) for r in data if len(r)>iS and r[iS].isdigit())
    op=Counter(); st=Counter()
    for r in data:
        if len(r)<=iE or not r[iE].isdigit(): continue
        o=[x for x in r[1].strip().split() if not x.startswith('@')]
        op[o[0]]+=int(r[iE]); st[o[0]]+=int(r[iS])
    print(b["name"][:80], "instrs", tot, "samples", ts)
    for k,v in op.most_common(16): print(f"  {k:30s} {100*v/tot:5.1f}%  stall {100*st[k]/ts:.1f}%")
    reasons=[h for h in hdr if h.startswith('stall_') and 'Not' not in h]
    agg={h:sum(int(r[cols[h]]) for r in data if len(r)>cols[h] and r[cols[h]].isdigit()) for h in reasons}
    print("  ", [(k[6:], round(100*v/ts,1)) for k,v in sorted(agg.items(), key=lambda kv:-kv[1])[:8]])
