# per-level k_step durations of one step (after one warm-up step) and --set full of the heaviest levels
cfg=${1:-C3}; nlev=${2:-26}; heavy=${3:-7}
ncu --metrics gpu__time_duration.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,dram__throughput.avg.pct_of_peak_sustained_elapsed,lts__t_bytes.sum --clock-control none -k regex:k_step --launch-skip $nlev -c $nlev --csv --log-file gpurun_out/kstep_levels_$cfg.csv \
  python tools/profile_step.py --config $cfg --warmup 1 --steps 1 > gpurun_out/ncu_kstep_levels.log 2>&1
python - <<PY
import csv
rows=[r for r in csv.reader(l for l in open("gpurun_out/kstep_levels_$cfg.csv") if l.startswith('"'))]
h=rows[0]; c={k:i for i,k in enumerate(h)}
lev={}
for r in rows[1:]:
    lev.setdefault(int(r[c["ID"]]),{})[r[c["Metric Name"]]]=(r[c["Metric Value"]],r[c["Metric Unit"]])
tot=0
for i,(k,m) in enumerate(sorted(lev.items())):
    d=float(m["gpu__time_duration.sum"][0].replace(",","")); u=m["gpu__time_duration.sum"][1]
    us=d/1000 if u.startswith("n") else d
    tot+=us
    print(i, round(us,1),"us issue",m["smsp__issue_active.avg.pct_of_peak_sustained_active"][0],"% dram",m["dram__throughput.avg.pct_of_peak_sustained_elapsed"][0],"% l2 bytes",m["lts__t_bytes.sum"][0],m["lts__t_bytes.sum"][1])
print("total",round(tot,1),"us")
PY
ncu --set full --clock-control none --import-source on -k regex:k_step --launch-skip $((nlev + heavy)) -c 2 -o gpurun_out/kstep_heavy_$cfg -f \
  python tools/profile_step.py --config $cfg --warmup 1 --steps 1 > gpurun_out/ncu_kstep_heavy.log 2>&1
python tools/ncu_summary.py gpurun_out/kstep_heavy_$cfg.ncu-rep
