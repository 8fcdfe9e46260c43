"""Summarise an ncu report: key throughput / occupancy / stall metrics per kernel."""
import csv
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(raw.splitlines()))
h, units = r[0], r[1]
keys = ["gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed.sum.per_cycle_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "smsp__thread_inst_executed_per_inst_executed.ratio",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
        "smsp__sass_thread_inst_executed_op_ffma_pred_on.sum", "smsp__sass_thread_inst_executed_op_dfma_pred_on.sum"]
for row in r[2:]:
    print("=====", row[h.index("Kernel Name")][:80])
    for k in keys:
        if k in h:
            print(f"  {k:80s} {row[h.index(k)]} {units[h.index(k)]}")
    stalls = [(k, float(row[i])) for i, k in enumerate(h)
              if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")
              and row[i] not in ("", "n/a")]
    tot = sum(v for _, v in stalls) or 1
    print("  stalls:", ", ".join(f"{k.replace('smsp__pcsamp_warps_issue_stalled_', '')} {100 * v / tot:.0f}%"
                                 for k, v in sorted(stalls, key=lambda x: -x[1]) if v / tot > 0.02))

# optional: per-kernel DRAM traffic of this capture as JSON (read by bench.py's roofline.traffic)
if len(sys.argv) > 2:
    import json
    import re

    def num(row, k):
        v = row[h.index(k)].replace(",", "")
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ms": 1.0, "us": 1e-3, "ns": 1e-6,
                 "msecond": 1.0, "usecond": 1e-3, "nsecond": 1e-6}.get(units[h.index(k)], 1)
        return float(v) * scale

    out = {}
    for row in r[2:]:
        name = row[h.index("Kernel Name")]
        m = re.search(r"(k_[a-z0-9_]+)", name)
        key = m.group(1) if m else name[:40]
        out[key] = {"dram_bytes_per_launch": num(row, "dram__bytes_read.sum") + num(row, "dram__bytes_write.sum"),
                    "gpu_time_ms": num(row, "gpu__time_duration.sum"), "report": rep}
    with open(sys.argv[2], "w") as f:
        json.dump(out, f, indent=1)
