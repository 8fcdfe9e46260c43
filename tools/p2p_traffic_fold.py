"""Fold the ncu CSVs of tools/p2p_traffic.sh into profiles/ncu_traffic.json ("by_config").

bench.py reads by_config["<config>/<precision>"] for its roofline.traffic field.
"""
import csv
import glob
import json
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
data = json.load(open(path))
by = data.setdefault("by_config", {})
for f in sorted(glob.glob(os.path.join(ROOT, "gpurun_out", "traffic_*_*.csv"))):
    cfg, prec = re.match(r".*traffic_(C\d)_(fp\d\d)\.csv", f).groups()
    lines = open(f).read().splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
    vals, kernel = {}, None
    for row in csv.DictReader(lines[start:]):
        kernel = row["Kernel Name"].split("(")[0].split("<")[0].strip().split("::")[-1]
        v = float(row["Metric Value"].replace(",", ""))
        unit = row["Metric Unit"]
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-6, "us": 1e-3, "ms": 1, "msecond": 1,
                 "usecond": 1e-3, "nsecond": 1e-6}[unit]
        vals[row["Metric Name"]] = v * scale
    by[f"{cfg}/{prec}"] = {
        "kernel": kernel,
        "dram_bytes_per_launch": vals["dram__bytes_read.sum"] + vals["dram__bytes_write.sum"],
        "gpu_time_ms": vals["gpu__time_duration.sum"],
        "how": "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum "
               "--clock-control none, first P2P launch of bench.py (tools/p2p_traffic.sh)",
    }
json.dump(data, open(path, "w"), indent=1)
print(json.dumps(by, indent=1))
