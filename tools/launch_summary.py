"""Per-kernel share of one step from an ncu launch list (--metrics gpu__time_duration.sum --csv):
the launches of the last `--steps` evaluate() calls are grouped by kernel name.
Usage: python tools/launch_summary.py launches.csv [n_last_launches]"""
import csv
import re
import sys
from collections import OrderedDict


def main(path, last=None):
    rows = []
    with open(path) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    for r in csv.DictReader(lines):
        if r.get("Metric Name") == "gpu__time_duration.sum":
            name = re.sub(r"\(.*", "", r["Kernel Name"]).replace("fmmb::<unnamed>::", "")
            rows.append((name, float(r["Metric Value"]) / 1e6 if r["Metric Unit"] == "ns" else float(r["Metric Value"])))
    if last:
        rows = rows[-last:]
    agg = OrderedDict()
    for n, t in rows:
        a = agg.setdefault(n, [0, 0.0])
        a[0] += 1
        a[1] += t
    tot = sum(a[1] for a in agg.values())
    print(f"{len(rows)} launches, {tot:.3f} ms total (serialised under ncu)")
    for n, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{t:9.3f} ms {100 * t / tot:5.1f} %  x{c:<4d} {n}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else None)
