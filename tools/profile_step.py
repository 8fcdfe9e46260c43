"""Runs `--warmup` + `--steps` FMM evaluations of a BASELINE config (for ncu launch lists /
full captures of one step). Prints per-stage device times of the last step."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1203_0889_b200 as fb  # noqa: E402
from bench import CONFIGS  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C2")
ap.add_argument("--steps", type=int, default=1)
ap.add_argument("--warmup", type=int, default=2)
ap.add_argument("--precision", default="fp32")
ap.add_argument("--n", type=int, default=0, help="override the body count")
ap.add_argument("--serial", action="store_true", help="stages serialised on one stream")
ap.add_argument("--overlap", action="store_true", help="upward pass concurrent with the traversal")
ap.add_argument("--overlap-level", type=int, default=-1, help="fmm_set_overlap level (0, 1, 2)")
a = ap.parse_args()
gen, n, p, n_crit, theta = CONFIGS[a.config]
if a.n:
    n = a.n
b = fb.generate_bodies(gen, n, 1)
ctx = fb.Context(order=p, n_crit=n_crit, theta=theta, precision=a.precision)
ctx.set_bodies(b)
if a.serial:
    ctx.set_overlap(False)
if a.overlap:
    ctx.set_overlap(1)
if a.overlap_level >= 0:
    ctx.set_overlap(a.overlap_level)
for _ in range(a.warmup):
    ctx.evaluate()
acc = {}
for _ in range(a.steps):  # stage times averaged over the timed steps
    ctx.evaluate()
    t = ctx.stage_times()
    for k, _ in t._fields_:
        acc[k] = acc.get(k, 0.0) + getattr(t, k) / a.steps
print({k: round(v, 3) for k, v in acc.items()})
info = ctx.tree_info()
print("cells", info.ncells, "leaves", info.nleaves, "depth", info.depth, "m2l", info.n_m2l,
      "p2p", info.n_p2p, "pairs", info.p2p_body_pairs)
