"""Phase breakdown of sampled P2P CTAs (variant library built with -DFMM_P2P_TRACE=1):
  bash tools/build_variant.sh trace p2p "-DFMM_P2P_TRACE=1"
  FMM_B200_LIB=$PWD/paper_1203_0889_b200/lib/libfmm_b200_trace.so python tools/p2p_trace.py --config C5"""
import argparse, ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1203_0889_b200 as fb
from bench import CONFIGS

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C5")
a = ap.parse_args()
gen, n, p, n_crit, theta = CONFIGS[a.config]
ctx = fb.Context(order=p, n_crit=n_crit, theta=theta, precision="fp32")
ctx.set_bodies(fb.generate_bodies(gen, n, 1))
ctx.set_overlap(False)
for _ in range(2):
    ctx.evaluate()
st = ctx.stage_times()
nct = 1 << 16
buf = np.zeros((nct, 16), np.uint64)
rc = ctx.lib.fmm_debug_p2p_trace(buf.ctypes.data_as(C.POINTER(C.c_ulonglong)), nct)
assert rc == 0
ok = buf[:, 9] > 0
t = buf[ok].astype(np.int64)
print(a.config, "p2p kernel ms", round(st.p2p_kernel_ms, 3), "sampled CTAs", len(t))
names = ["entry->item+sync", "->tile0 set up (entries loaded)", "->copies issued", "->copies landed", "->converted+published",
         "consumer sees tile0 (from entry)", "pair loops (tile0 seen->done)", "reduce+write", "whole CTA"]
d = np.stack([t[:, 1] - t[:, 0], t[:, 2] - t[:, 1], t[:, 3] - t[:, 2], t[:, 4] - t[:, 3], t[:, 5] - t[:, 4],
              t[:, 7] - t[:, 0], t[:, 8] - t[:, 7], t[:, 9] - t[:, 8], t[:, 9] - t[:, 0]], axis=1)
print("tiles per item: mean %.2f  targets per item: mean %.1f" % (t[:, 10].mean(), t[:, 11].mean()))
for i, nm in enumerate(names):  # noqa
    print(f"  {nm:40s} mean {d[:, i].mean():9.0f}  median {np.median(d[:, i]):9.0f}  p90 {np.percentile(d[:, i], 90):9.0f} cycles")
