"""SM clock and board power while ONE stage runs back to back (is a kernel power-capped?).
  python tools/stage_clock_probe.py --config C5 --stage m2l --seconds 2"""
import argparse, os, sys, threading, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import pynvml
import paper_1203_0889_b200 as fb
from bench import CONFIGS

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C5")
ap.add_argument("--stage", default="m2l")
ap.add_argument("--seconds", type=float, default=2.0)
a = ap.parse_args()
gen, n, p, n_crit, theta = CONFIGS[a.config]
ctx = fb.Context(order=p, n_crit=n_crit, theta=theta, precision="fp32")
ctx.set_bodies(fb.generate_bodies(gen, n, 1))
ctx.set_overlap(False)
ctx.evaluate()
pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(0)
samples, stop = [], False
def sampler():
    while not stop:
        samples.append((pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM), pynvml.nvmlDeviceGetPowerUsage(h) / 1000.0,
                        pynvml.nvmlDeviceGetCurrentClocksThrottleReasons(h)))
        time.sleep(0.01)
th = threading.Thread(target=sampler); th.start()
t0 = time.time(); k = 0
fn = getattr(ctx, a.stage)
while time.time() - t0 < a.seconds:
    fn(); k += 1
import torch
torch.cuda.synchronize()
dt = time.time() - t0
stop = True; th.join()
half = samples[len(samples) // 2:]
print(a.config, a.stage, f"{1e3 * dt / k:.3f} ms/call", "sm MHz median", int(np.median([s[0] for s in half])),
      "min", min(s[0] for s in half), "power W median", round(float(np.median([s[1] for s in half])), 1),
      "max", round(max(s[1] for s in half), 1), "reasons", sorted({hex(s[2]) for s in half}))
