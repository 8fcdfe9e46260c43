"""FP32-P2P mode accuracy at full BASELINE sizes: rel-L2 of phi and acceleration of the FP32-P2P
run against the FP64 run of the same tree and lists (FP64 mode is checked against the oracle
at 1e-15 in tests/). Prints one JSON line per config."""
import json
import sys
import os

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1203_0889_b200 as fb  # noqa: E402

CONFIGS = {"C1": (1, 16384, 4, 64, 0.5), "C2": (2, 1 << 20, 6, 64, 0.5), "C3": (3, 1 << 20, 6, 64, 0.5),
           "C4": (4, 1 << 24, 8, 128, 0.4), "C5": (5, 1 << 22, 10, 64, 0.5)}


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


for name in (sys.argv[1:] or list(CONFIGS)):
    gen, n, p, nc, th = CONFIGS[name]
    bodies = fb.generate_bodies(gen, n, 1)
    out = {}
    for prec in ("fp64", "fp32"):
        ctx = fb.Context(order=p, n_crit=nc, theta=th, precision=prec)
        ctx.set_bodies(bodies)
        ctx.evaluate()
        out[prec] = ctx.results("tree")
        ctx.close()
    (p64, a64), (p32, a32) = out["fp64"], out["fp32"]
    amag = np.linalg.norm(a64.reshape(-1, 3), axis=1)
    err = np.linalg.norm((a32 - a64).reshape(-1, 3), axis=1)
    worst = int(np.argmax(err))
    print(json.dumps({"config": name, "rel_l2_phi": rel(p32, p64), "rel_l2_acc": rel(a32, a64),
                      "max_body_rel_acc": float((err / np.maximum(amag, 1e-300)).max()),
                      "worst_body_share_of_acc_norm2": float(amag[worst] ** 2 / (amag ** 2).sum())}),
          flush=True)
