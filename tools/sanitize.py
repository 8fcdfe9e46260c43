"""Small FMM steps for compute-sanitizer (memcheck / racecheck / synccheck / initcheck): FP32 and
FP64, p = 4 / 8 / 10 (both M2L kernels), mutual, tree reuse, the forced 64-bit-key traversal with
its look-back emission and the overflow regrow path, and the stage-isolated entry points.
Usage: compute-sanitizer --tool <tool> python tools/sanitize.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1203_0889_b200 as fb  # noqa: E402

b = fb.generate_bodies(3, 3000, 1)
for p, prec, mutual, dbg in ((4, "fp32", False, None), (4, "fp64", False, None), (8, "fp32", False, None),
                             (10, "fp32", False, None), (6, "fp64", False, None), (4, "fp32", True, None),
                             (6, "fp32", False, (True, 256)), (6, "fp64", False, (True, 0))):
    ctx = fb.Context(order=p, n_crit=32, theta=0.5, precision=prec, mutual=mutual)
    ctx.set_bodies(b)
    if dbg:
        ctx.set_traversal_debug(*dbg)
    ctx.evaluate()
    ctx.evaluate()
    if not mutual:
        ctx.update_bodies(b)
        ctx.evaluate_reuse()
    phi, acc = ctx.results("input")
    print(p, prec, mutual, dbg, float(phi[:4].sum()), flush=True)
    ctx.close()
# staged entry points (the sharded building blocks): world 2 emulated sequentially
ctxs = [fb.Context(order=6, n_crit=32, theta=0.5, precision="fp32") for _ in range(2)]
import numpy as np  # noqa: E402
import torch  # noqa: E402
sends = []
for r, ctx in enumerate(ctxs):
    ctx.set_bodies(b)
    ctx.set_partition(r, 2)
    ctx.build_tree()
    ctx.traverse()
    info = ctx.shard_info()
    s = torch.zeros(max(info.chunk_doubles, 1), dtype=torch.float64, device="cuda")
    ctx.upward_local(s.data_ptr())
    ctx.synchronize()
    sends.append(s)
recv = torch.cat(sends)
torch.cuda.synchronize()
for ctx in ctxs:
    ctx.upward_finish(recv.data_ptr())
    ctx.reset_accumulators()
    ctx.m2l()
    ctx.p2p()
    ctx.downward()
    print("sharded rank", ctx.shard_info().rank, float(ctx.results("tree")[0][:4].sum()), flush=True)
    ctx.close()
print("sanitize.py done")
