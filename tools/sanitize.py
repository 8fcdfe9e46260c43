"""Small FMM steps for compute-sanitizer (memcheck / racecheck / synccheck): FP32 and FP64,
mutual, p = 4 and p = 8 (both M2L kernels), tree reuse."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1203_0889_b200 as fb  # noqa: E402

b = fb.generate_bodies(3, 3000, 1)
for p, prec, mutual in ((4, "fp32", False), (4, "fp64", False), (8, "fp32", False), (10, "fp32", False),
                        (4, "fp32", True)):
    ctx = fb.Context(order=p, n_crit=32, theta=0.5, precision=prec, mutual=mutual)
    ctx.set_bodies(b)
    ctx.evaluate()
    ctx.evaluate()
    if not mutual:
        ctx.update_bodies(b)
        ctx.evaluate_reuse()
    phi, acc = ctx.results("input")
    print(p, prec, mutual, float(phi[:4].sum()))
    ctx.close()
