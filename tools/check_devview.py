# GPU check of the sharded e2e read-back: zero-copy torch views of the context result buffers
# (fmm_results_device) sliced to a body range equal fmm_get_results; NCCL all-gather at world 1.
import numpy as np, torch, sys, os
sys.path.insert(0, os.getcwd())
import paper_1203_0889_b200 as fb
import torch.distributed as dist
os.environ.setdefault("MASTER_ADDR", "127.0.0.1"); os.environ.setdefault("MASTER_PORT", "29533")
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
n = 1 << 14
b = fb.generate_bodies(1, n, 1)
ctx = fb.Context(order=4, n_crit=64, theta=0.5, precision="fp32", with_acc=True)
d_bodies = torch.empty((n, 4), dtype=torch.float64, device="cuda")
h_in = torch.from_numpy(np.ascontiguousarray(b[0:n])).pin_memory()
d_part = torch.empty_like(h_in, device="cuda")
d_part.copy_(h_in, non_blocking=True)
dist.all_gather_into_tensor(d_bodies, d_part)
ctx.set_bodies_device(d_bodies.data_ptr(), n)
ctx.evaluate()
class _Dev:
    def __init__(self, ptr, shape):
        self.__cuda_array_interface__ = {"shape": shape, "typestr": "<f8", "data": (ptr, False), "version": 3, "strides": None}
pphi, pacc = ctx.results_device()
d_phi = torch.as_tensor(_Dev(pphi, (n,)), device="cuda"); d_acc = torch.as_tensor(_Dev(pacc, (n, 3)), device="cuda")
h_phi = torch.empty(n, dtype=torch.float64).pin_memory(); h_acc = torch.empty((n, 3), dtype=torch.float64).pin_memory()
b0, b1 = 100, 9000
h_phi[:b1-b0].copy_(d_phi[b0:b1], non_blocking=True); h_acc[:b1-b0].copy_(d_acc[b0:b1], non_blocking=True)
torch.cuda.current_stream().synchronize()
phi, acc = ctx.results(order="tree")
print("phi eq", np.array_equal(phi[b0:b1], h_phi[:b1-b0].numpy()), "acc eq", np.array_equal(acc.reshape(-1,3)[b0:b1], h_acc[:b1-b0].numpy()))
dist.destroy_process_group()
