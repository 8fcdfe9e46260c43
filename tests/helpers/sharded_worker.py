"""One rank of the multi-process sharded-step test (tests/test_gpu_sharded_procs.py): the library's
fmm_evaluate_sharded with its exchange routed through a gloo all-gather on the host
(fmm_set_allgather), so two processes can share one GPU (NCCL refuses two ranks on one device).
Usage: python sharded_worker.py <rank> <world> <port> <precision> <out.npz>"""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_1203_0889_b200 as fb  # noqa: E402


class _Dev:  # zero-copy torch view of a device pointer
    def __init__(self, ptr, n):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<f8", "data": (ptr, False),
                                         "version": 3, "strides": None}


def main():
    rank, world, port, precision, out = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3], sys.argv[4], sys.argv[5]
    dist.init_process_group("gloo", rank=rank, world_size=world, init_method=f"tcp://127.0.0.1:{port}")
    torch.cuda.set_device(0)
    n = 60000
    bodies = fb.generate_bodies(3, n, 21)
    ctx = fb.Context(order=6, n_crit=64, theta=0.5, precision=precision)
    ctx.set_partition(rank, world)
    calls = []

    def all_gather(d_send, d_recv, count, stream):
        torch.cuda.ExternalStream(stream).synchronize()  # the library's send buffer is complete
        send = torch.as_tensor(_Dev(d_send, count), device="cuda").cpu()
        parts = [torch.empty(count, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(parts, send)
        torch.as_tensor(_Dev(d_recv, world * count), device="cuda").copy_(torch.cat(parts).cuda())
        torch.cuda.synchronize()
        calls.append(count)

    ctx.set_allgather(all_gather)
    chunk = (n + world - 1) // world
    b0, b1 = min(n, rank * chunk), min(n, (rank + 1) * chunk)
    res = {}
    for step in range(3):
        if step == 0:
            ctx.set_bodies(bodies)
        else:  # the rank's share only, all-gathered through the same callback
            ctx.set_bodies_shard(bodies[b0:b1], n)
        info = ctx.evaluate_sharded()
        phi, acc, idx = ctx.owned_results(info)
        res[f"phi{step}"], res[f"acc{step}"], res[f"idx{step}"] = phi, acc, idx
        res[f"range{step}"] = np.array([info.body_begin, info.body_end])
        res[f"exch{step}"] = np.array([ctx.stage_times().exchange_ms])
    res["calls"] = np.array(calls)
    np.savez(out, **res)
    ctx.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
