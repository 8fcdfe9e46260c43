"""Multi-GPU host logic on the CPU: the partition plan of the C-ABI
(fmm_plan_partition, host-only) and the sharded multipole exchange protocol, run as a
world_size-2 gloo job. The CPU oracle stands in for the per-rank GPU kernels (test
infrastructure only): each rank computes its own cells' multipoles, all-gathers equal-size chunks,
unpacks the others and recomputes the straddling ancestors; the assembled multipoles must equal
the single-process ones bit for bit."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_1203_0889_b200 import fmm

CELL_KEYS = ["body_begin", "body_end", "child_count"]


def leaf_costs(orc, t, theta):
    c = t.cells()
    m, p = orc.traverse(t, theta)
    nb = (c.body_end - c.body_begin).astype(np.float64)
    cost = np.zeros(len(c))
    np.add.at(cost, p[:, 0], nb[p[:, 0]] * nb[p[:, 1]])
    np.add.at(cost, m[:, 0], 70.0)
    cost[c.child_count > 0] = 0.0
    return c, cost


@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_partition_plan(orc, world):
    bodies = fmm.generate_bodies(3, 20000, 4)  # Plummer: uneven costs
    t = orc.build_tree(bodies, 64, 4)
    c, cost = leaf_costs(orc, t, 0.5)
    cells = {k: getattr(c, k) for k in CELL_KEYS}
    bounds, owner = fmm.plan_partition(cells, cost, world)
    assert bounds[0] == 0 and bounds[-1] == len(bodies) and np.all(np.diff(bounds) >= 0)
    leaves = np.where(c.child_count == 0)[0]
    # every leaf is owned by exactly the rank whose range contains it (leaves never straddle)
    for leaf in leaves:
        r = owner[leaf]
        assert r >= 0 and bounds[r] <= c.body_begin[leaf] and c.body_end[leaf] <= bounds[r + 1]
    # non-leaf cells: owned iff inside one range, else shared (-1)
    for i in np.where(c.child_count > 0)[0]:
        inside = [r for r in range(world) if bounds[r] <= c.body_begin[i] and c.body_end[i] <= bounds[r + 1]
                  and bounds[r] < bounds[r + 1]]
        assert owner[i] == (inside[0] if inside else -1)
    # balanced: no rank above its fair share by more than the largest leaf cost
    per = np.array([cost[leaves[owner[leaves] == r]].sum() for r in range(world)])
    assert per.sum() == pytest.approx(cost.sum())
    assert per.max() <= cost.sum() / world + cost.max() + 1e-9


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, results):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        orc = oracle.Oracle()
        p = 5
        bodies = fmm.generate_bodies(3, 12000, 9)
        t = orc.build_tree(bodies, 32, p)  # identical tree on every rank (deterministic)
        c, cost = leaf_costs(orc, t, 0.5)
        bounds, owner = fmm.plan_partition({k: getattr(c, k) for k in CELL_KEYS}, cost, world)
        # reference multipoles (single process) and this rank's own cells
        orc.evaluate(t, 0.5, with_acc=False)
        M_full = t.multipoles()
        nc = M_full.shape[1]
        mine = [np.where(owner == r)[0] for r in range(world)]
        chunk = max(len(m) for m in mine)
        send = torch.zeros(chunk * nc, dtype=torch.float64)
        send[: len(mine[rank]) * nc] = torch.from_numpy(M_full[mine[rank]].ravel())
        recv = torch.zeros(world * chunk * nc, dtype=torch.float64)
        dist.all_gather_into_tensor(recv, send)
        M = np.zeros_like(M_full)
        rv = recv.numpy().reshape(world, chunk, nc)
        for r in range(world):
            M[mine[r]] = rv[r, : len(mine[r])]
        # straddling cells, deepest level first, M2M from children in child order
        ops = oracle.OracleOps(orc, p)
        shared = np.where(owner == -1)[0]
        for ci in sorted(shared, key=lambda i: -c.level[i]):
            acc = np.zeros(nc)
            for k in range(c.child_count[ci]):
                ch = c.child_begin[ci] + k
                acc += ops.m2m(M[ch], c.center[ch] - c.center[ci])
            M[ci] = acc
        results[rank] = (bool(np.array_equal(M[owner >= 0], M_full[owner >= 0])),
                         float(np.abs(M[shared] - M_full[shared]).max() / np.abs(M_full).max()) if len(shared) else 0.0,
                         int(len(shared)), [int(b) for b in bounds])
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_sharded_exchange_gloo(world):
    mgr = mp.Manager()
    results = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), results), nprocs=world, join=True)
    assert len(results) == world
    for r in range(world):
        exact_owned, shared_err, nshared, bounds = results[r]
        assert exact_owned
        assert shared_err < 1e-13  # recomputed ancestors: same M2M arithmetic, summed per child
        assert nshared >= 1
    assert results[0][3] == results[1][3]  # every rank derives the same plan
