"""The library-owned NCCL path on one GPU (a world-1 communicator): fmm_comm_init,
fmm_set_bodies_shard (H2D of the share + ncclAllGather) and fmm_evaluate_sharded give the same
bits as fmm_set_bodies + fmm_evaluate. (NCCL refuses two ranks on one device, so world > 1 runs
only on a multi-GPU node; its data path is covered by the emulated-rank tests in
test_gpu_parity.py, which call the same pack / exchange / unpack stages.)"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("precision", ["fp32", "fp64"])
def test_world1_comm_matches_evaluate(fmmlib, precision):
    fb = fmmlib
    bodies = fb.generate_bodies(3, 50000, 9)
    ref = fb.Context(order=6, n_crit=64, theta=0.5, precision=precision)
    ref.set_bodies(bodies)
    ref.evaluate()
    phi_ref, acc_ref = ref.results("input")
    ctx = fb.Context(order=6, n_crit=64, theta=0.5, precision=precision)
    ctx.comm_init(fb.fmm.comm_unique_id(), 0, 1)
    for _ in range(2):
        ctx.set_bodies_shard(bodies, len(bodies))
        info = ctx.evaluate_sharded()
    assert (info.rank, info.world, info.body_begin, info.body_end) == (0, 1, 0, len(bodies))
    phi, acc, idx = ctx.owned_results(info)
    assert np.array_equal(np.sort(idx), np.arange(len(bodies)))
    assert np.array_equal(phi, phi_ref[idx]) and np.array_equal(acc, acc_ref[idx])
    assert ctx.stage_times().exchange_ms == 0.0
    ctx.comm_destroy()
    ctx.close()
    ref.close()


def test_shard_size_is_checked(fmmlib):
    fb = fmmlib
    ctx = fb.Context(order=4)
    with pytest.raises(fb.FMMError, match="no communicator"):
        ctx.set_bodies_shard(np.zeros((10, 4)), 10)
    ctx.comm_init(fb.fmm.comm_unique_id(), 0, 1)
    with pytest.raises(fb.FMMError, match="share size"):
        ctx.set_bodies_shard(np.zeros((9, 4)), 10)
    ctx.close()
