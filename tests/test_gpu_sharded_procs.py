"""fmm_evaluate_sharded with world = 2 in two processes on one GPU: the library's whole sharded
step (partition plan, own-cell upward on the exchange stream under the P2P kernel, all-gather,
shared ancestors, M2L, L2L/L2P) with the all-gather routed through gloo by fmm_set_allgather,
and fmm_set_bodies_shard's share exchange. The union of the ranks' owned results equals one
context's fmm_evaluate (first step: full traversal + plan; later steps: kept plan, filtered
traversal)."""
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("precision,tol", [("fp64", 1e-12), ("fp32", 1e-6)])
def test_sharded_step_two_processes(fmmlib, tmp_path, precision, tol):
    fb = fmmlib
    world, port = 2, str(_port())
    outs = [str(tmp_path / f"r{r}.npz") for r in range(world)]
    procs = [subprocess.Popen([sys.executable, os.path.join(HERE, "helpers", "sharded_worker.py"), str(r),
                               str(world), port, precision, outs[r]], stdout=subprocess.PIPE,
                              stderr=subprocess.STDOUT, text=True) for r in range(world)]
    logs = [p.communicate(timeout=600)[0] for p in procs]
    for p, log in zip(procs, logs):
        assert p.returncode == 0, log
    bodies = fb.generate_bodies(3, 60000, 21)
    ref = fb.Context(order=6, n_crit=64, theta=0.5, precision=precision)
    ref.set_bodies(bodies)
    ref.evaluate()
    phi_ref, acc_ref = ref.results("input")
    ref.close()
    r = [np.load(o) for o in outs]
    for step in range(3):
        phi = np.full(len(bodies), np.nan)
        acc = np.full((len(bodies), 3), np.nan)
        ranges = [x[f"range{step}"] for x in r]
        assert ranges[0][0] == 0 and ranges[0][1] == ranges[1][0] and ranges[1][1] == len(bodies)
        for x in r:
            phi[x[f"idx{step}"]] = x[f"phi{step}"]
            acc[x[f"idx{step}"]] = x[f"acc{step}"]
        assert np.isfinite(phi).all() and np.isfinite(acc).all()  # every body owned exactly once
        e_phi = np.linalg.norm(phi - phi_ref) / np.linalg.norm(phi_ref)
        e_acc = np.linalg.norm(acc - acc_ref) / np.linalg.norm(acc_ref)
        assert e_phi < tol and e_acc < tol, (precision, step, e_phi, e_acc)
    # per step: one multipole exchange; steps 1-2 also exchange the body shares
    assert len(r[0]["calls"]) == 5
