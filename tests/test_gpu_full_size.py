"""GPU parity at the full BASELINE.json sizes (north_star: "per-particle potential and
acceleration match the reference FMM within a relative L2 error of 1e-6 in FP64 mode and 1e-4 in
FP32-P2P mode, with trees and interaction lists bit-exact").

Reference contract: proj/tests/test_traversal.cpp:292-318 (serial pipeline), acceptance.cpp:99-123
(sorted list multisets), oracle.cpp:25-47 (compare). The checker is the oracle's OpenMP
pipeline (orc_evaluate_par), bit-identical to its serial restatement
(tests/test_oracle.py::test_parallel_checker_is_bit_identical), which is itself pinned to the
unmodified reference build.

  C2, C3, C5  every cell, the permutation, both CSR lists and every body's phi / acceleration;
  C4          every cell, the permutation and both lists (242 M + 83 M pairs); phi / acceleration
              on every 64th leaf (the oracle's pipeline restricted to those leaves and their
              ancestors: identical bits there, 1/64 of the near-field work).
C3-C5 have > 2^16 cells: the production traversal emits 64-bit keys with the ordered look-back
emission there, and C4 regrows its buffers; `test_traversal_debug_paths` forces both paths on
small trees too.

Each measured rel-L2 is appended to $FMM_PARITY_LOG (default gpurun_out/parity_full_size.jsonl);
the committed copy is profiles/r2_parity_full_size.jsonl.
"""
import json
import os
import time

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CELL_KEYS = ["level", "key", "center", "radius", "body_begin", "body_end", "child_begin",
             "child_count", "parent"]
TOL = {"fp64": 1e-6, "fp32": 1e-4}
FULL = {  # BASELINE.json configs: generator, N, p, n_crit, theta
    "C2": (2, 1 << 20, 6, 64, 0.5),
    "C3": (3, 1 << 20, 6, 64, 0.5),
    "C4": (4, 1 << 24, 8, 128, 0.4),
    "C5": (5, 1 << 22, 10, 64, 0.5),
}


def rel_l2(a, b):
    a = np.asarray(a, dtype=np.float64).ravel()
    b = np.asarray(b, dtype=np.float64).ravel()
    return float(np.sqrt(((a - b) ** 2).sum() / (b * b).sum()))


def _log(rec):
    path = os.environ.get("FMM_PARITY_LOG", os.path.join(ROOT, "gpurun_out", "parity_full_size.jsonl"))
    try:
        os.makedirs(os.path.dirname(path), exist_ok=True)
        with open(path, "a") as f:
            f.write(json.dumps(rec) + "\n")
    except OSError:
        pass


def _check_tree_and_lists(ctx, ocells, operm, olists, name):
    cells = ctx.cells()
    for k in CELL_KEYS:
        assert np.array_equal(cells[k], getattr(ocells, k)), (name, k)
    assert np.array_equal(ctx.permutation(), operm), name
    mo, ms, po, ps = ctx.lists()
    omo, oms, opo, ops = olists
    assert np.array_equal(mo, omo) and np.array_equal(ms, oms), (name, "m2l list")
    assert np.array_equal(po, opo) and np.array_equal(ps, ops), (name, "p2p list")


@pytest.mark.parametrize("name", ["C2", "C3", "C5"])
def test_full_size_parity(fmmlib, orc, name):
    """Whole-problem parity at the BASELINE size, both precision modes."""
    gen, n, p, n_crit, theta = FULL[name]
    bodies = orc.generate_baseline_bodies(gen, n, 1)
    t0 = time.time()
    t = orc.build_tree(bodies, n_crit, p)
    olists = orc.lists_csr(t, theta)
    orc.evaluate_par(t, theta, with_acc=True)
    t_oracle = time.time() - t0
    ocells, operm = t.cells(), t.perm()
    ophi, oacc = t.phi(), t.acc()
    del t
    for precision in ("fp64", "fp32"):
        ctx = fmmlib.Context(order=p, n_crit=n_crit, theta=theta, precision=precision, with_acc=True)
        ctx.set_bodies(bodies)
        ctx.evaluate()
        _check_tree_and_lists(ctx, ocells, operm, olists, name)
        phi, acc = ctx.results("tree")
        e_phi, e_acc = rel_l2(phi, ophi), rel_l2(acc, oacc)
        info = ctx.tree_info()
        _log({"config": name, "n": n, "precision": precision, "ncells": int(info.ncells),
              "n_m2l": int(info.n_m2l), "n_p2p": int(info.n_p2p),
              "p2p_body_pairs": int(info.p2p_body_pairs), "tree_bit_exact": True,
              "lists_bit_exact": True, "rel_l2_phi": e_phi, "rel_l2_acc": e_acc,
              "bodies_compared": n, "tol": TOL[precision], "oracle_s": round(t_oracle, 1)})
        assert e_phi <= TOL[precision], (name, precision, e_phi)
        assert e_acc <= TOL[precision], (name, precision, e_acc)
        ctx.close()


def test_c4_full_size(fmmlib, orc):
    """C4 (N = 16 777 216, p = 8, n_crit = 128, theta = 0.4): tree, permutation and lists
    bit-exact at full size; phi / acceleration on every 64th leaf in both modes."""
    gen, n, p, n_crit, theta = FULL["C4"]
    bodies = orc.generate_baseline_bodies(gen, n, 1)
    t = orc.build_tree(bodies, n_crit, p)
    ocells, operm = t.cells(), t.perm()
    olists = orc.lists_csr(t, theta)
    leaves = np.flatnonzero(ocells.child_count == 0)[::64]
    mask = np.zeros(len(ocells), bool)
    mask[leaves] = True
    orc.evaluate_par(t, theta, with_acc=True, leaf_mask=mask)
    sel = np.concatenate([np.arange(ocells.body_begin[k], ocells.body_end[k]) for k in leaves])
    ophi, oacc = t.phi()[sel], t.acc()[sel]
    del t
    for precision in ("fp32", "fp64"):
        ctx = fmmlib.Context(order=p, n_crit=n_crit, theta=theta, precision=precision, with_acc=True)
        ctx.set_bodies(bodies)
        ctx.evaluate()
        if precision == "fp32":  # the tree and lists do not depend on the precision mode
            _check_tree_and_lists(ctx, ocells, operm, olists, "C4")
        phi, acc = ctx.results("tree")
        e_phi, e_acc = rel_l2(phi[sel], ophi), rel_l2(acc[sel], oacc)
        info = ctx.tree_info()
        _log({"config": "C4", "n": n, "precision": precision, "ncells": int(info.ncells),
              "n_m2l": int(info.n_m2l), "n_p2p": int(info.n_p2p),
              "p2p_body_pairs": int(info.p2p_body_pairs), "tree_bit_exact": True,
              "lists_bit_exact": True, "rel_l2_phi": e_phi, "rel_l2_acc": e_acc,
              "bodies_compared": int(len(sel)), "leaves_compared": int(len(leaves)),
              "traversal_regrows": ctx.traversal_regrows(), "tol": TOL[precision]})
        assert e_phi <= TOL[precision], (precision, e_phi)
        assert e_acc <= TOL[precision], (precision, e_acc)
        ctx.close()


DEBUG_CASES = [  # name, generator, N, p, n_crit, theta, mutual
    ("C2-60k", 2, 60000, 6, 64, 0.5, False),
    ("C3-40k", 3, 40000, 6, 64, 0.5, False),
    ("C5-30k-mutual", 5, 30000, 8, 64, 0.5, True),
]


@pytest.mark.parametrize("case", DEBUG_CASES, ids=[c[0] for c in DEBUG_CASES])
def test_traversal_debug_paths(fmmlib, orc, case):
    """The traversal paths that only large trees take in production, forced on small trees
    (fmm_set_traversal_debug): 64-bit keys with the ordered look-back emission (> 2^16 cells:
    C3-C5), and the overflow regrow-and-rerun from a 512-entry start (C4). Lists bit-exact and
    potentials within the FP64 bar in every combination."""
    name, gen, n, p, n_crit, theta, mutual = case
    bodies = orc.generate_baseline_bodies(gen, n, 3)
    t = orc.build_tree(bodies, n_crit, p)
    olists = orc.lists_csr(t, theta, mutual=mutual)
    if mutual:
        orc.evaluate(t, theta, mutual=True, with_acc=True)
    else:
        orc.evaluate_par(t, theta, with_acc=True)
    ophi, oacc = t.phi(), t.acc()
    for keys64, cap in ((True, 0), (False, 512), (True, 512)):
        ctx = fmmlib.Context(order=p, n_crit=n_crit, theta=theta, precision="fp64", with_acc=True,
                             mutual=mutual)
        ctx.set_bodies(bodies)
        ctx.set_traversal_debug(keys64, cap)
        ctx.evaluate()
        mo, ms, po, ps = ctx.lists()
        assert np.array_equal(mo, olists[0]) and np.array_equal(ms, olists[1]), (name, keys64, cap)
        assert np.array_equal(po, olists[2]) and np.array_equal(ps, olists[3]), (name, keys64, cap)
        if cap:
            assert ctx.traversal_regrows() > 0
        phi, acc = ctx.results("tree")
        assert rel_l2(phi, ophi) <= 1e-6, (name, keys64, cap, rel_l2(phi, ophi))
        assert rel_l2(acc, oacc) <= 1e-6, (name, keys64, cap, rel_l2(acc, oacc))
        ctx.close()
