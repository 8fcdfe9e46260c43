"""Generates the committed golden fixtures from the UNMODIFIED reference (oracle/_ref).

Run in the build container (needs /root/reference to have built oracle/_ref):

    python tests/golden/make_golden.py

Outputs (all small, committed):
  ref_cases.npz    per case: input bodies, tree cells, body permutation, sorted M2L/P2P
                   emitted pairs, potentials (tree order), multipoles and locals of the
                   reference's serial pipeline (test_traversal.cpp:292-318 semantics); the
                   same lists and potentials in mutual mode (test_traversal.cpp:320-345).
  aggregates.json  the proj/test_output.txt aggregates reproduced by the reference build, plus
                   BASELINE C1 tree / list counts for the repo's synthetic generator.
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402


def pair_keys(p):
    p = np.asarray(p, dtype=np.int64).reshape(-1, 2)
    return np.sort((p[:, 0] << 32) | p[:, 1])


# (name, bodies generator, n_crit, p, theta)
def cases(ref: oracle.Reference):
    out = []
    out.append(("cube2048_p6", ref.generate_bodies(0, 2048, 15), 64, 6, 0.5))
    out.append(("cluster512_p3", ref.generate_bodies(2, 512, 12), 16, 3, 0.5))
    out.append(("sphere2000_p5", ref.generate_bodies(1, 2000, 18), 32, 5, 0.5))
    out.append(("cube4096_p3_q", ref.generate_bodies(0, 4096, 3), 64, 3, 0.5))
    b = np.zeros((9, 4))
    b[:, :3] = 0.25
    b[:, 3] = 1.0
    out.append(("coincident9_p2", b, 8, 2, 0.5))
    one = np.array([[1.0, 2.0, 3.0, 1.0]])
    out.append(("single_p3", one, 8, 3, 0.5))
    g = (np.arange(8) + 0.5) / 8
    X, Y, Z = np.meshgrid(g, g, g, indexing="ij")
    grid = np.stack([X.ravel(), Y.ravel(), Z.ravel(), np.where((np.arange(512) % 2) == 0, 1.0, -1.0)], 1)
    out.append(("grid512_p4_theta04", grid, 8, 4, 0.4))
    return out


def main():
    ref = oracle.Reference()
    data = {}
    for name, bodies, n_crit, p, theta in cases(ref):
        t = ref.build_tree(bodies, n_crit, p)
        c = t.cells()
        m, pp = t.traverse(theta)
        t.pipeline(theta)
        M, L = t.expansions()
        data[f"{name}/bodies"] = bodies
        data[f"{name}/params"] = np.array([n_crit, p, theta])
        for k in ["level", "key", "center", "radius", "body_begin", "body_end", "child_begin",
                  "child_count", "parent"]:
            data[f"{name}/{k}"] = getattr(c, k)
        data[f"{name}/perm"] = t.perm()
        data[f"{name}/m2l"] = pair_keys(m)
        data[f"{name}/p2p"] = pair_keys(pp)
        data[f"{name}/phi"] = t.potentials()
        data[f"{name}/multipole"] = M
        data[f"{name}/local"] = L
        # mutual mode (traversal.hpp:76-84; m2l_mutual / mutual p2p): emitted once per
        # unordered pair, in the emitted orientation; potentials of the mutual pipeline
        tm = ref.build_tree(bodies, n_crit, p)
        mm, mp = tm.traverse(theta, mutual=True)
        tm.pipeline(theta, mutual=True)
        data[f"{name}/m2l_mutual"] = pair_keys(mm)
        data[f"{name}/p2p_mutual"] = pair_keys(mp)
        data[f"{name}/phi_mutual"] = tm.potentials()
    np.savez_compressed(os.path.join(HERE, "ref_cases.npz"), **data)

    agg = {}
    errs = {}
    for p in (3, 6, 9):
        e, _ = ref.run_once(10000, p, 0.5, 64, threads=1, seed=1)
        errs[str(p)] = e
    agg["rel_l2_N1e4_seed1"] = errs
    t = ref.build_tree(ref.generate_bodies(0, 4096, 3), 64, 3)
    m, pp = t.traverse(0.5, queue_threshold=64)
    agg["emitted_N4096_seed3_p3"] = int(len(m) + len(pp))
    evals = {}
    for mutual in (False, True):
        ref.counters_reset()
        ref.run_once(10000, 4, 0.5, 64, threads=1, mutual=mutual, seed=1, check=False)
        evals["mutual" if mutual else "non_mutual"] = ref.counters()[1]
    agg["p2p_evals_N1e4_p4"] = evals

    # BASELINE C1 with the repo generator (config 1, seed 1): tree and list sizes
    import paper_1203_0889_b200.fmm as fb  # host-side generator only (no GPU needed)
    c1 = fb.generate_bodies(1, 16384, 1)
    t = ref.build_tree(c1, 64, 4)
    c = t.cells()
    m, pp = t.traverse(0.5)
    nb = c.body_end - c.body_begin
    agg["C1"] = {"ncells": int(len(c)), "nleaves": int((c.child_count == 0).sum()),
                 "depth": int(c.level.max()), "n_m2l": int(len(m)), "n_p2p": int(len(pp)),
                 "p2p_body_pairs": int((nb[pp[:, 0]].astype(np.int64) * nb[pp[:, 1]]).sum())}
    with open(os.path.join(HERE, "aggregates.json"), "w") as f:
        json.dump(agg, f, indent=1, sort_keys=True)
    print(json.dumps(agg, indent=1))


if __name__ == "__main__":
    main()
