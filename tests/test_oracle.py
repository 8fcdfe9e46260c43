"""Pins the CPU oracle (oracle/fmm_oracle.c) before it is trusted as the parity checker.

* known answers of proj/tests/test_{kernels,multi_index,tree,traversal}.cpp,
* the golden aggregates of proj/test_output.txt:12-20,
* the committed fixtures of tests/golden/ (produced by the unmodified reference),
* bit-exact agreement with oracle/_ref when it is present,
* the acceleration extension against a long-double direct-sum gradient.
"""
import json
import os

import numpy as np
import pytest

import oracle
from conftest import sorted_pairs

GOLD = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def fixtures():
    return np.load(os.path.join(GOLD, "ref_cases.npz"))


@pytest.fixture(scope="module")
def aggregates():
    with open(os.path.join(GOLD, "aggregates.json")) as f:
        return json.load(f)


def case_names(fx):
    return sorted({k.split("/")[0] for k in fx.files})


# ------------------------------------------------------------- golden aggregates ----
def test_golden_accuracy_aggregates(orc, aggregates):
    """test_output.txt:12 — rel_l2 3.34e-03 > 5.89e-05 > 1.78e-06 (N=1e4, cube, seed 1)."""
    bodies = orc.generate_reference_bodies(0, 10000, 1)
    got = {}
    for p in (3, 6, 9):
        t = orc.build_tree(bodies, 64, p)
        orc.evaluate(t, 0.5, with_acc=False)
        phi_d, _ = orc.direct_sum(t.positions(), t.charges(), with_acc=False)
        got[p] = orc.compare(t.phi(), phi_d)[0]
    assert f"{got[3]:.2e}" == "3.34e-03"
    assert f"{got[6]:.2e}" == "5.89e-05"
    assert f"{got[9]:.2e}" == "1.78e-06"
    for p in (3, 6, 9):
        assert got[p] == pytest.approx(aggregates["rel_l2_N1e4_seed1"][str(p)], rel=1e-9)


def test_golden_emitted_count(orc, aggregates):
    """test_output.txt:14 — 46 523 emitted interactions (N=4096, seed 3, p=3)."""
    t = orc.build_tree(orc.generate_reference_bodies(0, 4096, 3), 64, 3)
    m, p = orc.traverse(t, 0.5)
    assert len(m) + len(p) == 46523 == aggregates["emitted_N4096_seed3_p3"]


def test_golden_p2p_evals(orc, aggregates):
    """test_output.txt:15 — P2P evaluations 20 255 578 non-mutual, 10 127 789 mutual."""
    bodies = orc.generate_reference_bodies(0, 10000, 1)
    ev = {}
    for mutual in (False, True):
        t = orc.build_tree(bodies, 64, 4)
        ev[mutual] = orc.evaluate(t, 0.5, mutual=mutual, with_acc=False)[0]
    assert ev[False] == 20255578 == aggregates["p2p_evals_N1e4_p4"]["non_mutual"]
    assert ev[True] == 10127789 == aggregates["p2p_evals_N1e4_p4"]["mutual"]


def test_c1_counts_match_survey(orc, aggregates):
    """C1 = 585 cells / 512 leaves / depth 3, 93 536 M2L, 52 352 P2P, 53.4 M pairs."""
    import paper_1203_0889_b200.fmm as fb
    t = orc.build_tree(fb.generate_bodies(1, 16384, 1), 64, 4)
    c = t.cells()
    m, p = orc.traverse(t, 0.5)
    nb = (c.body_end - c.body_begin).astype(np.int64)
    got = {"ncells": len(c), "nleaves": int((c.child_count == 0).sum()), "depth": int(c.level.max()),
           "n_m2l": len(m), "n_p2p": len(p), "p2p_body_pairs": int((nb[p[:, 0]] * nb[p[:, 1]]).sum())}
    assert got == aggregates["C1"]


# ------------------------------------------------------------------ fixtures ----------
def test_oracle_reproduces_reference_fixtures(orc, fixtures):
    """Tree, permutation and lists bit-exact; serial-pipeline potentials bit-exact (the oracle
    applies the same operators in the same FIFO order as KernelVisitor)."""
    for name in case_names(fixtures):
        g = lambda k: fixtures[f"{name}/{k}"]  # noqa: E731
        n_crit, p, theta = g("params")
        t = orc.build_tree(g("bodies"), int(n_crit), int(p))
        c = t.cells()
        for k in ["level", "key", "center", "radius", "body_begin", "body_end", "child_begin",
                  "child_count", "parent"]:
            assert np.array_equal(getattr(c, k), g(k)), (name, k)
        assert np.array_equal(t.perm(), g("perm")), name
        m, pp = orc.traverse(t, float(theta))
        assert np.array_equal(sorted_pairs(m), g("m2l")), name
        assert np.array_equal(sorted_pairs(pp), g("p2p")), name
        orc.evaluate(t, float(theta), with_acc=False)
        assert np.array_equal(t.phi(), g("phi")), name
        assert np.array_equal(t.multipoles(), g("multipole")), name
        assert np.array_equal(t.locals(), g("local")), name


def test_oracle_mutual_reproduces_reference_fixtures(orc, fixtures):
    """Mutual mode (traversal.hpp:76-84, m2l_mutual / mutual p2p kernels.cpp:113-126, :153-180):
    the emitted lists, in their emitted orientation, and the mutual pipeline's potentials are
    bit-exact with the reference; the symmetrised mutual lists equal the non-mutual ones
    (test_traversal.cpp:182-210)."""
    for name in case_names(fixtures):
        g = lambda k: fixtures[f"{name}/{k}"]  # noqa: E731
        n_crit, p, theta = g("params")
        t = orc.build_tree(g("bodies"), int(n_crit), int(p))
        m, pp = orc.traverse(t, float(theta), mutual=True)
        assert np.array_equal(sorted_pairs(m), g("m2l_mutual")), name
        assert np.array_equal(sorted_pairs(pp), g("p2p_mutual")), name
        sym = lambda a: np.concatenate([a, a[a[:, 0] != a[:, 1]][:, ::-1]])  # noqa: E731
        assert np.array_equal(sorted_pairs(sym(m)), g("m2l")), name
        assert np.array_equal(sorted_pairs(sym(pp)), g("p2p")), name
        orc.evaluate(t, float(theta), mutual=True, with_acc=False)
        assert np.array_equal(t.phi(), g("phi_mutual")), name


def test_oracle_matches_reference_build(orc, ref):
    """Against the unmodified reference compiled here (bit-exact), on fresh inputs."""
    for dist, n, seed, n_crit, p in [(0, 3000, 7, 32, 4), (1, 2500, 8, 16, 6), (2, 3000, 9, 24, 5)]:
        b = ref.generate_bodies(dist, n, seed)
        assert np.array_equal(b, orc.generate_reference_bodies(dist, n, seed))
        rt = ref.build_tree(b, n_crit, p)
        t = orc.build_tree(b, n_crit, p)
        assert rt.cells().equal(t.cells())
        assert np.array_equal(rt.perm(), t.perm())
        rm, rp = rt.traverse(0.5, queue_threshold=64)
        m, pp = orc.traverse(t, 0.5)
        assert np.array_equal(sorted_pairs(rm), sorted_pairs(m))
        assert np.array_equal(sorted_pairs(rp), sorted_pairs(pp))
        rt.pipeline(0.5)
        orc.evaluate(t, 0.5, with_acc=True)
        assert np.array_equal(rt.potentials(), t.phi())


# ---------------------------------------------------------------- known answers -------
def test_known_answers_operators(orc):
    ops5 = oracle.OracleOps(orc, 5)
    M = ops5.p2m([[0.25, -0.5, 1.0, 2.0]], [0.25, -0.5, 1.0])  # test_kernels.cpp:25-34
    assert M[0] == 2.0 and np.abs(M[1:]).max() == 0.0
    ops3 = oracle.OracleOps(orc, 3)
    off = np.array([0.1, 0.2, -0.3])
    M = ops3.p2m([[*off, 1.0], [*(-off), -1.0]], [0, 0, 0])  # :36-49
    assert M[0] == pytest.approx(0.0)
    from paper_1203_0889_b200.fmm import index_of
    assert M[index_of(1, 0, 0)] == pytest.approx(2 * off[0])
    assert M[index_of(0, 1, 0)] == pytest.approx(2 * off[1])
    assert M[index_of(0, 0, 1)] == pytest.approx(2 * off[2])
    Mm = np.zeros(ops3.n)
    Mm[0] = 5.0
    assert ops3.m2l(Mm, [2.0, 0, 0])[0] == pytest.approx(2.5)  # :108-115
    assert oracle.OracleOps(orc, 1).m2l([-1.5], [1.0, 2.0, -2.0])[0] == pytest.approx(-0.5)  # :117-125
    with pytest.raises(oracle.OracleError, match="singular M2L displacement"):
        oracle.OracleOps(orc, 2).m2l(np.zeros(4), [0, 0, 0])
    ops6 = oracle.OracleOps(orc, 6)
    M6 = np.zeros(ops6.n)
    M6[0] = 2.0
    assert ops6.evaluate_multipole(M6, [1, 5, 1], [1, 1, 1]) == pytest.approx(0.5)  # :325-335
    phi, _, _ = ops3.p2p([[0, 0, 0, 1.0], [1, 0, 0, 1.0]])  # :285-297
    assert phi == pytest.approx([1.0, 1.0])
    phi, _, ev = ops3.p2p([[0, 0, 0, 1.0], [0, 0, 0, 2.0], [0, 0, 2, 4.0]])  # :314-323
    assert phi == pytest.approx([2.0, 2.0, 1.5])
    assert ev == 4


def test_multi_index_order():
    """test_multi_index.cpp:8-24."""
    from paper_1203_0889_b200.fmm import exponents, n_coef
    assert n_coef(6) == 56 and n_coef(9) == 165
    e = exponents(2)
    assert e.tolist()[:4] == [[0, 0, 0], [0, 0, 1], [0, 1, 0], [1, 0, 0]]
    assert e[4].tolist() == [0, 0, 2] and e[9].tolist() == [2, 0, 0]


def test_tree_known_answers(orc):
    """test_tree.cpp:13-92: bounds, Morton (0.6,0.3,0.8)@L2 = 46, coincident chain of 22 cells."""
    c, h = orc.compute_bounds(np.array([[0, 0, 0, 0], [1, 1, 1, 0]], float))
    assert np.allclose(c, 0.5) and h == pytest.approx(0.5 * (1 + 1e-6), rel=1e-12)
    c, h = orc.compute_bounds(np.array([[3, 4, 5, 0]], float))
    assert h == 0.5
    assert orc.morton_key([0.6, 0.3, 0.8], [0.5, 0.5, 0.5], 0.5, 2) == 46
    assert orc.morton_key([1 - 1e-12] * 3, [0.5] * 3, 0.5, 1) == 7
    with pytest.raises(oracle.OracleError, match="level overflow"):
        orc.morton_key([0, 0, 0], [0.5] * 3, 0.5, 22)
    b = np.zeros((9, 4))
    b[:, :3] = 0.25
    t = orc.build_tree(b, 8, 2)
    cells = t.cells()
    assert len(cells) == 22
    leaves = np.where(cells.child_count == 0)[0]
    assert len(leaves) == 1 and cells.level[leaves[0]] == 21
    with pytest.raises(oracle.OracleError, match="empty input"):
        orc.build_tree(np.zeros((0, 4)), 8, 2)
    with pytest.raises(oracle.OracleError, match="n_crit must be >= 1"):
        orc.build_tree(b, 0, 2)
    with pytest.raises(oracle.OracleError, match="expansion order must be >= 1"):
        orc.build_tree(b, 8, 0)


def test_traversal_known_answers(orc):
    """test_traversal.cpp:161-180: a single-leaf tree emits one self P2P pair."""
    t = orc.build_tree(np.array([[0.5, 0.5, 0.5, 1.0]]), 8, 3)
    m, p = orc.traverse(t, 0.5)
    assert len(m) == 0 and p.tolist() == [[0, 0]]


# ---------------------------------------------------------- acceleration extension ----
def test_direct_sum_equals_p2p(orc):
    """test_oracle.cpp:26-33: direct sum vs P2P within 1e-12 (phi and the acc extension)."""
    rng = np.random.default_rng(5)
    b = np.concatenate([rng.uniform(-1, 1, (300, 3)), rng.uniform(-1, 1, (300, 1))], 1)
    phi_d, acc_d = orc.direct_sum(b[:, :3], b[:, 3])
    phi_p, acc_p, _ = oracle.OracleOps(orc, 2).p2p(b)
    assert orc.compare(phi_p, phi_d)[0] <= 1e-12
    assert orc.compare(acc_p.ravel(), acc_d.ravel())[0] <= 1e-12


def test_acc_extension_finite_difference(orc):
    """P2P acceleration = -grad phi (central differences of the oracle's own potential)."""
    rng = np.random.default_rng(11)
    src = np.concatenate([rng.uniform(-1, 1, (50, 3)), rng.uniform(-1, 1, (50, 1))], 1)
    x = np.array([[2.5, 0.3, -0.7, 0.0]])
    ops = oracle.OracleOps(orc, 2)
    _, acc, _ = ops.p2p(x, src)
    h = 1e-5
    for d in range(3):
        xp, xm = x.copy(), x.copy()
        xp[0, d] += h
        xm[0, d] -= h
        fd = -(ops.p2p(xp, src)[0][0] - ops.p2p(xm, src)[0][0]) / (2 * h)
        assert acc[0, d] == pytest.approx(fd, rel=1e-7, abs=1e-9)
    # L2P gradient: local polynomial -grad vs central differences
    ops6 = oracle.OracleOps(orc, 6)
    L = rng.uniform(-1, 1, ops6.n)
    c = np.array([0.1, -0.2, 0.3])
    pts = np.concatenate([c + 0.2 * rng.uniform(-1, 1, (5, 3)), np.zeros((5, 1))], 1)
    _, acc = ops6.l2p(L, c, pts)
    for d in range(3):
        pp, pm = pts.copy(), pts.copy()
        pp[:, d] += h
        pm[:, d] -= h
        fd = -(ops6.l2p(L, c, pp, False)[0] - ops6.l2p(L, c, pm, False)[0]) / (2 * h)
        assert np.allclose(acc[:, d], fd, rtol=1e-6, atol=1e-8)


def test_acc_extension_fmm_vs_direct(orc):
    """Oracle FMM acceleration against the long-double direct-sum gradient (p-convergent)."""
    bodies = orc.generate_reference_bodies(0, 3000, 21)
    errs = []
    for p in (4, 8):
        t = orc.build_tree(bodies, 64, p)
        orc.evaluate(t, 0.5, with_acc=True)
        _, acc_d = orc.direct_sum(t.positions(), t.charges())
        errs.append(orc.compare(t.acc().ravel(), acc_d.ravel())[0])
    assert errs[1] < errs[0] and errs[0] < 5e-2 and errs[1] < 5e-4


@pytest.mark.parametrize("case", [(1, 16384, 4, 64, 0.5), (3, 30000, 6, 64, 0.5),
                                  (5, 20000, 10, 64, 0.5), (4, 40000, 8, 128, 0.4)],
                         ids=["C1", "C3", "C5", "C4"])
def test_parallel_checker_is_bit_identical(orc, case):
    """orc_evaluate_par (OpenMP, used by the full-size GPU parity tests) reproduces the serial
    pipeline bit for bit: potentials, accelerations, multipoles, locals, counts; a leaf mask
    gives the same bits on the marked leaves."""
    cfg, n, p, n_crit, theta = case
    bodies = orc.generate_baseline_bodies(cfg, n, 1)
    ts = orc.build_tree(bodies, n_crit, p)
    rs = orc.evaluate(ts, theta, with_acc=True)
    tp = orc.build_tree(bodies, n_crit, p)
    rp = orc.evaluate_par(tp, theta, with_acc=True)
    assert rs == rp
    for a, b in ((ts.phi(), tp.phi()), (ts.acc(), tp.acc()), (ts.multipoles(), tp.multipoles()),
                 (ts.locals(), tp.locals())):
        assert np.array_equal(a, b)
    c = tp.cells()
    leaves = np.flatnonzero(c.child_count == 0)[::5]
    mask = np.zeros(tp.ncells, bool)
    mask[leaves] = True
    tm = orc.build_tree(bodies, n_crit, p)
    orc.evaluate_par(tm, theta, with_acc=True, leaf_mask=mask)
    sel = np.concatenate([np.arange(c.body_begin[k], c.body_end[k]) for k in leaves])
    assert np.array_equal(tm.phi()[sel], ts.phi()[sel])
    assert np.array_equal(tm.acc()[sel], ts.acc()[sel])


def test_lists_csr_canonical(orc):
    """CSR grouping of the FIFO lists: offsets = per-target counts, sources ascending, same
    multiset as the emitted pairs."""
    bodies = orc.generate_baseline_bodies(3, 20000, 2)
    t = orc.build_tree(bodies, 64, 6)
    m, p = orc.traverse(t, 0.5)
    mo, ms, po, ps = orc.lists_csr(t, 0.5)
    for pairs, off, src in ((m, mo, ms), (p, po, ps)):
        assert off[-1] == len(pairs)
        assert np.array_equal(np.diff(off), np.bincount(pairs[:, 0], minlength=t.ncells))
        tgt = np.repeat(np.arange(t.ncells, dtype=np.int64), np.diff(off))
        keys = (tgt << 32) | src.astype(np.int64)
        assert np.all(np.diff(keys) > 0)  # strictly ascending: no duplicate pairs
        ref = np.sort((pairs[:, 0].astype(np.int64) << 32) | pairs[:, 1].astype(np.int64))
        assert np.array_equal(keys, ref)


@pytest.mark.parametrize("cfg", [1, 2, 3, 4, 5])
def test_baseline_generator_matches_library(orc, cfg):
    """The oracle's BASELINE generator (used by the reference arm, which must not load the
    product library) is bit-identical to fmm_generate_bodies (host code, no GPU needed)."""
    import paper_1203_0889_b200 as fb
    a = orc.generate_baseline_bodies(cfg, 5000, 7)
    b = fb.generate_bodies(cfg, 5000, 7)
    assert np.array_equal(a, b)
