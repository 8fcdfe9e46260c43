"""GPU parity: the sm_100a path (through the C-ABI) against the pinned CPU oracle and the
reference fixtures. Bars (BASELINE.json north_star): trees and lists bit-exact; potentials and
accelerations within rel-L2 1e-6 (FP64 mode) and 1e-4 (FP32-P2P mode)."""
import os

import numpy as np
import pytest

import oracle
from conftest import sorted_pairs

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(__file__), "golden")
CELL_KEYS = ["level", "key", "center", "radius", "body_begin", "body_end", "child_begin",
             "child_count", "parent"]
TOL = {"fp64": 1e-6, "fp32": 1e-4}


@pytest.fixture(scope="module")
def fx():
    return np.load(os.path.join(GOLD, "ref_cases.npz"))


def rel_l2(a, b):
    a = np.asarray(a, dtype=np.float64).ravel()
    b = np.asarray(b, dtype=np.float64).ravel()
    den = np.sqrt((b * b).sum())
    return np.sqrt(((a - b) ** 2).sum()) / (den if den > 0 else 1.0)


def run_gpu(fb, bodies, n_crit, p, theta, precision="fp64", with_acc=True):
    ctx = fb.Context(order=p, n_crit=n_crit, theta=theta, precision=precision, with_acc=with_acc)
    ctx.set_bodies(bodies)
    ctx.evaluate()
    return ctx


def oracle_run(orc, bodies, n_crit, p, theta):
    t = orc.build_tree(bodies, n_crit, p)
    orc.evaluate(t, theta, with_acc=True)
    return t


# ---------------------------------------------------------------- operators ----------
def test_operator_known_answers(fmmlib):
    fb = fmmlib
    M = fb.p2m(5, [np.array([[0.25, -0.5, 1.0, 2.0]])], [[0.25, -0.5, 1.0]])[0]
    assert M[0] == 2.0 and np.abs(M[1:]).max() == 0.0  # test_kernels.cpp:25-34
    off = np.array([0.1, 0.2, -0.3])
    M = fb.p2m(3, [np.array([[*off, 1.0], [*(-off), -1.0]])], [[0, 0, 0]])[0]
    assert abs(M[0]) < 1e-15 and np.allclose(M[[3, 2, 1]], 2 * off)  # :36-49
    Mm = np.zeros(fb.n_coef(3))
    Mm[0] = 5.0
    assert fb.m2l(3, Mm, [2.0, 0, 0])[0, 0] == pytest.approx(2.5)  # :108-115
    assert fb.m2l(1, [-1.5], [1.0, 2.0, -2.0])[0, 0] == pytest.approx(-0.5)  # :117-125
    with pytest.raises(fb.FMMError, match="singular M2L displacement"):
        fb.m2l(2, np.zeros(4), [0.0, 0.0, 0.0])
    M6 = np.zeros(fb.n_coef(6))
    M6[0] = 2.0
    assert fb.evaluate_multipole(6, M6, [1, 5, 1], [1, 1, 1])[0] == pytest.approx(0.5)  # :325-335
    assert fb.evaluate_multipole(6, np.zeros(56), [2, 3, 4], [1, 1, 1])[0] == 0.0
    with pytest.raises(fb.FMMError, match="singular evaluation point"):
        fb.evaluate_multipole(6, M6, [1, 1, 1], [1, 1, 1])
    for prec in ("fp64", "fp32"):
        phi, _ = fb.p2p(np.array([[0, 0, 0, 1.0], [1, 0, 0, 1.0]]), precision=prec)  # :285-297
        assert phi == pytest.approx([1.0, 1.0])
        phi, _ = fb.p2p(np.array([[0.5, 0.5, 0.5, 3.0]]), precision=prec)
        assert phi[0] == 0.0
        phi, _ = fb.p2p(np.array([[0, 0, 0, 1.0], [0, 0, 0, 2.0], [0, 0, 2, 4.0]]), precision=prec)
        assert phi == pytest.approx([2.0, 2.0, 1.5])  # :314-323
    L = np.zeros(fb.n_coef(4))
    L[0] = 2.5
    c = np.array([0.1, 0.2, 0.3])
    pts = np.array([[*(c + [0.05, 0, 0]), 0], [*(c - [0, 0.1, 0]), 0], [*c, 0]])
    phi, acc = fb.l2p(4, L, c, pts)
    assert phi == pytest.approx([2.5, 2.5, 2.5]) and np.abs(acc).max() == 0.0  # :249-269
    # M2M zero shift identity, monopole shift (test_kernels.cpp:65-88)
    rng = np.random.default_rng(3)
    Mr = rng.uniform(-1, 1, fb.n_coef(5))
    assert np.allclose(fb.m2m(5, Mr, [0, 0, 0])[0], Mr, atol=0)
    # L2L zero shift identity and constant invariance (:237-247)
    assert np.allclose(fb.l2l(4, Mr[:20], [0, 0, 0])[0], Mr[:20], atol=0)
    cst = np.zeros(20)
    cst[0] = 4.2
    sh = fb.l2l(4, cst, [0.3, -0.8, 0.5])[0]
    assert sh[0] == pytest.approx(4.2) and np.abs(sh[1:]).max() == 0.0


@pytest.mark.parametrize("p", [1, 2, 3, 4, 5, 6, 7, 8, 9, 10])
def test_operators_match_oracle(fmmlib, orc, p):
    fb = fmmlib
    ops = oracle.OracleOps(orc, p)
    n = ops.n
    rng = np.random.default_rng(100 + p)
    K = 16
    Ms = rng.uniform(-1, 1, (K, n))
    R = rng.uniform(1.5, 3.0, (K, 3)) * rng.choice([-1, 1], (K, 3))
    sh = rng.uniform(-0.5, 0.5, (K, 3))
    g_m2l = fb.m2l(p, Ms, R)
    g_m2m = fb.m2m(p, Ms, sh)
    g_l2l = fb.l2l(p, Ms, sh)
    for k in range(K):
        o = ops.m2l(Ms[k], R[k])
        assert rel_l2(g_m2l[k], o) < 1e-12, ("m2l", k)
        assert rel_l2(g_m2m[k], ops.m2m(Ms[k], sh[k])) < 1e-13, ("m2m", k)
        assert rel_l2(g_l2l[k], ops.l2l(Ms[k], sh[k])) < 1e-13, ("l2l", k)
    bodies = [np.concatenate([rng.uniform(-0.5, 0.5, (20, 3)), rng.uniform(-1, 1, (20, 1))], 1) for _ in range(4)]
    cen = rng.uniform(-0.1, 0.1, (4, 3))
    g = fb.p2m(p, bodies, cen)
    for k in range(4):
        assert rel_l2(g[k], ops.p2m(bodies[k], cen[k])) < 1e-13
    phi, acc = fb.l2p(p, Ms[0], cen[0], bodies[0])
    ophi, oacc = ops.l2p(Ms[0], cen[0], bodies[0])
    assert rel_l2(phi, ophi) < 1e-13 and rel_l2(acc, oacc) < 1e-13
    x = rng.uniform(2, 3, (K, 3))
    g = fb.evaluate_multipole(p, Ms, x, np.zeros((K, 3)))
    for k in range(K):
        assert g[k] == pytest.approx(ops.evaluate_multipole(Ms[k], x[k], [0, 0, 0]), rel=1e-12, abs=1e-14)


def test_mutual_operators_match_oracle(fmmlib, orc):
    """m2l_mutual (kernels.cpp:113-126) and mutual p2p (kernels.cpp:167-180) through the GPU
    operators (two target-owned directions) against the oracle's mutual kernels; the reference's
    test_kernels.cpp:187-200 check (m2l_mutual = two one-directional translations)."""
    fb = fmmlib
    rng = np.random.default_rng(11)
    for p in (3, 6, 8):
        ops = oracle.OracleOps(orc, p)
        Ms, Mt = rng.uniform(-1, 1, ops.n), rng.uniform(-1, 1, ops.n)
        R = np.array([2.2, -1.7, 0.9])
        tl, sl = fb.m2l_mutual(p, Ms, Mt, R)
        otl, osl = ops.m2l_mutual(Ms, Mt, R)
        assert rel_l2(tl[0], otl) < 1e-12 and rel_l2(sl[0], osl) < 1e-12, p
        with pytest.raises(fb.FMMError, match="singular M2L displacement"):
            fb.m2l_mutual(p, Ms, Mt, [0.0, 0.0, 0.0])
    t = np.concatenate([rng.uniform(-0.5, 0.5, (40, 3)), rng.uniform(-1, 1, (40, 1))], 1)
    s_ = np.concatenate([rng.uniform(0.6, 1.4, (30, 3)), rng.uniform(-1, 1, (30, 1))], 1)
    (gt, gs) = fb.p2p(t, s_, mutual=True)
    (ot, os_) = ops.p2p_mutual(t, s_)
    for g, o in ((gt, ot), (gs, os_)):
        assert rel_l2(g[0], o[0]) < 1e-13 and rel_l2(g[1], o[1]) < 1e-13


def test_laplace_derivatives_match_reference(fmmlib, ref):
    rng = np.random.default_rng(7)
    for md in (0, 3, 5, 9):
        r = rng.uniform(-2, 2, (8, 3)) + np.array([0, 0, 3.0])
        g = fmmlib.laplace_derivatives(md, r)
        for k in range(8):
            assert rel_l2(g[k], ref.op_laplace_derivatives(md, r[k])) < 1e-13


def test_bounds_morton_mac_bit_exact(fmmlib, orc):
    fb = fmmlib
    rng = np.random.default_rng(9)
    for n in (1, 7, 1000, 100_001):
        b = np.concatenate([rng.normal(size=(n, 3)) * 3 + 1, rng.uniform(-1, 1, (n, 1))], 1)
        c, h = fb.compute_bounds(b)
        oc, oh = orc.compute_bounds(b)
        assert np.array_equal(c, oc) and h == oh
    pts = rng.uniform(0, 1, (500, 3))
    for level in (0, 1, 2, 5, 21):
        g = fb.morton_key(pts, [0.5] * 3, 0.5, level)
        o = [orc.morton_key(p, [0.5] * 3, 0.5, level) for p in pts]
        assert np.array_equal(g, np.array(o, dtype=np.uint64))
    assert fb.morton_key([[0.6, 0.3, 0.8]], [0.5] * 3, 0.5, 2)[0] == 46
    with pytest.raises(fb.FMMError, match="level overflow"):
        fb.morton_key([[0.0, 0, 0]], [0.5] * 3, 0.5, 22)
    # MAC on the boundary: identical cells fail, point-like pass, formula case (test_traversal.cpp:83-102)
    assert not fb.mac([[0, 0, 0]], 1.0, [[0, 0, 0]], 1.0, 0.9)[0]
    assert fb.mac([[0, 0, 0]], 0.0, [[0, 0, 1e-3]], 0.0, 0.5)[0]
    assert fb.mac([[0, 0, 0]], 1.0, [[10, 0, 0]], 1.0, 0.5)[0]


# ---------------------------------------------------------- fixtures (reference) ------
def fixture_cases(fx):
    return sorted({k.split("/")[0] for k in fx.files})


@pytest.mark.parametrize("precision", ["fp64", "fp32"])
def test_reference_fixtures(fmmlib, fx, precision):
    """GPU tree + lists bit-exact with the unmodified reference; potentials within tolerance
    of the reference's serial pipeline; expansions within 1e-12 (FP64)."""
    for name in fixture_cases(fx):
        g = lambda k: fx[f"{name}/{k}"]  # noqa: E731
        n_crit, p, theta = g("params")
        ctx = run_gpu(fmmlib, g("bodies"), int(n_crit), int(p), float(theta), precision)
        cells = ctx.cells()
        for k in CELL_KEYS:
            assert np.array_equal(cells[k], g(k)), (name, k)
        assert np.array_equal(ctx.permutation(), g("perm")), name
        m, pp = ctx.pair_lists()
        assert np.array_equal(sorted_pairs(m), g("m2l")), name
        assert np.array_equal(sorted_pairs(pp), g("p2p")), name
        phi, _ = ctx.results("tree", with_acc=False)
        assert rel_l2(phi, g("phi")) <= TOL[precision], (name, rel_l2(phi, g("phi")))
        M, L = ctx.expansions()
        assert rel_l2(M, g("multipole")) < 1e-12, name
        if np.abs(g("local")).max() > 0:
            assert rel_l2(L, g("local")) < 1e-11, name


def symmetrised(pairs):
    """Mutual list -> both orientations (test_traversal.cpp:36-46)."""
    pairs = np.asarray(pairs).reshape(-1, 2)
    return np.concatenate([pairs, pairs[pairs[:, 0] != pairs[:, 1]][:, ::-1]])


@pytest.mark.parametrize("precision", ["fp64", "fp32"])
def test_reference_fixtures_mutual(fmmlib, fx, precision):
    """Mutual mode: the GPU's emitted lists are bit-exact with the reference's mutual traversal
    (each unordered pair once, same orientation); potentials within tolerance of the reference's
    mutual pipeline and of the GPU's own non-mutual run to rounding (the symmetrised lists are the
    non-mutual lists, executed by the same target-owned kernels in another summation order)."""
    for name in fixture_cases(fx):
        g = lambda k: fx[f"{name}/{k}"]  # noqa: E731
        n_crit, p, theta = g("params")
        ctx = fmmlib.Context(order=int(p), n_crit=int(n_crit), theta=float(theta), precision=precision,
                             mutual=True)
        ctx.set_bodies(g("bodies"))
        ctx.evaluate()
        m, pp = ctx.pair_lists()
        assert np.array_equal(sorted_pairs(m), g("m2l_mutual")), name
        assert np.array_equal(sorted_pairs(pp), g("p2p_mutual")), name
        info = ctx.tree_info()
        assert info.mutual == 1 and info.n_m2l == len(m) and info.n_p2p == len(pp)
        assert info.n_m2l_exec == len(g("m2l")) and info.n_p2p_exec == len(g("p2p"))
        phi_m, acc_m = ctx.results("tree")
        assert rel_l2(phi_m, g("phi_mutual")) <= TOL[precision], (name, rel_l2(phi_m, g("phi_mutual")))
        ctx.set_mutual(False)
        ctx.evaluate()
        m2, pp2 = ctx.pair_lists()
        assert np.array_equal(sorted_pairs(m2), g("m2l")) and np.array_equal(sorted_pairs(pp2), g("p2p"))
        phi, acc = ctx.results("tree")
        tol = 1e-13 if precision == "fp64" else 1e-6
        assert rel_l2(phi_m, phi) < tol and rel_l2(acc_m, acc) < 100 * tol, name
        ctx.close()


def test_mutual_pipeline_vs_oracle(fmmlib, orc):
    """Mutual mode at C3/C5 shapes against the oracle's mutual traversal and pipeline
    (m2l_mutual / mutual p2p), plus the reference API mirror's KernelVisitor(mutual=True)."""
    for gen, n, seed, n_crit, p in ((3, 30000, 2, 64, 6), (5, 20000, 3, 64, 8)):
        bodies = fmmlib.generate_bodies(gen, n, seed)
        t = orc.build_tree(bodies, n_crit, p)
        om, op = orc.traverse(t, 0.5, mutual=True)
        orc.evaluate(t, 0.5, mutual=True, with_acc=True)
        for precision in ("fp64", "fp32"):
            ctx = fmmlib.Context(order=p, n_crit=n_crit, theta=0.5, precision=precision, mutual=True)
            ctx.set_bodies(bodies)
            ctx.evaluate()
            m, pp = ctx.pair_lists()
            assert np.array_equal(sorted_pairs(m), sorted_pairs(om))
            assert np.array_equal(sorted_pairs(pp), sorted_pairs(op))
            phi, acc = ctx.results("tree")
            assert rel_l2(phi, t.phi()) <= TOL[precision], (gen, precision, rel_l2(phi, t.phi()))
            assert rel_l2(acc, t.acc()) <= TOL[precision], (gen, precision, rel_l2(acc, t.acc()))
            ctx.close()
    # reference API: dual_tree_traverse(tree, tree, cfg(mutual), KernelVisitor(mutual))
    bodies = fmmlib.generate_bodies(1, 8192, 5)
    tree = fmmlib.build_tree(bodies, 64, 5, precision="fp64")
    kt = fmmlib.KernelTables(5)
    fmmlib.upward_pass(tree, kt)
    cfg = fmmlib.TraversalConfig(theta=0.5, mutual=True)
    fmmlib.dual_tree_traverse(tree, tree, cfg, fmmlib.KernelVisitor(tree, tree, kt, mutual=True))
    fmmlib.downward_pass(tree, kt)
    t = orc.build_tree(bodies, 64, 5)
    orc.evaluate(t, 0.5, mutual=True, with_acc=False)
    assert rel_l2(fmmlib.potentials(tree), t.phi()) <= 1e-6
    with pytest.raises(fmmlib.FMMError):
        fmmlib.dual_tree_traverse(tree, tree, cfg, fmmlib.KernelVisitor(tree, tree, kt, mutual=False))


# ------------------------------------------------------------------ pipelines ---------
CASES = [  # (config or dist, n, seed, n_crit, p, theta)
    ("C1", 16384, 1, 64, 4, 0.5),
    ("C3", 30000, 2, 64, 6, 0.5),
    ("C5", 30000, 3, 64, 10, 0.5),
    ("C4", 40000, 4, 128, 8, 0.4),
]


@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_pipeline_vs_oracle(fmmlib, orc, case):
    cfg, n, seed, n_crit, p, theta = case
    bodies = fmmlib.generate_bodies(int(cfg[1]), n, seed)
    t = oracle_run(orc, bodies, n_crit, p, theta)
    ocells = t.cells()
    om, op = orc.traverse(t, theta)
    for precision in ("fp64", "fp32"):
        ctx = run_gpu(fmmlib, bodies, n_crit, p, theta, precision)
        cells = ctx.cells()
        for k in CELL_KEYS:
            assert np.array_equal(cells[k], getattr(ocells, k)), (cfg, k)
        assert np.array_equal(ctx.permutation(), t.perm())
        m, pp = ctx.pair_lists()
        assert np.array_equal(sorted_pairs(m), sorted_pairs(om))
        assert np.array_equal(sorted_pairs(pp), sorted_pairs(op))
        phi, acc = ctx.results("tree")
        e_phi, e_acc = rel_l2(phi, t.phi()), rel_l2(acc, t.acc())
        assert e_phi <= TOL[precision], (cfg, precision, e_phi)
        assert e_acc <= TOL[precision], (cfg, precision, e_acc)
        # input-order results are the tree-order results permuted back
        phi_in, acc_in = ctx.results("input")
        perm = ctx.permutation()
        assert np.array_equal(phi_in[perm], phi) and np.array_equal(acc_in[perm], acc)
        info = ctx.tree_info()
        nb = (ocells.body_end - ocells.body_begin).astype(np.int64)
        assert info.p2p_body_pairs == int((nb[op[:, 0]] * nb[op[:, 1]]).sum())


@pytest.mark.parametrize("precision", ["fp64", "fp32"])
def test_time_step_tree_reuse(fmmlib, orc, precision):
    """fmm_update_bodies + fmm_evaluate_reuse (time stepping on the kept tree): bodies moved
    inside their leaf cubes reuse the tree and lists, and the result is bit-identical to the
    same tree loaded and evaluated stage by stage (fmm_load_tree) and within FMM accuracy of a
    fresh build; a body leaving its leaf falls back to the full rebuild (bit-identical to a
    fresh context)."""
    fb = fmmlib
    b0 = fb.generate_bodies(3, 20000, 5)
    ctx = fb.Context(order=6, n_crit=64, theta=0.5, precision=precision)
    ctx.set_bodies(b0)
    ctx.evaluate()
    cells, perm = ctx.cells(), ctx.permutation()
    # move every body toward its leaf centre (stays inside the cube) and change the charges
    leaf = np.zeros(len(b0), np.int64)
    for c in np.nonzero(cells["child_count"] == 0)[0]:
        leaf[cells["body_begin"][c]:cells["body_end"][c]] = c
    b1 = b0.copy()
    ctr = cells["center"][leaf]
    b1[perm, :3] = ctr + 0.9 * (b0[perm, :3] - ctr)
    b1[:, 3] = b0[:, 3] * np.random.default_rng(1).uniform(0.5, 1.5, len(b0))
    ctx.update_bodies(b1)
    assert ctx.evaluate_reuse()
    phi, acc = ctx.results("input")
    ref = fb.Context(order=6, n_crit=64, theta=0.5, precision=precision)
    ref.set_bodies(b1)
    ref.load_tree(cells, perm)
    ref.traverse()
    ref.upward()
    ref.m2l()
    ref.p2p()
    ref.downward()
    rphi, racc = ref.results("input")
    assert np.array_equal(phi, rphi) and np.array_equal(acc, racc)
    fresh = fb.Context(order=6, n_crit=64, theta=0.5, precision=precision)
    fresh.set_bodies(b1)
    fresh.evaluate()
    fphi, facc = fresh.results("input")
    assert rel_l2(phi, fphi) < 1e-4 and rel_l2(acc, facc) < 1e-3
    # a body leaves its leaf: full rebuild
    b2 = b1.copy()
    b2[0, :3] += 0.5
    ctx.update_bodies(b2)
    assert not ctx.evaluate_reuse()
    fresh.set_bodies(b2)
    fresh.evaluate()
    assert np.array_equal(ctx.results("input")[0], fresh.results("input")[0])
    for x in (ctx, ref, fresh):
        x.close()


@pytest.mark.parametrize("p", [1, 2, 3, 5, 7, 9])
def test_pipeline_other_orders(fmmlib, orc, p):
    """The orders the BASELINE configs do not use (each M2L / expansion kernel is instantiated
    per order): FP64 pipeline against the oracle."""
    bodies = fmmlib.generate_bodies(3, 6000, 20 + p)
    t = oracle_run(orc, bodies, 32, p, 0.5)
    ctx = run_gpu(fmmlib, bodies, 32, p, 0.5, "fp64")
    phi, acc = ctx.results("tree")
    assert rel_l2(phi, t.phi()) <= 1e-6, (p, rel_l2(phi, t.phi()))
    assert rel_l2(acc, t.acc()) <= 1e-6, (p, rel_l2(acc, t.acc()))
    ctx.close()


@pytest.mark.parametrize("coop", [True, False], ids=["cooperative-build", "per-level-build"])
def test_tree_reuse_across_distributions(fmmlib, orc, coop, monkeypatch):
    """One context, successive body sets of growing depth: the partial-digit sort keyed on the
    previous depth must fall back to the full sort (and the level batches must continue) so that
    every tree and permutation stays bit-exact with the reference restatement. Both tree builders:
    the cooperative all-levels kernel and the per-level launches it falls back to
    (FMM_NO_COOP_BUILD, read when the context is created)."""
    if not coop:
        monkeypatch.setenv("FMM_NO_COOP_BUILD", "1")
    ctx = fmmlib.Context(order=4, n_crit=32, theta=0.5, precision="fp64")
    for gen, n, seed in ((1, 20000, 3), (3, 20000, 4), (5, 30000, 6), (1, 5000, 7), (3, 40000, 8)):
        bodies = fmmlib.generate_bodies(gen, n, seed)
        t = oracle_run(orc, bodies, 32, 4, 0.5)
        ocells = t.cells()
        ctx.set_bodies(bodies)
        ctx.evaluate()
        cells = ctx.cells()
        for k in CELL_KEYS:
            assert np.array_equal(cells[k], getattr(ocells, k)), (gen, n, k)
        assert np.array_equal(ctx.permutation(), t.perm()), (gen, n)
        phi, _ = ctx.results("tree")
        assert rel_l2(phi, t.phi()) < 1e-12, (gen, n)
    ctx.close()


@pytest.mark.parametrize("gen,n,p", [(2, 20000, 6), (4, 12000, 8), (5, 8000, 10)],
                         ids=["p6-register", "p8-staged-rows", "p10-flat-partition"])
def test_stage_isolated_m2l_and_p2p(fmmlib, orc, gen, n, p):
    """Inject the oracle's tree, lists and multipoles; the GPU M2L locals and P2P near field
    then match the oracle's per coefficient / per body. One case per production M2L kernel:
    k_m2l_reg (p <= 6), k_m2l_big2 (p = 7..9) and k_m2l_flat (p >= 10; the sphere-surface tree's
    short lists put several targets into one 32-pair chunk and cut targets at warp ranges)."""
    bodies = fmmlib.generate_bodies(gen, n, 5)
    theta = 0.5
    t = oracle_run(orc, bodies, 64, p, theta)
    c = t.cells()
    m, pp = orc.traverse(t, theta)
    ctx = fmmlib.Context(order=p, n_crit=64, theta=theta, precision="fp64")
    ctx.set_bodies(bodies)
    ctx.load_tree({k: getattr(c, k) for k in CELL_KEYS}, t.perm())
    ctx.load_lists(m, pp)
    ctx.load_multipoles(t.multipoles())
    ctx.reset_accumulators()
    ctx.m2l()
    _, L = ctx.expansions(multipole=False)
    # the oracle's locals include L2L; compare the M2L-only part via a locals-only run
    t2 = orc.build_tree(bodies, 64, p)
    t2.set_multipoles(t.multipoles())
    ops = oracle.OracleOps(orc, p)
    Lo = np.zeros_like(L)
    for tt, ss in m:
        Lo[tt] += ops.m2l(t.multipoles()[ss], c.center[ss] - c.center[tt])
    assert rel_l2(L, Lo) < 1e-12
    ctx.p2p()
    ctx.downward()
    phi, acc = ctx.results("tree")
    assert rel_l2(phi, t.phi()) < 1e-12 and rel_l2(acc, t.acc()) < 1e-12


@pytest.mark.parametrize("precision,tol,shape", [("fp64", 1e-13, -1), ("fp32", 1e-6, 0), ("fp32", 1e-6, 1)],
                         ids=["fp64", "fp32-wide", "fp32-narrow"])
def test_stage_isolated_p2p_kernel(fmmlib, orc, precision, tol, shape):
    """The production P2P kernels alone (k_p2p_fp64 / k_p2p_fp32_ws) on injected tree and lists
    against the oracle's P2P (kernels.cpp:181-192 + gradient) applied over the same list: the
    locals are zero, so the downward pass adds nothing. FP64 mode differs from the reference's
    arithmetic only by the fused r^2 and a <= 1-ulp rsqrt: agreement to ~1e-15."""
    bodies = fmmlib.generate_bodies(5, 30000, 8)
    t = orc.build_tree(bodies, 64, 4)
    c = t.cells()
    m, pp = orc.traverse(t, 0.5)
    orc.apply_lists(t, np.zeros((0, 2), np.int32), pp)
    ctx = fmmlib.Context(order=4, n_crit=64, theta=0.5, precision=precision)
    ctx.set_p2p_shape(shape)  # FP32: both CTA shapes of k_p2p_fp32_ws (the choice is automatic otherwise)
    ctx.set_bodies(bodies)
    ctx.load_tree({k: getattr(c, k) for k in CELL_KEYS}, t.perm())
    ctx.load_lists(m, pp)
    ctx.reset_accumulators()
    ctx.p2p()
    ctx.downward()
    phi, acc = ctx.results("tree")
    e_phi, e_acc = rel_l2(phi, t.phi()), rel_l2(acc, t.acc())
    assert e_phi < tol and e_acc < tol, (precision, e_phi, e_acc)


# ------------------------------------------------------------------ edge cases ---------
def test_edge_cases(fmmlib, orc):
    fb = fmmlib
    # single body: one root leaf, zero potential
    ctx = run_gpu(fb, np.array([[1.0, 2.0, 3.0, 1.0]]), 8, 3, 0.5)
    assert ctx.tree_info().ncells == 1
    assert ctx.results()[0][0] == 0.0
    # coincident bodies: 22-cell chain down to level 21, all pairs skipped
    b = np.zeros((9, 4))
    b[:, :3] = 0.25
    b[:, 3] = 1.0
    ctx = run_gpu(fb, b, 8, 2, 0.5)
    cells = ctx.cells()
    assert len(cells["level"]) == 22 and cells["level"].max() == 21
    assert np.abs(ctx.results()[0]).max() == 0.0
    # oversized level-21 leaf (> one 1024-body P2P tile) next to ordinary bodies
    rng = np.random.default_rng(1)
    heavy = np.zeros((1500, 4))
    heavy[:, :3] = [0.1, 0.2, 0.3]
    heavy[:, 3] = rng.uniform(0.5, 1.0, 1500)
    rest = np.concatenate([rng.uniform(-1, 1, (3000, 3)), rng.uniform(-1, 1, (3000, 1))], 1)
    bodies = np.concatenate([rest[:1000], heavy, rest[1000:]])
    t = oracle_run(orc, bodies, 64, 5, 0.5)
    for precision in ("fp64", "fp32"):
        ctx = run_gpu(fb, bodies, 64, 5, 0.5, precision)
        assert np.array_equal(ctx.cells()["key"], t.cells().key)
        phi, acc = ctx.results("tree")
        assert rel_l2(phi, t.phi()) <= TOL[precision]
        assert rel_l2(acc, t.acc()) <= TOL[precision]
    # errors carry the reference's messages
    with pytest.raises(fb.FMMError, match="empty input"):
        c = fb.Context(order=3)
        c.set_bodies(np.zeros((0, 4)))
    with pytest.raises(fb.FMMError, match="theta must be in"):
        fb.Context(order=3, theta=1.5)
    with pytest.raises(fb.FMMError, match="expansion order must be >= 1"):
        fb.Context(order=0)


def test_deterministic(fmmlib):
    b = fmmlib.generate_bodies(3, 50000, 11)
    a = run_gpu(fmmlib, b, 64, 6, 0.5, "fp32").results("tree")
    c = run_gpu(fmmlib, b, 64, 6, 0.5, "fp32").results("tree")
    assert np.array_equal(a[0], c[0]) and np.array_equal(a[1], c[1])


def test_reference_api_mirror(fmmlib, orc):
    """The reference call sequence (test_traversal.cpp:292-318) through the Python mirror,
    with a collecting visitor for the list-only traversal (acceptance.cpp:93-123)."""
    fb = fmmlib
    bodies = orc.generate_reference_bodies(0, 2048, 15)
    tree = fb.build_tree(bodies, 64, 6, precision="fp64")
    kt = fb.KernelTables(6)
    fb.upward_pass(tree, kt)
    cfg = fb.TraversalConfig(theta=0.5, queue_threshold=1 << 30)

    class Collect:
        def __init__(self):
            self.m, self.p = [], []

        def m2l_pair(self, t, s):
            self.m.append((t, s))

        def p2p_pair(self, t, s):
            self.p.append((t, s))

    col = Collect()
    fb.dual_tree_traverse(tree, tree, cfg, col)
    t = orc.build_tree(bodies, 64, 6)
    om, op = orc.traverse(t, 0.5)
    assert np.array_equal(sorted_pairs(col.m), sorted_pairs(om))
    assert np.array_equal(sorted_pairs(col.p), sorted_pairs(op))
    fb.dual_tree_traverse(tree, tree, cfg, fb.KernelVisitor(tree, tree, kt))
    fb.downward_pass(tree, kt)
    orc.evaluate(t, 0.5, with_acc=True)
    assert rel_l2(fb.potentials(tree), t.phi()) < 1e-12
    assert rel_l2(fb.accelerations(tree), t.acc()) < 1e-12


# --------------------------------------------------------------- full BASELINE size ----
def test_c2_full_size_lists_and_properties(fmmlib, orc):
    """BASELINE C2 (N = 1 048 576): tree and lists bit-exact against the oracle at full size;
    size-independent properties of the potentials: FP32 vs FP64 agreement, and the FMM against
    a direct sum on a random sample of targets (truncation-level error)."""
    n = 1 << 20
    bodies = fmmlib.generate_bodies(2, n, 1)
    t = orc.build_tree(bodies, 64, 6)
    om, op = orc.traverse(t, 0.5)
    c64 = run_gpu(fmmlib, bodies, 64, 6, 0.5, "fp64")
    cells = c64.cells()
    oc = t.cells()
    for k in CELL_KEYS:
        assert np.array_equal(cells[k], getattr(oc, k)), k
    assert np.array_equal(c64.permutation(), t.perm())
    m, pp = c64.pair_lists()
    assert len(m) == len(om) and len(pp) == len(op)
    assert np.array_equal(sorted_pairs(m), sorted_pairs(om))
    assert np.array_equal(sorted_pairs(pp), sorted_pairs(op))
    phi64, acc64 = c64.results("input")
    phi32, acc32 = run_gpu(fmmlib, bodies, 64, 6, 0.5, "fp32").results("input")
    assert rel_l2(phi32, phi64) < 1e-5 and rel_l2(acc32, acc64) < 1e-4
    rng = np.random.default_rng(0)
    idx = rng.choice(n, 256, replace=False)
    x, q = bodies[:, :3], bodies[:, 3]
    dphi = np.zeros(len(idx))
    for k, i in enumerate(idx):
        d = x[i] - x
        r = np.sqrt((d * d).sum(1))
        r[i] = np.inf
        dphi[k] = (q / r).sum()
    assert rel_l2(phi64[idx], dphi) < 1e-3


# ---------------------------------------------------------------- sharded (emulated) ----
class _DevBuf:
    def __init__(self, n):
        import torch
        self.t = torch.zeros(int(n), dtype=torch.float64, device="cuda")
        self.ptr = self.t.data_ptr()


@pytest.mark.parametrize("world,gen,n,p,n_crit,theta",
                         [(2, 3, 60000, 6, 64, 0.5), (3, 3, 60000, 6, 64, 0.5), (2, 4, 40000, 8, 128, 0.4),
                          (2, 5, 30000, 10, 64, 0.5)],
                         ids=["2-ranks-p6", "3-ranks-p6", "2-ranks-C4-shape-p8", "2-ranks-C5-shape-p10"])
def test_sharded_step_emulated(fmmlib, world, gen, n, p, n_crit, theta):
    """The multi-GPU data path with `world` ranks emulated sequentially on one GPU (no rank waits
    on another): per-rank partition, local upward, the all-gather as a concatenation of the
    equal-size chunks, shared ancestors, then M2L/P2P/downward; the union of the ranks' own body
    ranges reproduces the single-context step. Two steps: the first plans the partition from its
    full lists, the second reuses it (Morton boundaries) with a target-filtered traversal."""
    import torch
    fb = fmmlib
    bodies = fb.generate_bodies(gen, n, 21)
    for precision, tol in (("fp64", 1e-12), ("fp32", 1e-6)):
        full = run_gpu(fb, bodies, n_crit, p, theta, precision)
        phi_full, acc_full = full.results("tree")
        n_m2l_full = full.tree_info().n_m2l
        ctxs = []
        for r in range(world):
            ctx = fb.Context(order=p, n_crit=n_crit, theta=theta, precision=precision)
            ctx.set_bodies(bodies)
            ctx.set_partition(r, world)
            ctxs.append(ctx)
        bounds_seen = []
        for step in range(2):
            sends, infos = [], []
            for ctx in ctxs:
                ctx.build_tree()
                ctx.traverse()
                info = ctx.shard_info()
                send = _DevBuf(max(info.chunk_doubles, 1))
                ctx.upward_local(send.ptr)
                ctx.synchronize()
                sends.append(send)
                infos.append((info.body_begin, info.body_end, info.chunk_doubles))
            assert len({i[2] for i in infos}) == 1  # equal chunks on every rank
            assert infos[0][0] == 0 and infos[-1][1] == len(bodies)
            for a, b in zip(infos, infos[1:]):
                assert a[1] == b[0]
            bounds_seen.append([i[:2] for i in infos])
            if step == 1:  # filtered traversal: each rank holds only lists of targets meeting its range
                assert max(c.tree_info().n_m2l for c in ctxs) < n_m2l_full
            recv = _DevBuf(1)
            recv.t = torch.cat([s.t for s in sends])
            recv.ptr = recv.t.data_ptr()
            torch.cuda.synchronize()
            phi = np.zeros_like(phi_full)
            acc = np.zeros_like(acc_full)
            for r, ctx in enumerate(ctxs):
                ctx.upward_finish(recv.ptr)
                ctx.reset_accumulators()
                ctx.m2l()
                ctx.p2p()
                ctx.downward()
                p_r, a_r = ctx.results("tree")
                b0, b1, _ = infos[r]
                phi[b0:b1] = p_r[b0:b1]
                acc[b0:b1] = a_r[b0:b1]
            assert rel_l2(phi, phi_full) < tol, (precision, step, rel_l2(phi, phi_full))
            assert rel_l2(acc, acc_full) < tol, (precision, step, rel_l2(acc, acc_full))
        assert bounds_seen[0] == bounds_seen[1]  # the kept plan maps back onto the same leaves
        for ctx in ctxs:
            ctx.close()


@pytest.mark.gpu
def test_sharded_step_threads(fmmlib):
    """fmm.sharded_step (the bench's multi-GPU step) driven by two host threads on one GPU, one
    context per rank; the all-gather is a host-side rendezvous (device synchronised, chunks
    concatenated), so no kernel ever waits on another rank. Three steps: the first plans the
    partition, the later ones reuse it. The union of the ranks' ranges matches one context."""
    import threading

    import torch
    fb = fmmlib
    world = 2
    bodies = fb.generate_bodies(2, 50000, 5)
    full = run_gpu(fb, bodies, 64, 6, 0.5, "fp32")
    phi_full, acc_full = full.results("tree")
    barrier = threading.Barrier(world)
    sends = [None] * world
    out = [None] * world
    errors = []

    class Buf:
        def __init__(self, k):
            self.t = torch.zeros(int(k), dtype=torch.float64, device="cuda")
            self.ptr = self.t.data_ptr()

    def worker(rank):
        try:
            ctx = fb.Context(order=6, n_crit=64, theta=0.5, precision="fp32")

            def all_gather(recv, send):
                torch.cuda.synchronize()
                sends[rank] = send.t
                barrier.wait()
                recv.t.copy_(torch.cat(sends))
                torch.cuda.synchronize()
                barrier.wait()

            res = []
            for _ in range(3):
                ctx.set_bodies(bodies)
                info = fb.fmm.sharded_step(ctx, rank, world, all_gather, Buf)
                p, a = ctx.results("tree")
                res.append((int(info.body_begin), int(info.body_end), p, a))
            out[rank] = res
            ctx.close()
        except Exception as e:  # surfaced below
            errors.append(e)
            barrier.abort()

    ths = [threading.Thread(target=worker, args=(r,)) for r in range(world)]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    assert not errors, errors
    for step in range(3):
        phi = np.zeros_like(phi_full)
        acc = np.zeros_like(acc_full)
        for r in range(world):
            b0, b1, p, a = out[r][step]
            phi[b0:b1] = p[b0:b1]
            acc[b0:b1] = a[b0:b1]
        assert out[0][step][1] == out[1][step][0] and out[1][step][1] == len(bodies)
        assert rel_l2(phi, phi_full) < 1e-6, (step, rel_l2(phi, phi_full))
        assert rel_l2(acc, acc_full) < 1e-6, (step, rel_l2(acc, acc_full))
