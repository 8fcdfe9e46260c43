"""ctypes front-end for the CPU oracle — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline / reference arm
may import this package. It never participates in the product path
(``paper_1203_0889_b200``), which fails loudly when its CUDA library is missing.

Two libraries:

* ``Oracle`` — ``_build/liboracle.so``, the C restatement in ``fmm_oracle.c`` (always built by
  ``make -C oracle``). It restates proj/src/{tree,multi_index,kernels,traversal,oracle,
  dataset}.cpp and adds the acceleration extension.
* ``Reference`` — ``_ref/libfmmref.so``, the UNMODIFIED reference sources compiled against the
  Eigen shim with ``ref_harness.cpp`` (built only where /root/reference exists; the prebuilt
  file travels to the GPU box).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_build", "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libfmmref.so")

_i32p = C.POINTER(C.c_int32)
_i64p = C.POINTER(C.c_int64)
_u64p = C.POINTER(C.c_uint64)
_dp = C.POINTER(C.c_double)

ERRORS = {
    1: "empty input",
    2: "n_crit must be >= 1",
    3: "expansion order must be >= 1",
    4: "level overflow",
    5: "singular M2L displacement",
    6: "singular evaluation point",
    7: "cannot split leaf pair",
    8: "theta must be in (0,1)",
    100: "allocation failure",
}


class OracleError(ValueError):
    pass


def build(quiet: bool = True) -> None:
    """Compile the oracle (and, when /root/reference is present, the reference harness)."""
    subprocess.run(["make", "-C", HERE, "-s"], check=True,
                   stdout=subprocess.DEVNULL if quiet else None)


def _ptr(a: np.ndarray, t):
    return a.ctypes.data_as(t)


def n_coef(p: int) -> int:
    return p * (p + 1) * (p + 2) // 6


class _Cell(C.Structure):
    _fields_ = [("level", C.c_int32), ("key", C.c_uint64), ("center", C.c_double * 3),
                ("radius", C.c_double), ("body_begin", C.c_int32), ("body_end", C.c_int32),
                ("child_begin", C.c_int32), ("child_count", C.c_int32), ("parent", C.c_int32)]


class _Tree(C.Structure):
    _fields_ = [("center", C.c_double * 3), ("half_side", C.c_double), ("n_crit", C.c_int),
                ("order", C.c_int), ("ncoef", C.c_int), ("ncells", C.c_int64),
                ("nbodies", C.c_int64), ("cells", C.POINTER(_Cell)), ("pos", _dp), ("q", _dp),
                ("perm", _i64p), ("multipole", _dp), ("local", _dp), ("phi", _dp), ("acc", _dp)]


CELL_DTYPE = np.dtype([("level", "<i4"), ("key", "<u8"), ("center", "<f8", (3,)),
                       ("radius", "<f8"), ("body_begin", "<i4"), ("body_end", "<i4"),
                       ("child_begin", "<i4"), ("child_count", "<i4"), ("parent", "<i4")],
                      align=True)


@dataclass
class Cells:
    """Structure-of-arrays view of a tree's cell array (reference Cell, tree.hpp:21-36)."""
    level: np.ndarray
    key: np.ndarray
    center: np.ndarray
    radius: np.ndarray
    body_begin: np.ndarray
    body_end: np.ndarray
    child_begin: np.ndarray
    child_count: np.ndarray
    parent: np.ndarray

    def __len__(self) -> int:
        return len(self.level)

    def equal(self, other: "Cells") -> bool:
        names = ["level", "key", "center", "radius", "body_begin", "body_end", "child_begin",
                 "child_count", "parent"]
        return all(np.array_equal(getattr(self, n), getattr(other, n)) for n in names)

    @classmethod
    def empty(cls, n: int) -> "Cells":
        return cls(np.zeros(n, np.int32), np.zeros(n, np.uint64), np.zeros((n, 3)), np.zeros(n),
                   np.zeros(n, np.int32), np.zeros(n, np.int32), np.zeros(n, np.int32),
                   np.zeros(n, np.int32), np.zeros(n, np.int32))


class OracleTree:
    """Owning wrapper of an ``orc_tree`` (restated build_tree, tree.cpp:52-119)."""

    def __init__(self, lib, tree: _Tree):
        self._lib = lib
        self._t = tree

    def __del__(self):
        try:
            self._lib.orc_tree_free(C.byref(self._t))
        except Exception:
            pass

    @property
    def ncells(self) -> int:
        return self._t.ncells

    @property
    def nbodies(self) -> int:
        return self._t.nbodies

    @property
    def order(self) -> int:
        return self._t.order

    @property
    def domain(self):
        return np.array(self._t.center[:]), self._t.half_side

    def cells(self) -> Cells:
        raw = np.ctypeslib.as_array(
            C.cast(self._t.cells, C.POINTER(C.c_uint8)), shape=(self.ncells * C.sizeof(_Cell),))
        arr = np.frombuffer(raw.tobytes(), dtype=CELL_DTYPE)
        return Cells(arr["level"].copy(), arr["key"].copy(), arr["center"].copy(),
                     arr["radius"].copy(), arr["body_begin"].copy(), arr["body_end"].copy(),
                     arr["child_begin"].copy(), arr["child_count"].copy(), arr["parent"].copy())

    def _arr(self, p, n, shape=None):
        a = np.ctypeslib.as_array(p, shape=(n,)).copy()
        return a.reshape(shape) if shape else a

    def perm(self) -> np.ndarray:
        return self._arr(self._t.perm, self.nbodies)

    def positions(self) -> np.ndarray:
        return self._arr(self._t.pos, 3 * self.nbodies, (self.nbodies, 3))

    def charges(self) -> np.ndarray:
        return self._arr(self._t.q, self.nbodies)

    def phi(self) -> np.ndarray:
        return self._arr(self._t.phi, self.nbodies)

    def acc(self) -> np.ndarray:
        return self._arr(self._t.acc, 3 * self.nbodies, (self.nbodies, 3))

    def multipoles(self) -> np.ndarray:
        nc = self._t.ncoef
        return self._arr(self._t.multipole, self.ncells * nc, (self.ncells, nc))

    def locals(self) -> np.ndarray:
        nc = self._t.ncoef
        return self._arr(self._t.local, self.ncells * nc, (self.ncells, nc))

    def set_multipoles(self, m: np.ndarray) -> None:
        nc = self._t.ncoef
        m = np.ascontiguousarray(m, dtype=np.float64).reshape(self.ncells * nc)
        C.memmove(self._t.multipole, m.ctypes.data, m.nbytes)


class Oracle:
    """The C restatement (fmm_oracle.c)."""

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            build()
        L = C.CDLL(path)
        self.lib = L
        L.orc_build_tree.argtypes = [C.c_int64, _dp, C.c_int, C.c_int, C.POINTER(_Tree)]
        L.orc_tree_free.argtypes = [C.POINTER(_Tree)]
        L.orc_traverse.argtypes = [C.POINTER(_Tree), C.c_double, C.c_int, _i64p,
                                   C.POINTER(_i32p), _i64p, C.POINTER(_i32p)]
        L.orc_evaluate.argtypes = [C.POINTER(_Tree), C.c_double, C.c_int, C.c_int, _u64p, _i64p,
                                   _i64p]
        L.orc_direct_sum.argtypes = [C.c_int64, _dp, _dp, _dp, _dp]
        L.orc_compare.argtypes = [C.c_int64, _dp, _dp, _dp, _dp, C.POINTER(C.c_int)]
        L.orc_generate_reference_bodies.argtypes = [C.c_int, C.c_int64, C.c_uint64, _dp]
        L.orc_morton_key.argtypes = [_dp, _dp, C.c_double, C.c_int, _u64p]
        L.orc_compute_bounds.argtypes = [C.c_int64, _dp, _dp, _dp]
        L.orc_free.argtypes = [C.c_void_p]
        L.orc_n_coef.restype = C.c_int64
        L.orc_n_coef.argtypes = [C.c_int64]
        L.orc_index_of.argtypes = [C.c_int, C.c_int, C.c_int]
        L.orc_apply_lists.argtypes = [C.POINTER(_Tree), C.c_void_p, C.c_int64, _i32p, C.c_int64, _i32p,
                                      C.c_int, _u64p]
        L.orc_evaluate_par.argtypes = [C.POINTER(_Tree), C.c_double, C.c_int, C.c_void_p, _u64p,
                                       _i64p, _i64p]
        L.orc_group_by_target.argtypes = [C.c_int64, C.c_int64, _i32p, _i64p, _i32p, C.c_int]
        L.orc_direct_sum_targets.argtypes = [C.c_int64, _dp, _dp, C.c_int64, _i64p, _dp, _dp]
        L.orc_generate_baseline_bodies.argtypes = [C.c_int, C.c_int64, C.c_uint64, _dp]

    # ---- tree / traversal / pipeline ------------------------------------------------
    def build_tree(self, xyzq: np.ndarray, n_crit: int, p: int) -> OracleTree:
        xyzq = np.ascontiguousarray(xyzq, dtype=np.float64).reshape(-1, 4)
        t = _Tree()
        rc = self.lib.orc_build_tree(len(xyzq), _ptr(xyzq, _dp), n_crit, p, C.byref(t))
        if rc:
            raise OracleError(ERRORS.get(rc, str(rc)))
        return OracleTree(self.lib, t)

    def traverse(self, tree: OracleTree, theta: float, mutual: bool = False):
        """Emitted (M2L pairs, P2P pairs) in FIFO order, each an (n, 2) int32 array."""
        nm, npp = C.c_int64(), C.c_int64()
        pm, pp = _i32p(), _i32p()
        rc = self.lib.orc_traverse(C.byref(tree._t), theta, int(mutual), C.byref(nm), C.byref(pm),
                                   C.byref(npp), C.byref(pp))
        if rc:
            raise OracleError(ERRORS.get(rc, str(rc)))
        m = np.ctypeslib.as_array(pm, shape=(2 * nm.value,)).reshape(-1, 2).copy() if nm.value else np.zeros((0, 2), np.int32)
        p = np.ctypeslib.as_array(pp, shape=(2 * npp.value,)).reshape(-1, 2).copy() if npp.value else np.zeros((0, 2), np.int32)
        self.lib.orc_free(C.cast(pm, C.c_void_p))
        self.lib.orc_free(C.cast(pp, C.c_void_p))
        return m, p

    def evaluate(self, tree: OracleTree, theta: float, mutual: bool = False,
                 with_acc: bool = True):
        """Serial pipeline (upward, traversal + kernels, downward); fills the tree in place.
        Returns (p2p_evals, n_m2l, n_p2p)."""
        ev, nm, npp = C.c_uint64(), C.c_int64(), C.c_int64()
        rc = self.lib.orc_evaluate(C.byref(tree._t), theta, int(mutual), int(with_acc),
                                   C.byref(ev), C.byref(nm), C.byref(npp))
        if rc:
            raise OracleError(ERRORS.get(rc, str(rc)))
        return ev.value, nm.value, npp.value

    def evaluate_par(self, tree: OracleTree, theta: float, with_acc: bool = True,
                     leaf_mask: np.ndarray | None = None):
        """Non-mutual pipeline on all host cores (OpenMP), bit-identical to ``evaluate``.
        leaf_mask (bool per cell) limits phi/acc to the marked leaves. Returns
        (p2p_evals, n_m2l, n_p2p)."""
        ev, nm, npp = C.c_uint64(), C.c_int64(), C.c_int64()
        mask = None
        if leaf_mask is not None:
            mask = np.ascontiguousarray(leaf_mask, dtype=np.uint8)
            assert len(mask) == tree.ncells
        rc = self.lib.orc_evaluate_par(C.byref(tree._t), theta, int(with_acc),
                                       mask.ctypes.data if mask is not None else None,
                                       C.byref(ev), C.byref(nm), C.byref(npp))
        if rc:
            raise OracleError(ERRORS.get(rc, str(rc)))
        return ev.value, nm.value, npp.value

    def apply_lists(self, tree: OracleTree, m2l: np.ndarray, p2p: np.ndarray, mutual: bool = False):
        """KernelVisitor over given lists (traversal.hpp:138-164): M2L into the locals, P2P (+ acc)
        into the body accumulators, in list order; no upward / downward pass. Returns evals."""
        m2l = np.ascontiguousarray(m2l, dtype=np.int32).reshape(-1, 2)
        p2p = np.ascontiguousarray(p2p, dtype=np.int32).reshape(-1, 2)
        ops = OracleOps(self, tree.order)
        ev = C.c_uint64()
        rc = self.lib.orc_apply_lists(C.byref(tree._t), C.cast(C.byref(ops.kt), C.c_void_p), len(m2l),
                                      _ptr(m2l, _i32p), len(p2p), _ptr(p2p, _i32p), int(mutual), C.byref(ev))
        del ops
        if rc:
            raise OracleError(ERRORS.get(rc, str(rc)))
        return ev.value

    def group_by_target(self, ncells: int, pairs: np.ndarray, sort_sources: bool = True):
        """(offsets[ncells+1], sources): CSR by target; sources ascending per target when
        sort_sources (the canonical multiset form, comparable with fmm_get_lists)."""
        pairs = np.ascontiguousarray(pairs, dtype=np.int32).reshape(-1, 2)
        off = np.zeros(ncells + 1, np.int64)
        src = np.zeros(max(len(pairs), 1), np.int32)
        rc = self.lib.orc_group_by_target(ncells, len(pairs), _ptr(pairs, _i32p), _ptr(off, _i64p),
                                          _ptr(src, _i32p), int(sort_sources))
        if rc:
            raise OracleError("bad target index")
        return off, src[:len(pairs)]

    def lists_csr(self, tree: OracleTree, theta: float, mutual: bool = False):
        """Traversal lists as canonical CSR: (m2l_off, m2l_src, p2p_off, p2p_src)."""
        m, p = self.traverse(tree, theta, mutual)
        mo, ms = self.group_by_target(tree.ncells, m)
        del m
        po, ps = self.group_by_target(tree.ncells, p)
        return mo, ms, po, ps

    def direct_sum_targets(self, pos: np.ndarray, q: np.ndarray, idx: np.ndarray):
        """Long-double direct sum (oracle.cpp:8-23 + acc) for the listed targets only."""
        pos = np.ascontiguousarray(pos, dtype=np.float64).reshape(-1, 3)
        q = np.ascontiguousarray(q, dtype=np.float64)
        idx = np.ascontiguousarray(idx, dtype=np.int64)
        phi = np.zeros(len(idx))
        acc = np.zeros((len(idx), 3))
        self.lib.orc_direct_sum_targets(len(q), _ptr(pos, _dp), _ptr(q, _dp), len(idx),
                                        _ptr(idx, _i64p), _ptr(phi, _dp), _ptr(acc, _dp))
        return phi, acc

    def generate_baseline_bodies(self, config: int, n: int, seed: int = 1) -> np.ndarray:
        """BASELINE.json config 1..5 bodies (AoS x, y, z, q), SURVEY.md section 8d."""
        out = np.zeros((n, 4))
        rc = self.lib.orc_generate_baseline_bodies(config, n, seed, _ptr(out, _dp))
        if rc:
            raise OracleError(ERRORS.get(rc, str(rc)))
        return out

    def direct_sum(self, pos: np.ndarray, q: np.ndarray, with_acc: bool = True):
        pos = np.ascontiguousarray(pos, dtype=np.float64).reshape(-1, 3)
        q = np.ascontiguousarray(q, dtype=np.float64)
        n = len(q)
        phi = np.zeros(n)
        acc = np.zeros((n, 3)) if with_acc else None
        self.lib.orc_direct_sum(n, _ptr(pos, _dp), _ptr(q, _dp), _ptr(phi, _dp),
                                _ptr(acc, _dp) if with_acc else None)
        return phi, acc

    def compare(self, a: np.ndarray, b: np.ndarray):
        a = np.ascontiguousarray(a, dtype=np.float64).ravel()
        b = np.ascontiguousarray(b, dtype=np.float64).ravel()
        if a.shape != b.shape:
            raise OracleError("length mismatch")
        l2, linf, ab = C.c_double(), C.c_double(), C.c_int()
        self.lib.orc_compare(len(a), _ptr(a, _dp), _ptr(b, _dp), C.byref(l2), C.byref(linf),
                             C.byref(ab))
        return l2.value, linf.value, bool(ab.value)

    def generate_reference_bodies(self, dist: int, n: int, seed: int) -> np.ndarray:
        out = np.zeros((n, 4))
        rc = self.lib.orc_generate_reference_bodies(dist, n, seed, _ptr(out, _dp))
        if rc:
            raise OracleError(ERRORS.get(rc, str(rc)))
        return out

    def morton_key(self, p, center, half_side: float, level: int) -> int:
        p = np.ascontiguousarray(p, dtype=np.float64)
        c = np.ascontiguousarray(center, dtype=np.float64)
        out = C.c_uint64()
        rc = self.lib.orc_morton_key(_ptr(p, _dp), _ptr(c, _dp), half_side, level, C.byref(out))
        if rc:
            raise OracleError(ERRORS.get(rc, str(rc)))
        return out.value

    def compute_bounds(self, xyzq: np.ndarray):
        xyzq = np.ascontiguousarray(xyzq, dtype=np.float64).reshape(-1, 4)
        c = np.zeros(3)
        h = C.c_double()
        rc = self.lib.orc_compute_bounds(len(xyzq), _ptr(xyzq, _dp), _ptr(c, _dp), C.byref(h))
        if rc:
            raise OracleError(ERRORS.get(rc, str(rc)))
        return c, h.value


class Reference:
    """The unmodified reference (oracle/_ref/libfmmref.so via ref_harness.cpp)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} not built (needs /root/reference; make -C oracle)")
        L = C.CDLL(path)
        self.lib = L
        L.ref_last_error.restype = C.c_char_p
        L.ref_build.restype = C.c_void_p
        L.ref_build.argtypes = [_dp, C.c_int64, C.c_int, C.c_int, _i64p]
        L.ref_free.argtypes = [C.c_void_p]
        L.ref_free_buf.argtypes = [C.c_void_p]
        L.ref_ncells.restype = C.c_int64
        L.ref_ncells.argtypes = [C.c_void_p]
        L.ref_domain.argtypes = [C.c_void_p, _dp, _dp]
        L.ref_cells.argtypes = [C.c_void_p, _i32p, _u64p, _dp, _dp, _i32p, _i32p, _i32p, _i32p,
                                _i32p]
        L.ref_traverse.argtypes = [C.c_void_p, C.c_double, C.c_int, C.c_int64, _i64p,
                                   C.POINTER(_i32p), _i64p, C.POINTER(_i32p)]
        L.ref_pipeline.argtypes = [C.c_void_p, C.c_double, C.c_int, C.c_int64, C.c_int, _dp]
        L.ref_step.argtypes = [_dp, C.c_int64, C.c_int, C.c_int, C.c_double, C.c_int64, C.c_int,
                               _dp, _dp]
        L.ref_potentials.argtypes = [C.c_void_p, _dp]
        L.ref_expansions.argtypes = [C.c_void_p, _dp, _dp]
        L.ref_counters.argtypes = [_u64p, _u64p, _u64p]
        L.ref_direct_sum.argtypes = [_dp, C.c_int64, _dp]
        L.ref_generate_bodies.argtypes = [C.c_int, C.c_int64, C.c_uint64, _dp]
        L.ref_run_once.argtypes = [C.c_int64, C.c_int, C.c_double, C.c_int, C.c_int, C.c_int,
                                   C.c_int, C.c_uint64, C.c_int64, _dp, _dp]
        L.ref_op_m2l.argtypes = [C.c_int, _dp, _dp, _dp]
        L.ref_op_laplace_derivatives.argtypes = [C.c_int, _dp, _dp]
        L.ref_op_p2m.argtypes = [C.c_int, C.c_int64, _dp, _dp, _dp]
        L.ref_op_m2m.argtypes = [C.c_int, _dp, _dp, _dp]
        L.ref_op_l2l.argtypes = [C.c_int, _dp, _dp, _dp]
        L.ref_op_l2p.argtypes = [C.c_int, _dp, _dp, C.c_int64, _dp, _dp]
        L.ref_op_p2p.argtypes = [C.c_int64, _dp, C.c_int64, _dp, _dp]
        L.ref_op_evaluate_multipole.argtypes = [C.c_int, _dp, _dp, _dp, _dp]

    def _check(self, rc):
        if rc:
            raise OracleError(self.lib.ref_last_error().decode())

    def build_tree(self, xyzq: np.ndarray, n_crit: int, p: int):
        xyzq = np.ascontiguousarray(xyzq, dtype=np.float64).reshape(-1, 4)
        perm = np.zeros(len(xyzq), np.int64)
        h = self.lib.ref_build(_ptr(xyzq, _dp), len(xyzq), n_crit, p, _ptr(perm, _i64p))
        if not h:
            raise OracleError(self.lib.ref_last_error().decode())
        return RefTree(self, h, perm, p)

    def step(self, xyzq, n_crit, p, theta, queue_threshold, threads, want_phi=False):
        xyzq = np.ascontiguousarray(xyzq, dtype=np.float64).reshape(-1, 4)
        times = np.zeros(4)
        phi = np.zeros(len(xyzq)) if want_phi else None
        self._check(self.lib.ref_step(_ptr(xyzq, _dp), len(xyzq), n_crit, p, theta,
                                      queue_threshold, threads, _ptr(times, _dp),
                                      _ptr(phi, _dp) if want_phi else None))
        return times, phi

    def run_once(self, n, p, theta=0.5, n_crit=64, threads=1, mutual=False, dist=0, seed=1,
                 queue_threshold=0, check=True):
        err = C.c_double()
        times = np.zeros(4)
        self._check(self.lib.ref_run_once(n, p, theta, n_crit, threads, int(mutual), dist, seed,
                                          queue_threshold, C.byref(err) if check else None,
                                          _ptr(times, _dp)))
        return (err.value if check else None), times

    def counters(self):
        a, b, c = C.c_uint64(), C.c_uint64(), C.c_uint64()
        self.lib.ref_counters(C.byref(a), C.byref(b), C.byref(c))
        return a.value, b.value, c.value

    def counters_reset(self):
        self.lib.ref_counters_reset()

    def direct_sum(self, xyzq):
        xyzq = np.ascontiguousarray(xyzq, dtype=np.float64).reshape(-1, 4)
        out = np.zeros(len(xyzq))
        self.lib.ref_direct_sum(_ptr(xyzq, _dp), len(xyzq), _ptr(out, _dp))
        return out

    def generate_bodies(self, dist: int, n: int, seed: int):
        out = np.zeros((n, 4))
        self._check(self.lib.ref_generate_bodies(dist, n, seed, _ptr(out, _dp)))
        return out

    # operator-level entry points
    def op_m2l(self, order, M, R):
        M = np.ascontiguousarray(M, dtype=np.float64)
        R = np.ascontiguousarray(R, dtype=np.float64)
        L = np.zeros(n_coef(order))
        self._check(self.lib.ref_op_m2l(order, _ptr(M, _dp), _ptr(R, _dp), _ptr(L, _dp)))
        return L

    def op_laplace_derivatives(self, max_degree, R):
        R = np.ascontiguousarray(R, dtype=np.float64)
        out = np.zeros(n_coef(max_degree + 1))
        self._check(self.lib.ref_op_laplace_derivatives(max_degree, _ptr(R, _dp), _ptr(out, _dp)))
        return out

    def op_p2m(self, order, xyzq, center):
        xyzq = np.ascontiguousarray(xyzq, dtype=np.float64).reshape(-1, 4)
        c = np.ascontiguousarray(center, dtype=np.float64)
        M = np.zeros(n_coef(order))
        self._check(self.lib.ref_op_p2m(order, len(xyzq), _ptr(xyzq, _dp), _ptr(c, _dp), _ptr(M, _dp)))
        return M

    def op_m2m(self, order, child, shift):
        child = np.ascontiguousarray(child, dtype=np.float64)
        s = np.ascontiguousarray(shift, dtype=np.float64)
        out = np.zeros(n_coef(order))
        self._check(self.lib.ref_op_m2m(order, _ptr(child, _dp), _ptr(s, _dp), _ptr(out, _dp)))
        return out

    def op_l2l(self, order, parent, shift):
        parent = np.ascontiguousarray(parent, dtype=np.float64)
        s = np.ascontiguousarray(shift, dtype=np.float64)
        out = np.zeros(n_coef(order))
        self._check(self.lib.ref_op_l2l(order, _ptr(parent, _dp), _ptr(s, _dp), _ptr(out, _dp)))
        return out

    def op_l2p(self, order, L, center, xyzq):
        L = np.ascontiguousarray(L, dtype=np.float64)
        c = np.ascontiguousarray(center, dtype=np.float64)
        xyzq = np.ascontiguousarray(xyzq, dtype=np.float64).reshape(-1, 4)
        phi = np.zeros(len(xyzq))
        self._check(self.lib.ref_op_l2p(order, _ptr(L, _dp), _ptr(c, _dp), len(xyzq),
                                        _ptr(xyzq, _dp), _ptr(phi, _dp)))
        return phi

    def op_p2p(self, txyzq, sxyzq):
        t = np.ascontiguousarray(txyzq, dtype=np.float64).reshape(-1, 4)
        s = np.ascontiguousarray(sxyzq, dtype=np.float64).reshape(-1, 4)
        phi = np.zeros(len(t))
        self._check(self.lib.ref_op_p2p(len(t), _ptr(t, _dp), len(s), _ptr(s, _dp), _ptr(phi, _dp)))
        return phi

    def op_evaluate_multipole(self, order, M, x, center):
        M = np.ascontiguousarray(M, dtype=np.float64)
        x = np.ascontiguousarray(x, dtype=np.float64)
        c = np.ascontiguousarray(center, dtype=np.float64)
        out = C.c_double()
        self._check(self.lib.ref_op_evaluate_multipole(order, _ptr(M, _dp), _ptr(x, _dp),
                                                       _ptr(c, _dp), C.byref(out)))
        return out.value


class RefTree:
    def __init__(self, ref: Reference, handle, perm, order):
        self._ref = ref
        self.h = C.c_void_p(handle)
        self.perm_ = perm
        self.order = order

    def __del__(self):
        try:
            self._ref.lib.ref_free(self.h)
        except Exception:
            pass

    @property
    def ncells(self) -> int:
        return self._ref.lib.ref_ncells(self.h)

    def perm(self):
        return self.perm_.copy()

    @property
    def domain(self):
        c = np.zeros(3)
        h = C.c_double()
        self._ref.lib.ref_domain(self.h, _ptr(c, _dp), C.byref(h))
        return c, h.value

    def cells(self) -> Cells:
        n = self.ncells
        c = Cells.empty(n)
        self._ref.lib.ref_cells(self.h, _ptr(c.level, _i32p), _ptr(c.key, _u64p),
                                _ptr(c.center, _dp), _ptr(c.radius, _dp),
                                _ptr(c.body_begin, _i32p), _ptr(c.body_end, _i32p),
                                _ptr(c.child_begin, _i32p), _ptr(c.child_count, _i32p),
                                _ptr(c.parent, _i32p))
        return c

    def traverse(self, theta: float, mutual: bool = False, queue_threshold: int = 1 << 30):
        nm, npp = C.c_int64(), C.c_int64()
        pm, pp = _i32p(), _i32p()
        self._ref._check(self._ref.lib.ref_traverse(self.h, theta, int(mutual), queue_threshold,
                                                    C.byref(nm), C.byref(pm), C.byref(npp),
                                                    C.byref(pp)))
        m = np.ctypeslib.as_array(pm, shape=(2 * nm.value,)).reshape(-1, 2).copy() if nm.value else np.zeros((0, 2), np.int32)
        p = np.ctypeslib.as_array(pp, shape=(2 * npp.value,)).reshape(-1, 2).copy() if npp.value else np.zeros((0, 2), np.int32)
        self._ref.lib.ref_free_buf(C.cast(pm, C.c_void_p))
        self._ref.lib.ref_free_buf(C.cast(pp, C.c_void_p))
        return m, p

    def pipeline(self, theta: float, mutual: bool = False, queue_threshold: int = 1 << 30,
                 threads: int = 0):
        times = np.zeros(3)
        self._ref._check(self._ref.lib.ref_pipeline(self.h, theta, int(mutual), queue_threshold,
                                                     threads, _ptr(times, _dp)))
        return times

    def potentials(self):
        out = np.zeros(len(self.perm_))
        self._ref.lib.ref_potentials(self.h, _ptr(out, _dp))
        return out

    def expansions(self):
        nc = n_coef(self.order)
        M = np.zeros((self.ncells, nc))
        L = np.zeros((self.ncells, nc))
        self._ref.lib.ref_expansions(self.h, _ptr(M, _dp), _ptr(L, _dp))
        return M, L


def reference_available() -> bool:
    return os.path.exists(REF_SO)


# ---- operator-level wrappers of the restatement (kernels.cpp) -------------------------
class _Tables(C.Structure):
    _fields_ = [("order", C.c_int), ("n", C.c_int), ("idx_max_degree", C.c_int),
                ("idx_size", C.c_int), ("_exps", C.c_void_p), ("_deg", C.c_void_p),
                ("_fact", C.c_void_p), ("_pi", C.c_void_p), ("_pa", C.c_void_p),
                ("n_m2l", C.c_int), ("_m", C.c_void_p), ("_l", C.c_void_p), ("_d", C.c_void_p),
                ("_wf", C.c_void_p), ("_wr", C.c_void_p), ("n_m2m", C.c_int), ("_ms", C.c_void_p),
                ("_msh", C.c_void_p), ("_md", C.c_void_p), ("n_l2l", C.c_int), ("_ls", C.c_void_p),
                ("_lsh", C.c_void_p), ("_ld", C.c_void_p), ("_lw", C.c_void_p), ("_ew", C.c_void_p)]


class OracleOps:
    """Batched single-instance calls into the C restatement's operators."""

    def __init__(self, orc: "Oracle", order: int):
        self.lib = orc.lib
        self.kt = _Tables()
        L = self.lib
        L.orc_tables_init.argtypes = [C.POINTER(_Tables), C.c_int]
        L.orc_tables_free.argtypes = [C.POINTER(_Tables)]
        rc = L.orc_tables_init(C.byref(self.kt), order)
        if rc:
            raise OracleError(ERRORS.get(rc, str(rc)))
        self.order = order
        self.n = self.kt.n
        kp = C.POINTER(_Tables)
        L.orc_p2m.argtypes = [kp, C.c_int64, _dp, _dp, _dp, _dp]
        L.orc_m2m.argtypes = [kp, _dp, _dp, _dp]
        L.orc_m2l.argtypes = [kp, _dp, _dp, _dp]
        L.orc_m2l_mutual.argtypes = [kp, _dp, _dp, _dp, _dp, _dp]
        L.orc_l2l.argtypes = [kp, _dp, _dp, _dp]
        L.orc_l2p.argtypes = [kp, _dp, _dp, C.c_int64, _dp, _dp, _dp]
        L.orc_p2p.restype = C.c_uint64
        L.orc_p2p.argtypes = [C.c_int64, _dp, _dp, _dp, _dp, C.c_int64, _dp, _dp, _dp, _dp, C.c_int, C.c_int]
        L.orc_evaluate_multipole.argtypes = [kp, _dp, _dp, _dp, _dp]

    def __del__(self):
        try:
            self.lib.orc_tables_free(C.byref(self.kt))
        except Exception:
            pass

    @staticmethod
    def _a(x, n=None):
        a = np.ascontiguousarray(x, dtype=np.float64)
        return a if n is None else a.reshape(n)

    def p2m(self, xyzq, center):
        b = self._a(xyzq).reshape(-1, 4)
        pos = np.ascontiguousarray(b[:, :3])
        q = np.ascontiguousarray(b[:, 3])
        M = np.zeros(self.n)
        self.lib.orc_p2m(C.byref(self.kt), len(b), _ptr(pos, _dp), _ptr(q, _dp), _ptr(self._a(center), _dp),
                         _ptr(M, _dp))
        return M

    def m2m(self, child, shift):
        out = np.zeros(self.n)
        self.lib.orc_m2m(C.byref(self.kt), _ptr(self._a(child), _dp), _ptr(self._a(shift), _dp), _ptr(out, _dp))
        return out

    def m2l(self, M, R):
        out = np.zeros(self.n)
        rc = self.lib.orc_m2l(C.byref(self.kt), _ptr(self._a(M), _dp), _ptr(self._a(R), _dp), _ptr(out, _dp))
        if rc:
            raise OracleError(ERRORS.get(rc, str(rc)))
        return out

    def m2l_mutual(self, Ms, Mt, R):
        """kernels.cpp:113-126 (orc_m2l_mutual): (target_l, source_l) from zero."""
        tl, sl = np.zeros(self.n), np.zeros(self.n)
        rc = self.lib.orc_m2l_mutual(C.byref(self.kt), _ptr(self._a(Ms), _dp), _ptr(self._a(Mt), _dp),
                                     _ptr(self._a(R), _dp), _ptr(tl, _dp), _ptr(sl, _dp))
        if rc:
            raise OracleError(ERRORS.get(rc, str(rc)))
        return tl, sl

    def p2p_mutual(self, txyzq, sxyzq):
        """kernels.cpp:167-180: distinct target and source spans, both updated."""
        t = self._a(txyzq).reshape(-1, 4)
        s_ = self._a(sxyzq).reshape(-1, 4)
        tp, tq = np.ascontiguousarray(t[:, :3]), np.ascontiguousarray(t[:, 3])
        sp, sq = np.ascontiguousarray(s_[:, :3]), np.ascontiguousarray(s_[:, 3])
        tphi, sphi = np.zeros(len(t)), np.zeros(len(s_))
        tacc, sacc = np.zeros((len(t), 3)), np.zeros((len(s_), 3))
        self.lib.orc_p2p(len(t), _ptr(tp, _dp), _ptr(tq, _dp), _ptr(tphi, _dp), _ptr(tacc, _dp), len(s_),
                         _ptr(sp, _dp), _ptr(sq, _dp), _ptr(sphi, _dp), _ptr(sacc, _dp), 0, 1)
        return (tphi, tacc), (sphi, sacc)

    def l2l(self, parent, shift):
        out = np.zeros(self.n)
        self.lib.orc_l2l(C.byref(self.kt), _ptr(self._a(parent), _dp), _ptr(self._a(shift), _dp), _ptr(out, _dp))
        return out

    def l2p(self, L, center, xyzq, with_acc=True):
        b = self._a(xyzq).reshape(-1, 4)
        pos = np.ascontiguousarray(b[:, :3])
        phi = np.zeros(len(b))
        acc = np.zeros((len(b), 3)) if with_acc else None
        self.lib.orc_l2p(C.byref(self.kt), _ptr(self._a(L), _dp), _ptr(self._a(center), _dp), len(b),
                         _ptr(pos, _dp), _ptr(phi, _dp), _ptr(acc, _dp) if with_acc else None)
        return phi, acc

    def p2p(self, txyzq, sxyzq=None, with_acc=True):
        t = self._a(txyzq).reshape(-1, 4)
        self_ = sxyzq is None
        s = t if self_ else self._a(sxyzq).reshape(-1, 4)
        tp, tq = np.ascontiguousarray(t[:, :3]), np.ascontiguousarray(t[:, 3])
        sp, sq = (tp, tq) if self_ else (np.ascontiguousarray(s[:, :3]), np.ascontiguousarray(s[:, 3]))
        phi = np.zeros(len(t))
        acc = np.zeros((len(t), 3)) if with_acc else None
        ev = self.lib.orc_p2p(len(t), _ptr(tp, _dp), _ptr(tq, _dp), _ptr(phi, _dp), _ptr(acc, _dp) if with_acc else None,
                              len(s), _ptr(sp, _dp), _ptr(sq, _dp), None, None, int(self_), 0)
        return phi, acc, ev

    def evaluate_multipole(self, M, x, center):
        out = C.c_double()
        rc = self.lib.orc_evaluate_multipole(C.byref(self.kt), _ptr(self._a(M), _dp), _ptr(self._a(x), _dp),
                                             _ptr(self._a(center), _dp), C.byref(out))
        if rc:
            raise OracleError(ERRORS.get(rc, str(rc)))
        return out.value
