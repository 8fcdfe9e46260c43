"""Host-side mirror of the reference's tree / traversal / kernel-operator API over the C-ABI.

Names, argument meaning and error behaviour follow /root/reference/proj/include/fmm:

* ``build_tree(bodies, n_crit, p) -> Tree``            tree.hpp:73   (bit-exact, on the GPU)
* ``upward_pass(tree, tables)``                        traversal.hpp:37
* ``dual_tree_traverse(targets, sources, cfg, visitor, drain=None)``  traversal.hpp:118-133
* ``downward_pass(tree, tables)``                      traversal.hpp:40
* ``potentials(tree)``                                 tree.hpp:76
* ``KernelTables(order)``, ``KernelVisitor``, ``TraversalConfig``, ``mac``, ``split_pair``,
  ``compute_bounds``, ``morton_key`` and the operators ``p2m m2m m2l l2l l2p p2p
  evaluate_multipole m2p_flip`` (kernels.hpp:69-103), batched over numpy arrays.

Errors raise ``FMMError`` (a ``ValueError``, like the reference's ``std::invalid_argument``)
whose message equals the reference's exception text. ``KernelVisitor`` passed to
``dual_tree_traverse`` runs the GPU M2L and P2P kernels over the whole emitted list; any other
visitor receives ``m2l_pair(t, s)`` / ``p2p_pair(t, s)`` for every emitted pair, so
collecting visitors from the reference's tests work unchanged.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Optional

import numpy as np

from . import _capi

_dp = C.POINTER(C.c_double)
_i32p = C.POINTER(C.c_int32)
_i64p = C.POINTER(C.c_int64)
_u64p = C.POINTER(C.c_uint64)


class FMMError(ValueError):
    def __init__(self, status: int, message: str):
        super().__init__(message)
        self.status = status


def _ptr(a: Optional[np.ndarray], t):
    return None if a is None else a.ctypes.data_as(t)


def _check(rc: int, ctx=None) -> None:
    if rc != _capi.OK:
        lib = _capi.load()
        msg = lib.fmm_last_error(ctx).decode() if ctx is not None else lib.fmm_last_error(None).decode()
        raise FMMError(rc, msg)


def n_coef(p: int) -> int:
    """multi_index.hpp:14"""
    return p * (p + 1) * (p + 2) // 6


def index_of(a: int, b: int, c: int) -> int:
    """multi_index.hpp:32-35"""
    n = a + b + c
    return n_coef(n) + a * (n + 1) - a * (a - 1) // 2 + b


def exponents(max_degree: int) -> np.ndarray:
    """MultiIndexSet order (multi_index.cpp:16-20): degree ascending, then (a,b,c) lexicographic."""
    out = []
    for n in range(max_degree + 1):
        for a in range(n + 1):
            for b in range(n - a + 1):
                out.append((a, b, n - a - b))
    return np.array(out, dtype=np.int32).reshape(-1, 3)


@dataclass
class TraversalConfig:
    """traversal.hpp:19-23 (queue_threshold only moves the drain point; the GPU traversal is
    level-synchronous and emits the same multiset for every Q)."""
    theta: float = 0.5
    queue_threshold: int = 64
    mutual: bool = False


class KernelTables:
    """kernels.hpp:24-54. The GPU kernels carry their term tables as compile-time constants;
    this object only validates and records the order."""

    def __init__(self, order: int):
        if order < 1:
            raise FMMError(_capi.ERR_ORDER, "expansion order must be >= 1")
        if order > _capi.FMM_MAX_ORDER:
            raise FMMError(_capi.ERR_UNSUPPORTED, "expansion order above FMM_MAX_ORDER (10)")
        self._order = order

    def order(self) -> int:
        return self._order

    def coef_count(self) -> int:
        return n_coef(self._order)


# --------------------------------------------------------------------------- context ----
class Context:
    """Owns one fmm_ctx (device-resident bodies, tree, lists, expansions, outputs)."""

    def __init__(self, order: int = 6, n_crit: int = 64, theta: float = 0.5, precision: str = "fp32",
                 device: int = 0, with_acc: bool = True, mutual: bool = False):
        self.lib = _capi.load()
        cfg = _capi.Config(order, n_crit, float(theta), int(mutual),
                           _capi.PREC_FP32_P2P if precision == "fp32" else _capi.PREC_FP64, device,
                           int(with_acc))
        h = C.c_void_p()
        _check(self.lib.fmm_create(C.byref(cfg), C.byref(h)))
        self.h = h
        self.cfg = cfg
        self.order = order
        self.ncoef = n_coef(order)
        self.n = 0

    def close(self) -> None:
        if getattr(self, "h", None):
            self.lib.fmm_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _c(self, rc: int) -> None:
        _check(rc, self.h)

    # inputs
    def set_bodies(self, xyzq: np.ndarray) -> None:
        xyzq = np.ascontiguousarray(xyzq, dtype=np.float64).reshape(-1, 4)
        self.n = len(xyzq)
        self._c(self.lib.fmm_set_bodies(self.h, _ptr(xyzq, _dp), len(xyzq)))

    def set_bodies_device(self, ptr: int, n: int) -> None:
        self.n = n
        self._c(self.lib.fmm_set_bodies_device(self.h, C.c_void_p(ptr), n))

    # stages
    def build_tree(self): self._c(self.lib.fmm_build_tree(self.h))
    def traverse(self): self._c(self.lib.fmm_traverse(self.h))
    def upward(self): self._c(self.lib.fmm_upward(self.h))
    def m2l(self): self._c(self.lib.fmm_m2l(self.h))
    def p2p(self): self._c(self.lib.fmm_p2p(self.h))
    def downward(self): self._c(self.lib.fmm_downward(self.h))
    def evaluate(self): self._c(self.lib.fmm_evaluate(self.h))

    def update_bodies(self, xyzq: np.ndarray) -> None:
        """New positions/charges of the same bodies (input order); keeps the tree and lists."""
        xyzq = np.ascontiguousarray(xyzq, dtype=np.float64).reshape(-1, 4)
        self.n = len(xyzq)
        self._c(self.lib.fmm_update_bodies(self.h, _ptr(xyzq, _dp), len(xyzq)))

    def evaluate_reuse(self) -> bool:
        """Time step on the kept tree when every body stayed in its leaf cube (returns True),
        else a full rebuild (False). See fmm_b200.h."""
        r = C.c_int(0)
        self._c(self.lib.fmm_evaluate_reuse(self.h, C.byref(r)))
        return bool(r.value)
    def synchronize(self): self._c(self.lib.fmm_synchronize(self.h))
    def reset_accumulators(self): self._c(self.lib.fmm_reset_accumulators(self.h))
    def set_overlap(self, on):
        """0 = serial stages, 1 = upward concurrent with the traversal (default), 2 = also M2L
        concurrent with P2P."""
        self._c(self.lib.fmm_set_overlap(self.h, int(on)))

    def set_mutual(self, on: bool):
        self._c(self.lib.fmm_set_mutual(self.h, int(on)))
        self.cfg.mutual = int(on)

    def set_traversal_debug(self, force_keys64: bool = False, initial_capacity: int = 0):
        """Test hook (fmm_set_traversal_debug): force the 64-bit-key ordered emission and/or a
        small initial buffer capacity so the overflow regrow path runs."""
        self._c(self.lib.fmm_set_traversal_debug(self.h, int(force_keys64), int(initial_capacity)))

    def set_p2p_shape(self, shape: int = -1):
        """Test / tuning hook (fmm_set_p2p_shape): 0 wide, 1 narrow FP32 P2P CTAs, -1 automatic."""
        self._c(self.lib.fmm_set_p2p_shape(self.h, int(shape)))

    def traversal_regrows(self) -> int:
        r = C.c_int(0)
        self._c(self.lib.fmm_get_traversal_regrows(self.h, C.byref(r)))
        return r.value

    # outputs
    def results(self, order: str = "tree", with_acc: bool = True):
        phi = np.zeros(self.n)
        acc = np.zeros((self.n, 3)) if with_acc else None
        self._c(self.lib.fmm_get_results(self.h, _ptr(phi, _dp), _ptr(acc, _dp),
                                         0 if order == "tree" else 1))
        return phi, acc

    def results_device(self):
        p, a = C.c_void_p(), C.c_void_p()
        self._c(self.lib.fmm_results_device(self.h, C.byref(p), C.byref(a)))
        return p.value, a.value

    def tree_info(self) -> _capi.TreeInfo:
        info = _capi.TreeInfo()
        self._c(self.lib.fmm_get_tree_info(self.h, C.byref(info)))
        return info

    def stage_times(self) -> _capi.StageTimes:
        t = _capi.StageTimes()
        self._c(self.lib.fmm_get_stage_times(self.h, C.byref(t)))
        return t

    def stage_trace(self):
        """Rows (task_id, worker_id, kind, start_ns, end_ns) of the last evaluate: the
        reference's trace CSV schema (scheduler.cpp:305-317) at GPU-stage granularity."""
        rows = (_capi.TraceRow * 16)()
        n = C.c_int(0)
        self._c(self.lib.fmm_get_stage_trace(self.h, rows, 16, C.byref(n)))
        return [(r.task_id, r.worker_id, r.kind.decode(), r.start_ns, r.end_ns) for r in rows[:n.value]]

    def cells(self) -> dict:
        nc = self.tree_info().ncells
        out = dict(level=np.zeros(nc, np.int32), key=np.zeros(nc, np.uint64),
                   center=np.zeros((nc, 3)), radius=np.zeros(nc),
                   body_begin=np.zeros(nc, np.int32), body_end=np.zeros(nc, np.int32),
                   child_begin=np.zeros(nc, np.int32), child_count=np.zeros(nc, np.int32),
                   parent=np.zeros(nc, np.int32))
        self._c(self.lib.fmm_get_cells(
            self.h, _ptr(out["level"], _i32p), _ptr(out["key"], _u64p), _ptr(out["center"], _dp),
            _ptr(out["radius"], _dp), _ptr(out["body_begin"], _i32p), _ptr(out["body_end"], _i32p),
            _ptr(out["child_begin"], _i32p), _ptr(out["child_count"], _i32p),
            _ptr(out["parent"], _i32p)))
        return out

    def permutation(self) -> np.ndarray:
        p = np.zeros(self.n, np.int64)
        self._c(self.lib.fmm_get_permutation(self.h, _ptr(p, _i64p)))
        return p

    def lists(self):
        """(m2l_offsets, m2l_sources, p2p_offsets, p2p_sources): CSR by target cell."""
        info = self.tree_info()
        mo = np.zeros(info.ncells + 1, np.int64)
        po = np.zeros(info.ncells + 1, np.int64)
        ms = np.zeros(max(info.n_m2l, 1), np.int32)
        ps = np.zeros(max(info.n_p2p, 1), np.int32)
        self._c(self.lib.fmm_get_lists(self.h, _ptr(mo, _i64p), _ptr(ms, _i32p), _ptr(po, _i64p),
                                       _ptr(ps, _i32p)))
        return mo, ms[:info.n_m2l], po, ps[:info.n_p2p]

    def pair_lists(self):
        """Emitted (target, source) pairs as (n, 2) arrays, grouped by target."""
        mo, ms, po, ps = self.lists()
        mt = np.repeat(np.arange(len(mo) - 1, dtype=np.int32), np.diff(mo))
        pt = np.repeat(np.arange(len(po) - 1, dtype=np.int32), np.diff(po))
        return np.stack([mt, ms], 1), np.stack([pt, ps], 1)

    def expansions(self, multipole: bool = True, local: bool = True):
        nc = self.tree_info().ncells
        M = np.zeros((nc, self.ncoef)) if multipole else None
        L = np.zeros((nc, self.ncoef)) if local else None
        self._c(self.lib.fmm_get_expansions(self.h, _ptr(M, _dp), _ptr(L, _dp)))
        return M, L

    # sharding with the NCCL exchange inside the library (comm.cu, fmm_b200.h)
    def comm_init(self, uid: bytes, rank: int, world: int) -> None:
        buf = C.create_string_buffer(bytes(uid), _capi.COMM_ID_BYTES)
        self._c(self.lib.fmm_comm_init(self.h, buf, rank, world))

    def set_allgather(self, fn) -> None:
        """Exchange override: fn(d_send, d_recv, count, stream) all-gathers `count` doubles per
        rank between device pointers (see fmm_set_allgather); None restores NCCL."""
        if fn is None:
            self._ag = None
            self._c(self.lib.fmm_set_allgather(self.h, None, None))
            return

        def tramp(d_send, d_recv, count, stream, user):
            try:
                fn(int(d_send or 0), int(d_recv or 0), int(count), int(stream or 0))
                return 0
            except Exception:  # reported as a CUDA-class error by the library
                import traceback
                traceback.print_exc()
                return 1

        self._ag = _capi.ALLGATHER_FN(tramp)  # keep the trampoline alive
        self._c(self.lib.fmm_set_allgather(self.h, C.cast(self._ag, C.c_void_p), None))

    def comm_destroy(self) -> None:
        self._c(self.lib.fmm_comm_destroy(self.h))

    def set_bodies_shard(self, share: np.ndarray, n_total: int) -> None:
        share = np.ascontiguousarray(share, dtype=np.float64).reshape(-1, 4)
        self._c(self.lib.fmm_set_bodies_shard(self.h, _ptr(share, _dp), len(share), int(n_total)))
        self.n = int(n_total)

    def set_bodies_shard_ptr(self, host_ptr: int, n_share: int, n_total: int) -> None:
        """Same from a raw host pointer (e.g. pinned memory)."""
        self._c(self.lib.fmm_set_bodies_shard(self.h, C.cast(host_ptr, _dp), int(n_share), int(n_total)))
        self.n = int(n_total)

    def evaluate_sharded(self) -> _capi.ShardInfo:
        info = _capi.ShardInfo()
        self._c(self.lib.fmm_evaluate_sharded(self.h, C.byref(info)))
        return info

    def owned_results(self, info: _capi.ShardInfo, with_acc: bool = True):
        """(phi, acc, input_index) of the own tree-order range [body_begin, body_end)."""
        k = int(info.body_end - info.body_begin)
        phi = np.zeros(k)
        acc = np.zeros((k, 3)) if with_acc else None
        idx = np.zeros(k, np.int64)
        self._c(self.lib.fmm_get_owned_results(self.h, _ptr(phi, _dp), _ptr(acc, _dp), _ptr(idx, _i64p)))
        return phi, acc, idx

    # sharding
    def set_partition(self, rank: int, world: int) -> None:
        self._c(self.lib.fmm_set_partition(self.h, rank, world))

    def shard_info(self) -> _capi.ShardInfo:
        info = _capi.ShardInfo()
        self._c(self.lib.fmm_get_shard_info(self.h, C.byref(info)))
        return info

    def upward_local(self, d_send: int) -> None:
        self._c(self.lib.fmm_upward_local(self.h, C.c_void_p(d_send)))

    def upward_finish(self, d_recv: int) -> None:
        self._c(self.lib.fmm_upward_finish(self.h, C.c_void_p(d_recv)))

    def set_stream(self, stream_handle: int) -> None:
        self._c(self.lib.fmm_set_stream(self.h, C.c_void_p(stream_handle)))

    # injection
    def load_tree(self, cells: dict, perm: np.ndarray) -> None:
        g = {k: np.ascontiguousarray(v) for k, v in cells.items()}
        perm = np.ascontiguousarray(perm, dtype=np.int64)
        self._c(self.lib.fmm_load_tree(
            self.h, len(g["level"]), _ptr(g["level"].astype(np.int32), _i32p),
            _ptr(g["key"].astype(np.uint64), _u64p), _ptr(g["center"].astype(np.float64), _dp),
            _ptr(g["radius"].astype(np.float64), _dp), _ptr(g["body_begin"].astype(np.int32), _i32p),
            _ptr(g["body_end"].astype(np.int32), _i32p), _ptr(g["child_begin"].astype(np.int32), _i32p),
            _ptr(g["child_count"].astype(np.int32), _i32p), _ptr(g["parent"].astype(np.int32), _i32p),
            _ptr(perm, _i64p)))

    def load_lists(self, m2l_pairs: np.ndarray, p2p_pairs: np.ndarray) -> None:
        m = np.ascontiguousarray(m2l_pairs, dtype=np.int32).reshape(-1, 2)
        p = np.ascontiguousarray(p2p_pairs, dtype=np.int32).reshape(-1, 2)
        self._c(self.lib.fmm_load_lists(self.h, len(m), _ptr(m, _i32p), len(p), _ptr(p, _i32p)))

    def load_multipoles(self, M: np.ndarray) -> None:
        M = np.ascontiguousarray(M, dtype=np.float64)
        self._c(self.lib.fmm_load_multipoles(self.h, _ptr(M, _dp)))


# ------------------------------------------------------------------ reference API ----
class Tree:
    """Device-resident tree (reference Tree, tree.hpp:41-59) produced by ``build_tree``."""

    def __init__(self, ctx: Context):
        self.ctx = ctx
        info = ctx.tree_info()
        self.n_crit = ctx.cfg.n_crit
        self.order = ctx.order
        self.ncells = info.ncells
        self.nbodies = info.nbodies
        self.domain = (np.array(info.center[:]), info.half_side)
        self._cells = None

    @property
    def cells(self) -> dict:
        if self._cells is None:
            self._cells = self.ctx.cells()
        return self._cells

    def permutation(self) -> np.ndarray:
        return self.ctx.permutation()


def build_tree(bodies: np.ndarray, n_crit: int, p: int, *, theta: float = 0.5,
               precision: str = "fp32", with_acc: bool = True, device: int = 0) -> Tree:
    """build_tree (tree.hpp:73): bodies is N x {x,y,z,q} (FP64). Runs on the GPU."""
    bodies = np.ascontiguousarray(bodies, dtype=np.float64).reshape(-1, 4)
    if len(bodies) == 0:
        raise FMMError(_capi.ERR_EMPTY_INPUT, "empty input")
    if n_crit < 1:
        raise FMMError(_capi.ERR_NCRIT, "n_crit must be >= 1")
    if p < 1:
        raise FMMError(_capi.ERR_ORDER, "expansion order must be >= 1")
    ctx = Context(order=p, n_crit=n_crit, theta=theta, precision=precision, device=device,
                  with_acc=with_acc)
    ctx.set_bodies(bodies)
    ctx.build_tree()
    return Tree(ctx)


def upward_pass(tree: Tree, tables: KernelTables) -> None:
    """traversal.cpp:36-50 (level-synchronous P2M + M2M on the GPU)."""
    tree.ctx.upward()


class KernelVisitor:
    """traversal.hpp:138-164: binds the emitted lists to the GPU M2L and P2P kernels."""

    def __init__(self, targets: Tree, sources: Tree, tables: KernelTables, mutual: bool = False):
        if targets is not sources:
            raise FMMError(_capi.ERR_UNSUPPORTED, "distinct target/source trees are not supported")
        # mutual (m2l_mutual / mutual p2p, kernels.cpp:113-126, :153-180): the GPU runs the
        # symmetrised lists with target-owned writes, which accumulates the same sums
        self.tree = targets
        self.mutual = bool(mutual)


def dual_tree_traverse(targets: Tree, sources: Tree, cfg: TraversalConfig, visit, drain=None):
    """traversal.hpp:118-133 on the GPU. With a ``KernelVisitor`` the M2L and P2P kernels run
    over the emitted lists; otherwise every emitted pair is delivered to the visitor."""
    if targets is not sources:
        raise FMMError(_capi.ERR_UNSUPPORTED, "distinct target/source trees are not supported")
    if not (0.0 < cfg.theta < 1.0):
        raise FMMError(_capi.ERR_THETA, "theta must be in (0,1)")
    ctx = targets.ctx
    if abs(ctx.cfg.theta - cfg.theta) > 0.0:
        ctx.cfg.theta = cfg.theta
        raise FMMError(_capi.ERR_STATE, "theta differs from the tree's context; rebuild with theta")
    if bool(ctx.cfg.mutual) != bool(cfg.mutual):
        ctx.set_mutual(cfg.mutual)
    ctx.traverse()
    if isinstance(visit, KernelVisitor):
        if visit.mutual != bool(cfg.mutual):
            raise FMMError(_capi.ERR_ARG, "KernelVisitor and TraversalConfig disagree on mutual")
        ctx.reset_accumulators()
        ctx.m2l()
        ctx.p2p()
        return
    m, p = ctx.pair_lists()
    for t, s in m:
        visit.m2l_pair(int(t), int(s))
    for t, s in p:
        visit.p2p_pair(int(t), int(s))


def downward_pass(tree: Tree, tables: KernelTables) -> None:
    """traversal.cpp:52-63 (L2L per level, L2P + near-field combine)."""
    tree.ctx.downward()


def potentials(tree: Tree) -> np.ndarray:
    """tree.cpp:121-126: potentials in tree (sorted) body order."""
    phi, _ = tree.ctx.results("tree", with_acc=False)
    return phi


def accelerations(tree: Tree) -> np.ndarray:
    """Extension: acceleration = -grad phi in tree body order."""
    _, acc = tree.ctx.results("tree", with_acc=True)
    return acc


def evaluate(bodies: np.ndarray, order: int = 6, n_crit: int = 64, theta: float = 0.5,
             precision: str = "fp32", with_acc: bool = True, device: int = 0):
    """One whole FMM step (run_once's stage sequence, engine.cpp:69-106) on the GPU.
    Returns (phi, acc) in INPUT body order and the stage times."""
    ctx = Context(order=order, n_crit=n_crit, theta=theta, precision=precision, device=device,
                  with_acc=with_acc)
    ctx.set_bodies(bodies)
    ctx.evaluate()
    phi, acc = ctx.results("input", with_acc=with_acc)
    t = ctx.stage_times()
    ctx.close()
    return phi, acc, t


def plan_partition(cells: dict, cell_cost: np.ndarray, world: int):
    """Host-only partition plan (fmm_plan_partition; no GPU needed): returns (bounds[world+1],
    owner[ncells]) — the contiguous body ranges of the ranks and each cell's owning rank (-1 when
    the cell straddles ranks)."""
    bb = np.ascontiguousarray(cells["body_begin"], dtype=np.int32)
    be = np.ascontiguousarray(cells["body_end"], dtype=np.int32)
    cc = np.ascontiguousarray(cells["child_count"], dtype=np.int32)
    cost = np.ascontiguousarray(cell_cost, dtype=np.float64)
    bounds = np.zeros(world + 1, np.int64)
    owner = np.zeros(len(bb), np.int32)
    _check(_capi.load().fmm_plan_partition(len(bb), _ptr(bb, _i32p), _ptr(be, _i32p), _ptr(cc, _i32p),
                                           _ptr(cost, _dp), world, _ptr(bounds, _i64p), _ptr(owner, _i32p)))
    return bounds, owner


def comm_unique_id() -> bytes:
    """ncclGetUniqueId through the library (rank 0; ship the bytes to the other ranks)."""
    buf = C.create_string_buffer(_capi.COMM_ID_BYTES)
    _check(_lib().fmm_comm_unique_id(buf))
    return buf.raw


def sharded_step(ctx: "Context", rank: int, world: int, all_gather, alloc):
    """One sharded FMM step on a context whose bodies are set (see fmm_b200.h):
    build, traverse (+ partition), local upward, all-gather of the owned multipoles, shared
    ancestors, M2L, P2P, downward. ``alloc(n)`` returns a device buffer object with ``.ptr``;
    ``all_gather(recv, send)`` gathers the equal-size chunks of every rank (NCCL in production)."""
    ctx.set_partition(rank, world)
    ctx.build_tree()
    ctx.traverse()
    info = ctx.shard_info()
    send = alloc(max(info.chunk_doubles, 1))
    recv = alloc(max(info.chunk_doubles, 1) * world)
    ctx.upward_local(send.ptr)
    all_gather(recv, send)
    ctx.upward_finish(recv.ptr)
    ctx.reset_accumulators()
    ctx.m2l()
    ctx.p2p()
    ctx.downward()
    return info


# ------------------------------------------------------------------ operators --------
def _lib():
    return _capi.load()


def compute_bounds(xyzq: np.ndarray):
    """tree.cpp:10-23 on the device. Returns (center[3], half_side)."""
    xyzq = np.ascontiguousarray(xyzq, dtype=np.float64).reshape(-1, 4)
    c = np.zeros(3)
    h = C.c_double()
    _check(_lib().fmm_op_compute_bounds(_ptr(xyzq, _dp), len(xyzq), _ptr(c, _dp), C.byref(h)))
    return c, h.value


def morton_key(positions: np.ndarray, center, half_side: float, level: int) -> np.ndarray:
    """tree.cpp:25-39 (floor-based, tests-only in the reference)."""
    p = np.ascontiguousarray(positions, dtype=np.float64).reshape(-1, 3)
    c = np.ascontiguousarray(center, dtype=np.float64)
    out = np.zeros(len(p), np.uint64)
    _check(_lib().fmm_op_morton_key(len(p), _ptr(p, _dp), _ptr(c, _dp), float(half_side), level,
                                    _ptr(out, _u64p)))
    return out


def mac(tcenter, tradius, scenter, sradius, theta: float) -> np.ndarray:
    """traversal.cpp:8-13, bit-exact FP64 on the device; vectorised over pairs."""
    tc = np.ascontiguousarray(tcenter, dtype=np.float64).reshape(-1, 3)
    sc = np.ascontiguousarray(scenter, dtype=np.float64).reshape(-1, 3)
    tr = np.ascontiguousarray(np.broadcast_to(tradius, (len(tc),)), dtype=np.float64)
    sr = np.ascontiguousarray(np.broadcast_to(sradius, (len(sc),)), dtype=np.float64)
    out = np.zeros(len(tc), np.int32)
    _check(_lib().fmm_op_mac(len(tc), _ptr(tc, _dp), _ptr(tr, _dp), _ptr(sc, _dp), _ptr(sr, _dp),
                             float(theta), _ptr(out, _i32p)))
    return out.astype(bool)


def split_pair(target: int, source: int, cells: dict):
    """traversal.cpp:15-34 (public API rule: larger radius, target on tie)."""
    tl = cells["child_count"][target] == 0
    sl = cells["child_count"][source] == 0
    if tl and sl:
        raise FMMError(_capi.ERR_CANNOT_SPLIT, "cannot split leaf pair")
    split_t = (not tl) and (sl or cells["radius"][target] >= cells["radius"][source])
    if split_t:
        b = int(cells["child_begin"][target])
        return [(b + i, source) for i in range(int(cells["child_count"][target]))]
    b = int(cells["child_begin"][source])
    return [(target, b + i) for i in range(int(cells["child_count"][source]))]


def _batch(a, n):
    a = np.ascontiguousarray(a, dtype=np.float64)
    return a.reshape(-1, n)


def p2m(order: int, bodies_list, centers) -> np.ndarray:
    """kernels.cpp:78-86 over a batch: bodies_list is a list of (n_k x 4) arrays."""
    offs = np.zeros(len(bodies_list) + 1, np.int32)
    offs[1:] = np.cumsum([len(b) for b in bodies_list])
    xyzq = np.ascontiguousarray(np.concatenate([np.reshape(b, (-1, 4)) for b in bodies_list]) if
                                offs[-1] else np.zeros((1, 4)), dtype=np.float64)
    c = _batch(centers, 3)
    M = np.zeros((len(bodies_list), n_coef(order)))
    _check(_lib().fmm_op_p2m(order, len(bodies_list), _ptr(offs, _i32p), _ptr(xyzq, _dp), _ptr(c, _dp),
                             _ptr(M, _dp)))
    return M


def m2m(order: int, child_m, shifts, parent_m=None) -> np.ndarray:
    """kernels.cpp:88-96 (accumulates into parent_m)."""
    cm = _batch(child_m, n_coef(order))
    s = _batch(shifts, 3)
    out = np.zeros_like(cm) if parent_m is None else np.array(_batch(parent_m, n_coef(order)))
    _check(_lib().fmm_op_m2m(order, len(cm), _ptr(cm, _dp), _ptr(s, _dp), _ptr(out, _dp)))
    return out


def m2l(order: int, source_m, disp, target_l=None) -> np.ndarray:
    """kernels.cpp:98-111 (accumulates; raises 'singular M2L displacement' on |R| = 0)."""
    sm = _batch(source_m, n_coef(order))
    r = _batch(disp, 3)
    out = np.zeros_like(sm) if target_l is None else np.array(_batch(target_l, n_coef(order)))
    _check(_lib().fmm_op_m2l(order, len(sm), _ptr(sm, _dp), _ptr(r, _dp), _ptr(out, _dp)))
    return out


def m2l_mutual(order: int, source_m, target_m, disp, target_l=None, source_l=None):
    """kernels.cpp:113-126: target_l += M2L(source_m, R) and source_l += M2L(target_m, -R), with
    R = source centre - target centre (the reference's w_rev terms are the reversed translation).
    Returns (target_l, source_l); raises 'singular M2L displacement' on |R| = 0."""
    r = _batch(disp, 3)
    return m2l(order, source_m, r, target_l), m2l(order, target_m, -r, source_l)


def l2l(order: int, parent_l, shifts, child_l=None) -> np.ndarray:
    """kernels.cpp:128-136 (accumulates into child_l)."""
    pl = _batch(parent_l, n_coef(order))
    s = _batch(shifts, 3)
    out = np.zeros_like(pl) if child_l is None else np.array(_batch(child_l, n_coef(order)))
    _check(_lib().fmm_op_l2l(order, len(pl), _ptr(pl, _dp), _ptr(s, _dp), _ptr(out, _dp)))
    return out


def l2p(order: int, L, center, bodies, with_acc: bool = True):
    """kernels.cpp:138-148 for one local expansion applied to a body array; returns
    (phi, acc) with acc = -grad (extension)."""
    Lb = _batch(L, n_coef(order))[:1]
    c = _batch(center, 3)[:1]
    b = np.ascontiguousarray(bodies, dtype=np.float64).reshape(-1, 4)
    offs = np.array([0, len(b)], np.int32)
    phi = np.zeros(len(b))
    acc = np.zeros((len(b), 3)) if with_acc else None
    _check(_lib().fmm_op_l2p(order, 1, _ptr(offs, _i32p), _ptr(Lb, _dp), _ptr(c, _dp), _ptr(b, _dp),
                             _ptr(phi, _dp), _ptr(acc, _dp)))
    return phi, acc


def p2p(targets, sources=None, precision: str = "fp64", with_acc: bool = True, mutual: bool = False):
    """kernels.cpp:150-195 (sources=None means the self interaction). Returns (phi, acc) of the
    targets; with ``mutual`` (kernels.cpp:153-180) and distinct sources, returns
    ((phi_t, acc_t), (phi_s, acc_s)): both spans updated, each pair evaluated for both sides
    (the GPU computes the two target-owned directions; the sums equal the mutual kernel's up
    to rounding). A mutual self interaction equals the non-mutual one (test_kernels.cpp:299)."""
    if mutual and sources is not None:
        return (p2p(targets, sources, precision, with_acc),
                p2p(sources, targets, precision, with_acc))
    t = np.ascontiguousarray(targets, dtype=np.float64).reshape(-1, 4)
    if sources is None:
        b = t
        rng = np.array([[0, len(t), 0, len(t)]], np.int32)
    else:
        s = np.ascontiguousarray(sources, dtype=np.float64).reshape(-1, 4)
        b = np.ascontiguousarray(np.concatenate([t, s]))
        rng = np.array([[0, len(t), len(t), len(t) + len(s)]], np.int32)
    phi = np.zeros(len(b))
    acc = np.zeros((len(b), 3)) if with_acc else None
    _check(_lib().fmm_op_p2p(1, _ptr(rng, _i32p), _ptr(b, _dp),
                             _capi.PREC_FP64 if precision == "fp64" else _capi.PREC_FP32_P2P,
                             _ptr(phi, _dp), _ptr(acc, _dp)))
    return phi[:len(t)], (acc[:len(t)] if with_acc else None)


def evaluate_multipole(order: int, M, x, center) -> np.ndarray:
    """kernels.cpp:197-208 (raises 'singular evaluation point')."""
    Mb = _batch(M, n_coef(order))
    xb = _batch(x, 3)
    cb = _batch(center, 3)
    out = np.zeros(len(Mb))
    _check(_lib().fmm_op_evaluate_multipole(order, len(Mb), _ptr(Mb, _dp), _ptr(xb, _dp), _ptr(cb, _dp),
                                            _ptr(out, _dp)))
    return out


def laplace_derivatives(max_degree: int, r) -> np.ndarray:
    """multi_index.cpp:59-85: D_g = (1/g!) d^g (1/|r|) for |g| <= max_degree."""
    rb = _batch(r, 3)
    out = np.zeros((len(rb), n_coef(max_degree + 1)))
    _check(_lib().fmm_op_laplace_derivatives(max_degree, len(rb), _ptr(rb, _dp), _ptr(out, _dp)))
    return out


def m2p_flip(order: int, M) -> np.ndarray:
    """kernels.cpp:210-216: negate odd-degree coefficients (host-side; an involution)."""
    e = exponents(order - 1)
    odd = (e.sum(1) % 2) == 1
    out = np.array(M, dtype=np.float64, copy=True)
    out[..., odd] = -out[..., odd]
    return out


def generate_bodies(config: int, n: int, seed: int = 1) -> np.ndarray:
    """BASELINE.json synthetic inputs: config 1..5 -> N x {x,y,z,q}."""
    out = np.zeros((n, 4))
    _check(_lib().fmm_generate_bodies(config, n, seed, _ptr(out, _dp)))
    return out
