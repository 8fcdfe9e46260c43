/* fmm_b200.h — C-ABI of the B200-native FMM hot path.
 *
 * Drop-in boundary for the reference's tree / traversal / kernel-operator API
 * (/root/reference/proj/include/fmm/{tree,traversal,kernels}.hpp). Plain pointers and sizes
 * only; device memory is owned by the context. Every entry point returns an fmm_status;
 * fmm_last_error() holds the message, whose text equals the reference's exception text where
 * one exists. Contexts are not thread-safe: one host thread per context,
 * mirroring the reference's master-thread-only rule (scheduler.cpp:48-52).
 *
 * Stage entry points are stream-ordered on the context's stream. The whole step is
 * fmm_evaluate (= run_once's stage sequence, engine.cpp:69-106, without the generator).
 */
#ifndef FMM_B200_H
#define FMM_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct fmm_ctx fmm_ctx;

/* Status codes; 1..8 map 1:1 onto the reference's std::invalid_argument texts. */
typedef enum {
  FMM_OK = 0,
  FMM_ERR_EMPTY_INPUT = 1,       /* "empty input"                   tree.cpp:11, :53 */
  FMM_ERR_NCRIT = 2,             /* "n_crit must be >= 1"           tree.cpp:54 */
  FMM_ERR_ORDER = 3,             /* "expansion order must be >= 1"  tree.cpp:55, kernels.cpp:26 */
  FMM_ERR_LEVEL_OVERFLOW = 4,    /* "level overflow"                tree.cpp:26 */
  FMM_ERR_SINGULAR_M2L = 5,      /* "singular M2L displacement"     kernels.cpp:101, :116 */
  FMM_ERR_SINGULAR_EVAL = 6,     /* "singular evaluation point"     kernels.cpp:200 */
  FMM_ERR_CANNOT_SPLIT = 7,      /* "cannot split leaf pair"        traversal.cpp:19 */
  FMM_ERR_THETA = 8,             /* "theta must be in (0,1)"        engine.cpp:63 */
  FMM_ERR_UNSUPPORTED = 20,      /* order > FMM_MAX_ORDER, mutual + sharded, ... */
  FMM_ERR_ARG = 21,              /* null pointer / bad size */
  FMM_ERR_STATE = 22,            /* stage called before its inputs exist */
  FMM_ERR_CUDA = 30,             /* CUDA runtime error (message has the detail) */
  FMM_ERR_NO_DEVICE = 31,        /* no CUDA device: there is no CPU fallback */
  FMM_ERR_OOM = 32
} fmm_status;

typedef enum {
  FMM_PREC_FP64 = 0,      /* every stage in FP64 (parity mode) */
  FMM_PREC_FP32_P2P = 1   /* P2P in FP32 with FP64 per-tile folding; expansions FP64 */
} fmm_precision;

#define FMM_MAX_ORDER 10  /* supported expansion orders p = 1..10 (n_coef <= 220) */
#define FMM_MAX_LEVEL 21  /* kMaxTreeLevel, tree.hpp:14 */

/* RunConfig / TraversalConfig subset (engine.hpp:16-36, traversal.hpp:19-23). */
typedef struct {
  int order;        /* p: degrees 0..p-1 (kernels.cpp:25) */
  int n_crit;       /* max bodies per leaf (tree.cpp:78) */
  double theta;     /* MAC opening parameter, in (0,1) (traversal.cpp:8-13) */
  int mutual;       /* 1: mutual traversal (traversal.hpp:76-84): each unordered pair emitted
                       once; executed by the target-owned kernels on the symmetrised lists */
  int precision;    /* fmm_precision */
  int device;       /* CUDA device ordinal */
  int with_acc;     /* 1: also produce acceleration = -grad phi (extension) */
} fmm_config;

typedef struct {
  int64_t nbodies;
  int64_t ncells;
  int64_t nleaves;
  int32_t depth;            /* deepest level present */
  double center[3];         /* Domain (types.hpp:21-28) */
  double half_side;
  int64_t n_m2l;            /* emitted M2L pairs (mutual: once per unordered pair) */
  int64_t n_p2p;            /* emitted P2P leaf pairs (mutual: once per unordered pair) */
  int64_t p2p_body_pairs;   /* sum over the executed P2P leaf pairs of n_t * n_s */
  int32_t level_start[FMM_MAX_LEVEL + 2]; /* cells of level l are [level_start[l], level_start[l+1]) */
  int32_t mutual;           /* lists were emitted by the mutual traversal */
  int64_t n_m2l_exec;       /* executed (target-owned) M2L pairs: n_m2l, or 2 n_m2l in mutual mode */
  int64_t n_p2p_exec;       /* executed P2P leaf pairs: n_p2p, or 2 n_p2p - nleaves in mutual mode */
} fmm_tree_info;

/* Per-stage device times (ms) of the last fmm_evaluate / stage call, CUDA-event timed. */
typedef struct {
  float build_ms, traverse_ms, upward_ms, m2l_ms, p2p_ms, downward_ms, total_ms;
  float p2p_kernel_ms;   /* the P2P kernel alone (roofline numerator's denominator) */
  float m2l_kernel_ms;   /* the M2L kernel alone */
  int32_t p2p_launches, m2l_launches, kernel_launches;
  float exchange_ms;     /* sharded step: the NCCL all-gather of the multipoles (0 otherwise) */
} fmm_stage_times;

/* ---- lifecycle --------------------------------------------------------------------- */
int fmm_create(const fmm_config* cfg, fmm_ctx** out);
void fmm_destroy(fmm_ctx* ctx);
const char* fmm_last_error(const fmm_ctx* ctx);  /* ctx may be NULL: last global error */
const char* fmm_version(void);

/* ---- inputs ------------------------------------------------------------------------ */
/* Bodies as N x {x,y,z,q} FP64 AoS in input order (Body, types.hpp:14-18). Copies in. */
int fmm_set_bodies(fmm_ctx* ctx, const double* xyzq, int64_t n);
/* Same, from a device pointer on the context's device (no H2D copy). */
int fmm_set_bodies_device(fmm_ctx* ctx, const double* d_xyzq, int64_t n);

/* ---- stages (reference call sites in engine.cpp:69-106) ----------------------------- */
int fmm_build_tree(fmm_ctx* ctx);   /* build_tree          tree.cpp:52-119 */
int fmm_traverse(fmm_ctx* ctx);     /* dual_tree_traverse  traversal.hpp:118-133 (lists) */
int fmm_upward(fmm_ctx* ctx);       /* upward_pass         traversal.cpp:36-50 */
int fmm_m2l(fmm_ctx* ctx);          /* KernelVisitor::m2l_pair over the M2L list */
int fmm_p2p(fmm_ctx* ctx);          /* KernelVisitor::p2p_pair over the P2P list */
int fmm_downward(fmm_ctx* ctx);     /* downward_pass       traversal.cpp:52-63 (+ output) */
int fmm_evaluate(fmm_ctx* ctx);     /* all of the above */
/* Time stepping with tree reuse (extension; the reference rebuilds every run; the
 * paper's motivating use). fmm_update_bodies replaces the positions/charges of
 * the same N bodies (input order) and keeps the tree and lists; fmm_evaluate_reuse then checks on
 * the device that every body still lies in its previous leaf's cube and, if so, re-gathers the
 * bodies in the kept tree order and runs upward / M2L / P2P / downward on the kept lists
 * (*reused = 1): the exact FMM of the kept tree (cell geometry, MAC decisions and lists depend
 * only on the cells). Otherwise it runs the full fmm_evaluate (*reused = 0). */
int fmm_update_bodies(fmm_ctx* ctx, const double* xyzq, int64_t n);
int fmm_evaluate_reuse(fmm_ctx* ctx, int* reused);
int fmm_synchronize(fmm_ctx* ctx);
/* 1 (default): fmm_evaluate runs the upward pass (P2M/M2M, needs only the tree) on a second
 * stream concurrently with the dual tree traversal and its list building; M2L joins both.
 * 0 serialises every stage on one stream (each kernel timed alone). */
int fmm_set_overlap(fmm_ctx* ctx, int on);
/* TraversalConfig::mutual (traversal.hpp:19-23) for the next traversal / load_lists: 1 = each
 * unordered pair emitted once (m2l_mutual / mutual p2p semantics, kernels.cpp:113-126, :153-180).
 * The GPU executes the symmetrised lists with target-owned writes (no atomics): results equal
 * the non-mutual mode's. Invalidates the current lists. Not supported with fmm_set_partition. */
int fmm_set_mutual(fmm_ctx* ctx, int on);
/* Test hook for the traversal's rarely taken paths (the production choice is automatic):
 * force_keys64 = 1 emits 64-bit (target, source) keys with the ordered look-back emission even
 * when the tree has <= 2^16 cells (the path C3-C5 take); initial_capacity > 0 starts the
 * frontier and list buffers at that many entries so the overflow regrow-and-rerun runs (the
 * path C4 needs); 0 restores the default sizing. *regrows (optional) = rerun attempts of the
 * last traversal. */
int fmm_set_traversal_debug(fmm_ctx* ctx, int force_keys64, int64_t initial_capacity);
int fmm_get_traversal_regrows(fmm_ctx* ctx, int* regrows);
/* Test / tuning hook for the FP32 P2P kernel's CTA shape (the production choice is automatic, by
 * the mean number of P2P sources per target body): shape = 0 wide CTAs (128 consumer threads,
 * 1 024-body tiles, 6 per SM), 1 narrow CTAs (64 consumer threads, 512-body tiles, 10 per SM),
 * -1 automatic. Results agree to FP32 rounding (the tiles, hence the FP32 partial sums, differ). */
int fmm_set_p2p_shape(fmm_ctx* ctx, int shape);

/* ---- outputs ------------------------------------------------------------------------ */
/* order: 0 = tree (sorted) body order (potentials(), tree.cpp:121-126), 1 = input order.
 * phi: N doubles; acc: 3N doubles (x,y,z per body) or NULL. Host pointers. */
int fmm_get_results(fmm_ctx* ctx, double* phi, double* acc, int order);
/* Device-side outputs in tree order (valid until the next stage call). */
int fmm_results_device(fmm_ctx* ctx, const double** d_phi, const double** d_acc);
int fmm_get_tree_info(fmm_ctx* ctx, fmm_tree_info* info);
int fmm_get_stage_times(fmm_ctx* ctx, fmm_stage_times* t);
/* Stage-level execution trace of the last fmm_evaluate, in the reference's trace CSV vocabulary
 * (Scheduler::export_trace, scheduler.cpp:305-317: task_id,worker_id,kind,start_ns,end_ns):
 * one row per GPU stage (build, traversal, upward, m2l, p2p, downward); worker_id = the stream
 * (0 = FMM stream, 1 = overlap stream); times from CUDA events, relative to the step start.
 * Writes min(max_rows, *n_rows) rows; *n_rows = rows available. */
typedef struct {
  int32_t task_id, worker_id;
  char kind[16];
  int64_t start_ns, end_ns;
} fmm_trace_row;
int fmm_get_stage_trace(fmm_ctx* ctx, fmm_trace_row* rows, int max_rows, int* n_rows);

/* ---- parity exports (reference layout; any pointer may be NULL) --------------------- */
int fmm_get_cells(fmm_ctx* ctx, int32_t* level, uint64_t* key, double* center3, double* radius,
                  int32_t* body_begin, int32_t* body_end, int32_t* child_begin,
                  int32_t* child_count, int32_t* parent);
int fmm_get_permutation(fmm_ctx* ctx, int64_t* perm); /* perm[i] = input index of body i */
/* Lists as CSR by target cell: offsets[ncells+1], sources[n]; sources are in ascending
 * order within each target (a canonical form of the emitted multiset). In mutual mode these
 * are the emitted pairs (n = info.n_m2l / n_p2p), each unordered pair once in the orientation
 * the mutual traversal emitted it. */
int fmm_get_lists(fmm_ctx* ctx, int64_t* m2l_offsets, int32_t* m2l_sources,
                  int64_t* p2p_offsets, int32_t* p2p_sources);
/* Multipoles / locals, ncells x n_coef in the reference coefficient order and convention
 * (kernels.hpp:15-23). */
int fmm_get_expansions(fmm_ctx* ctx, double* multipole, double* local);

/* ---- injection (stage-isolated parity: feed another producer's tree / lists / M) ----- */
/* Load a tree in reference layout with the bodies already set (fmm_set_bodies) and the
 * permutation perm[i] = input index of tree-order body i. */
int fmm_load_tree(fmm_ctx* ctx, int64_t ncells, const int32_t* level, const uint64_t* key,
                  const double* center3, const double* radius, const int32_t* body_begin,
                  const int32_t* body_end, const int32_t* child_begin,
                  const int32_t* child_count, const int32_t* parent, const int64_t* perm);
int fmm_load_lists(fmm_ctx* ctx, int64_t n_m2l, const int32_t* m2l_pairs, int64_t n_p2p,
                   const int32_t* p2p_pairs); /* (target, source) pairs, any order */
int fmm_load_multipoles(fmm_ctx* ctx, const double* multipole); /* ncells x n_coef */
/* Zero the outputs and locals (before re-running m2l/p2p/downward on injected data). */
int fmm_reset_accumulators(fmm_ctx* ctx);

/* ---- single-operator entry points (kernels.hpp:69-103), batched, host buffers --------
 * Thread-per-instance kernels (csrc/ops.cu, k_op / k_op_p2p) over `count` independent
 * instances: the same coefficient order, compile-time term tables and derivative recurrence
 * (expansions.cuh) as the stage kernels, but NOT the stage kernels themselves (those are checked
 * by the stage-isolated tests: injected tree / lists / multipoles, tests/test_gpu_parity.py).
 * Outputs ACCUMULATE (+=) like the reference operators. Coefficient vectors are n_coef(p)
 * doubles each, contiguous per instance. Return FMM_ERR_SINGULAR_* like the reference. */
int fmm_op_p2m(int order, int64_t count, const int32_t* body_offsets /*count+1*/,
               const double* xyzq, const double* centers3, double* M);
int fmm_op_m2m(int order, int64_t count, const double* child_m, const double* shifts3,
               double* parent_m);
int fmm_op_m2l(int order, int64_t count, const double* source_m, const double* disp3,
               double* target_l);
int fmm_op_l2l(int order, int64_t count, const double* parent_l, const double* shifts3,
               double* child_l);
/* L2P over `count` local expansions, each applied to its body range; acc may be NULL. */
int fmm_op_l2p(int order, int64_t count, const int32_t* body_offsets, const double* L,
               const double* centers3, const double* xyzq, double* phi, double* acc);
/* P2P over `count` (target range, source range) pairs of one body array (xyzq, FP64). */
int fmm_op_p2p(int64_t count, const int32_t* ranges4 /*tb,te,sb,se*/, const double* xyzq,
               int precision, double* phi, double* acc);
int fmm_op_evaluate_multipole(int order, int64_t count, const double* M, const double* x3,
                              const double* centers3, double* out);
/* D_g(R) = (1/g!) d^g (1/|R|) for all |g| <= max_degree (multi_index.cpp:59-85). */
int fmm_op_laplace_derivatives(int max_degree, int64_t count, const double* r3, double* out);
/* Bit-exact tree-level helpers (tree.cpp:10-39, traversal.cpp:8-13) on the device. */
int fmm_op_compute_bounds(const double* xyzq, int64_t n, double* center3, double* half_side);
int fmm_op_morton_key(int64_t count, const double* p3, const double* center3,
                      double half_side, int level, uint64_t* out);
int fmm_op_mac(int64_t count, const double* tcenter3, const double* tradius,
               const double* scenter3, const double* sradius, double theta, int32_t* out);

/* ---- multi-GPU sharding ----------------------------------------------
 * One process per GPU, every rank holds all bodies. After fmm_set_partition(rank, world) the
 * traversal also splits the target leaves into `world` contiguous body (Morton) ranges balanced
 * by cost, and a sharded step is:
 *   fmm_build_tree; fmm_traverse; fmm_upward_local(send);
 *   <all-gather: recv[world * chunk] <- send[chunk]  (NCCL, caller side; chunk = shard.chunk_doubles)>
 *   fmm_upward_finish(recv); fmm_m2l; fmm_p2p; fmm_downward;
 * after which the potentials/accelerations of bodies [shard.body_begin, shard.body_end) (tree
 * order) are final on this rank. send/recv are device pointers on the context's device. */
typedef struct {
  int32_t rank, world;
  int64_t body_begin, body_end;   /* own bodies, tree order */
  int64_t own_leaves, own_cells;  /* leaves / cells whose multipoles this rank computes */
  int64_t chunk_doubles;          /* all-gather chunk per rank (doubles) */
} fmm_shard_info;

int fmm_set_partition(fmm_ctx* ctx, int rank, int world);
int fmm_get_shard_info(fmm_ctx* ctx, fmm_shard_info* info);
int fmm_upward_local(fmm_ctx* ctx, double* d_send);
int fmm_upward_finish(fmm_ctx* ctx, const double* d_recv);
/* Run subsequent stages on `stream` (a cudaStream_t; NULL restores the context's own stream),
 * e.g. the stream an NCCL collective is issued on. */
int fmm_set_stream(fmm_ctx* ctx, void* stream);
/* ---- the sharded step with its NCCL exchange inside the library ----------------------
 * Bootstrap like NCCL itself: rank 0 calls fmm_comm_unique_id and ships the 128 bytes to the
 * other ranks (MPI_Bcast, torch.distributed, a file, ...); every rank then calls
 * fmm_comm_init(ctx, id, rank, world) (= ncclCommInitRank + fmm_set_partition). A step is
 *   fmm_set_bodies / fmm_set_bodies_shard;  fmm_evaluate_sharded(ctx, &info);
 * which runs build, traversal (cost plan on the first step, Morton-filtered targets later), the
 * own cells' P2M/M2M, one ncclAllGather of the owned multipoles (on a second stream, under the
 * P2P kernel), the shared ancestors, M2L, P2P and L2L/L2P of the own leaves. Afterwards the
 * tree-order body range [info.body_begin, info.body_end) is final on this rank:
 * fmm_get_owned_results copies it (and its input-order indices) to the host. NCCL is loaded at
 * run time (libnccl.so.2); FMM_ERR_UNSUPPORTED without it. world = 1 runs fmm_evaluate. */
#define FMM_COMM_ID_BYTES 128
int fmm_comm_unique_id(void* id);
int fmm_comm_init(fmm_ctx* ctx, const void* id, int rank, int world);
int fmm_comm_destroy(fmm_ctx* ctx);
/* Exchange override: a host callback that all-gathers `count` doubles per rank from d_send into
 * d_recv (rank-major, device pointers) for work queued on `stream` (a cudaStream_t the callback
 * must synchronise or enqueue on). When set, fmm_set_bodies_shard / fmm_evaluate_sharded use it
 * instead of NCCL and need no communicator (fmm_set_partition gives rank / world): hosts with
 * their own transport, and the multi-process test on one GPU (NCCL refuses two ranks on one
 * device). The callback returns 0 on success. fn = NULL restores NCCL. */
typedef int (*fmm_allgather_fn)(const double* d_send, double* d_recv, int64_t count, void* stream,
                                void* user);
int fmm_set_allgather(fmm_ctx* ctx, fmm_allgather_fn fn, void* user);
/* Bodies of all ranks from each rank's share: rank r passes bodies [r*chunk, min(n_total,
 * (r+1)*chunk)) of the input order, chunk = ceil(n_total / world); the shares are all-gathered
 * over NVLink into the full input array (one H2D of the share per rank). */
int fmm_set_bodies_shard(fmm_ctx* ctx, const double* xyzq_share, int64_t n_share, int64_t n_total);
int fmm_evaluate_sharded(fmm_ctx* ctx, fmm_shard_info* info);
/* Results of the own tree-order range (info.body_begin..body_end) to host buffers of
 * body_end - body_begin entries; input_index (optional) = their input-order indices. */
int fmm_get_owned_results(fmm_ctx* ctx, double* phi, double* acc, int64_t* input_index);

/* Host-only (no GPU): the partition plan the traversal uses. cell_cost holds each leaf's cost
 * (ignored for non-leaves). bounds[world+1] (body indices), owner[ncells] (rank or -1). */
int fmm_plan_partition(int64_t ncells, const int32_t* body_begin, const int32_t* body_end,
                       const int32_t* child_count, const double* cell_cost, int world,
                       int64_t* bounds, int32_t* owner);

/* ---- synthetic BASELINE inputs (host-side generator) ----------------- */
/* config: 1..5 = BASELINE configs C1..C5 distributions; writes N x {x,y,z,q}. */
int fmm_generate_bodies(int config, int64_t n, uint64_t seed, double* xyzq);

#ifdef __cplusplus
}
#endif
#endif
