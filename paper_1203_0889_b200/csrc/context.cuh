// context.cuh — the fmm_ctx state: device-resident bodies, tree, interaction lists,
// expansions and outputs, plus the stage entry points implemented across the .cu files.
//
// HBM layout (all tree-order unless noted):
//   xyzq_in   double4[N]   input bodies (input order)
//   bodies    double4[N]   x,y,z,q in tree order (FP64 P2P, P2M, L2P)
//   bodyf     float4[N]    x-cx,y-cy,z-cz,q relative to the body's own leaf centre (FP32 P2P)
//   bodyl     float4[N]    the FP32 rounding residuals of bodyf's x,y,z (compensated near tiles)
//   perm      int32[N]     tree-order body -> input index
//   cells     SoA: level i32, key u64, cr double4 (cx,cy,cz,radius), body_begin/end,
//             child_begin/count, parent (i32) — reference Cell (tree.hpp:21-36), BFS order
//   lists     CSR by target cell: m2l_off int64[ncells+1], m2l_src int32[n_m2l]; same for p2p
//   M, L      double[ncells * n_coef] reference coefficient order (multi_index.cpp:16-20)
//   phi, acc  double[N], double[3N] outputs in tree order
#pragma once

#include <cuda_runtime.h>

#include <string>
#include <vector>

#include "common.cuh"

struct fmm_ctx {
  fmm_config cfg{};
  int ncoef = 0;
  cudaStream_t stream = nullptr;
  cudaStream_t stream2 = nullptr;  // concurrent stream (upward pass alongside the traversal)
  cudaStream_t stream3 = nullptr;  // P2P list preparation alongside M2L (high priority)
  cudaStream_t own_stream = nullptr;  // the context's stream while a caller stream is set
  std::string err;

  // bodies
  int64_t N = 0;
  fmmb::DBuf<double4> xyzq_in;
  fmmb::DBuf<double4> bodies;
  fmmb::DBuf<float4> bodyf;
  fmmb::DBuf<float4> bodyl;
  fmmb::DBuf<int32_t> perm;
  fmmb::DBuf<int32_t> leaf_of_body;  // tree-order body -> leaf cell index

  // tree
  int64_t ncells = 0, nleaves = 0;
  int depth = 0;
  int32_t level_start[FMM_MAX_LEVEL + 2] = {};
  double center[3] = {0, 0, 0};
  double half_side = 0;
  fmmb::DBuf<int32_t> c_level, c_body_begin, c_body_end, c_child_begin, c_child_count, c_parent;
  fmmb::DBuf<uint64_t> c_key;
  fmmb::DBuf<double4> c_cr;
  fmmb::DBuf<int32_t> leaves;  // leaf cell indices, ascending

  // lists (CSR by target)
  int64_t n_m2l = 0, n_p2p = 0, p2p_body_pairs = 0;  // executed lists (mutual: symmetrised)
  int64_t n_m2l_emit = 0, n_p2p_emit = 0;            // emitted pairs (mutual: once per unordered pair)
  fmmb::DBuf<uint8_t> m2l_mir, p2p_mir;              // mutual: 1 = entry is a mirror of an emitted pair
  fmmb::DBuf<uint64_t> mut_keys;                     // mutual: emitted + mirrored keys
  fmmb::DBuf<int64_t> m2l_off, p2p_off;
  fmmb::DBuf<int32_t> m2l_src, p2p_src;
  fmmb::DBuf<int32_t> p2p_tgt;  // target cell of each P2P CSR entry
  fmmb::DBuf<int32_t> m2l_targets;  // cells with non-empty M2L lists
  int64_t n_m2l_targets = 0;

  // P2P work list (cost sorted)
  fmmb::DBuf<int4> p2p_items;       // target leaf, list begin, list end, partial slot (-1 = direct)
  int64_t n_p2p_items = 0;
  fmmb::DBuf<double> p2p_partial;   // [slot][target body][4] (phi, ax, ay, az)
  fmmb::DBuf<int4> p2p_reduce;      // target leaf, first slot, n slots, body begin
  fmmb::DBuf<int64_t> p2p_pre;      // exclusive prefix of source-body counts over the P2P list
  fmmb::DBuf<int4> p2p_ent;
  fmmb::DBuf<double4> leaf_lo, leaf_hi;  // tight body boxes of the leaves (FP32 P2P near test)
  fmmb::DBuf<int64_t> ent_cls, ent_pre;  // entry class counters (near | far << 32) and their scan
  // P2P list preparation: its own stream slot and scratch (it may run concurrently with M2L)
  cudaStream_t pstream = nullptr;        // = stream, or stream3 while evaluate overlaps it
  bool p2p_overlap = false;              // set by evaluate: prepare the P2P work list on stream3
  cudaEvent_t ev_lists = nullptr;        // emitted keys complete / P2P work list ready
  cudaEvent_t ev_l2l = nullptr;          // L2L done (it runs beside P2P)
  bool p2p_pending = false;              // work list begun, not finished (p2p_worklist_end)
  fmmb::DBuf<unsigned char> tmp2;        // CUB temporary storage of the P2P path
  fmmb::DBuf<uint64_t> p2p_keys_b2, p2p_keys_c;
  fmmb::DBuf<int32_t> p2p_i32a, p2p_i32b, p2p_i32c;
  fmmb::DBuf<int64_t> p2p_sum;
  fmmb::DBuf<int4> p2p_items_raw;
  int64_t n_p2p_reduce = 0;

  // expansions and outputs
  fmmb::DBuf<double> M, L;
  fmmb::DBuf<double> m2l_mt;          // detraced multipoles (p <= 6 kernel)
  fmmb::DBuf<double> m2l_scratch;     // per-warp-slot partial Lambda rows (p >= 7 kernel)
  fmmb::DBuf<double> phi, acc;
  fmmb::DBuf<double> phi_p2p, acc_p2p;  // near-field part (tree order)
  fmmb::DBuf<double> phi_in, acc_in;    // outputs scattered back to input order

  // scratch
  fmmb::DBuf<unsigned char> tmp;
  fmmb::DBuf<uint64_t> keys_a, keys_b;
  fmmb::DBuf<int32_t> idx_a, idx_b;
  fmmb::DBuf<int64_t> scan_a;
  fmmb::DBuf<int2> pairs_a, pairs_b, pairs_c;
  fmmb::DBuf<int32_t> i32_a, i32_b, i32_c;
  fmmb::DBuf<int64_t> d_counters;
  fmmb::DBuf<double> small;
  fmmb::DBuf<int2> pairs_d;         // second traversal frontier
  fmmb::DBuf<uint64_t> m2l_keys, p2p_keys;  // emitted (target << sbits | source)
  fmmb::DBuf<uint64_t> trav_ctr;            // traversal level counters + chunk tickets
  fmmb::DBuf<uint32_t> lb_flag;             // traversal look-back: per-chunk status (epoch tagged)
  fmmb::DBuf<uint64_t> lb_val;              // traversal look-back: per-chunk aggregate / prefix
  uint32_t trav_epoch = 0;                  // one epoch per k_step launch
  bool dbg_keys64 = false;                  // test hook: 64-bit keys on any tree
  int64_t dbg_cap = 0;                      // test hook: initial traversal buffer capacity
  uint64_t M_version = 0, mt_version = ~0ull;  // multipoles written / detraced rows built from them
  bool build_coop_ok = true;                // cooperative all-levels build kernel usable on this device
  int p2p_shape = -1;                       // FP32 P2P CTA shape: -1 automatic, 0 wide, 1 narrow
  int trav_regrows = 0;                     // rerun attempts of the last traversal
  fmmb::DBuf<int32_t> bnd;           // child boundaries of one level (9 per cell)
  fmmb::DBuf<int32_t> bnd_lev;       // device level table (tree build)
  int last_depth = 6;                // depth of the previous build (level batch, sorted digits)
  bool depth_known = false;
  int64_t* hpin = nullptr;           // pinned host scratch (64 x int64)

  // sharding: target leaves split by contiguous body (Morton) range
  int rank = 0, world = 1;
  int64_t shard_b0 = 0, shard_b1 = 0;      // own body range [b0, b1) in tree order
  const int32_t* wl = nullptr;             // work leaves: all leaves, or the rank's own leaves
  int64_t nwl = 0;
  fmmb::DBuf<int32_t> own_leaves;
  fmmb::DBuf<int32_t> owner;               // per cell: owning rank, -1 = straddles ranks
  fmmb::DBuf<int32_t> rank_cells;          // cells owned by each rank, concatenated
  std::vector<int64_t> rank_cells_off;     // world + 1 offsets into rank_cells
  int64_t chunk_cells = 0;                 // max cells owned by a rank (exchange chunk)
  bool shard_planned = false;
  // partition reuse: the first sharded step plans from its full lists (cost-balanced) and keeps
  // the rank boundaries as Morton keys; later steps map them onto the new tree (snapped to leaf
  // starts) and traverse only pairs whose target meets the rank's range
  std::vector<uint64_t> plan_keys;         // world + 1 boundary keys
  int plan_world = 0;                      // world the plan was made for (0 = none)
  bool shard_from_plan = false;            // this step's bounds came from plan_keys
  fmmb::DBuf<uint64_t> body_keys;          // sorted 63-bit body keys (tree order), sharded runs
  bool body_keys_valid = false;
  fmmb::DBuf<int64_t> shard_bounds;        // device copy of the world + 1 body bounds
  // NCCL (comm.cu): the communicator of fmm_comm_init and the exchange buffers of the step
  void* nccl_comm = nullptr;               // ncclComm_t
  fmm_allgather_fn ag_fn = nullptr;        // exchange override (fmm_set_allgather)
  void* ag_user = nullptr;
  int comm_rank = 0, comm_world = 0;
  fmmb::DBuf<double> shard_send, shard_recv;
  fmmb::DBuf<double4> body_share;          // fmm_set_bodies_shard staging (one chunk)
  int64_t trav_b0 = 0, trav_b1 = 0;        // traversal target filter [b0, b1)

  // fmm_evaluate: 1 = upward pass on stream2 concurrently with the traversal; 2 = also M2L and
  // P2P concurrently (M2L on the high-priority stream)
  int overlap = 1;

  // state
  bool have_bodies = false, have_tree = false, have_lists = false, have_M = false,
       have_L = false, have_out = false;

  // timing
  fmm_stage_times times{};
  cudaEvent_t ev[16] = {};  // stage events (capi.cu EV_*)
  int kernel_launches = 0;
};

namespace fmmb {

// tree_build.cu
void build_tree(fmm_ctx* c);
void unpermute_results(fmm_ctx* c, double* phi_in, double* acc_in);  // tree -> input order
void gather_bodies(fmm_ctx* c);  // bodies/bodyf/leaf_of_body from perm + tree
bool refit_bodies(fmm_ctx* c);   // tree reuse: false if a body left its leaf cube, else re-gather
// traverse.cu
void traverse(fmm_ctx* c);
void finish_lists(fmm_ctx* c, int64_t n_m2l, int64_t n_p2p);  // lists from c->m2l_keys/p2p_keys
void lists_from_pairs(fmm_ctx* c, const int2* d_m2l, int64_t n_m2l, const int2* d_p2p,
                      int64_t n_p2p);
// comm.cu (NCCL bound at run time)
void comm_unique_id(void* out128);
int comm_version();
void comm_init(fmm_ctx* c, const void* id128, int rank, int world);
void comm_destroy(fmm_ctx* c);
void comm_all_gather(fmm_ctx* c, const double* send, double* recv, size_t count, cudaStream_t s);
// shard.cu
void plan_shards(fmm_ctx* c);      // after the lists: partition, own leaves, owners
bool shard_bounds_from_plan(fmm_ctx* c);  // before the traversal: bounds from the kept plan
void shard_assign(fmm_ctx* c);     // owners, per-rank cell lists, own leaves from c->shard_bounds
void shard_pack(fmm_ctx* c, double* d_send, cudaStream_t s);
void shard_unpack(fmm_ctx* c, const double* d_recv, cudaStream_t s);
void plan_partition_host(int64_t ncells, const int32_t* bb, const int32_t* be, const int32_t* cc,
                         const double* cell_cost, int world, int64_t* bounds, int32_t* owner);
// p2p.cu
void build_p2p_worklist(fmm_ctx* c);  // begin + end on c->pstream
void p2p_worklist_begin(fmm_ctx* c);  // entry prefix, per-leaf sums, async read of the total
void p2p_worklist_end(fmm_ctx* c);    // items, entries, cost sort (host syncs on c->pstream)
void build_p2p_entries(fmm_ctx* c);  // FP32 entries (near test on the current bodies)
void run_p2p(fmm_ctx* c, cudaStream_t s);
// expansions.cu
void run_upward(fmm_ctx* c, cudaStream_t s, int mode = 0);  // 0 all, 1 own cells, 2 shared cells
void run_m2l(fmm_ctx* c, cudaStream_t s);
void run_detrace(fmm_ctx* c, cudaStream_t s);  // M2L's detraced source rows from the current multipoles
void run_downward(fmm_ctx* c, cudaStream_t s, int part = 3);  // 1: L2L, 2: L2P + combine, 3: both

// CUB temp helpers (the second one belongs to the P2P preparation path)
void* temp_storage(fmm_ctx* c, size_t bytes);
void* temp_storage2(fmm_ctx* c, size_t bytes);

}  // namespace fmmb

namespace fmmb {
// Single-operator entry points (fmm_op_*), device implementations; host buffers in/out.
void op_bounds(const double* xyzq, int64_t n, double* center3, double* half_side);
void op_morton(int64_t count, const double* p3, const double* center3, double half_side, int level,
               uint64_t* out);
void op_mac(int64_t count, const double* tc3, const double* tr, const double* sc3, const double* sr,
            double theta, int32_t* out);
void op_p2p(int64_t count, const int32_t* ranges4, const double* xyzq, int64_t nbodies, int precision,
            double* phi, double* acc);
void op_expansion(int kind, int order, int64_t count, const int32_t* offsets, const double* in,
                  const double* vec3, const double* xyzq, int64_t nbodies, double* out, double* out2);
// kinds for op_expansion
enum { OP_P2M = 0, OP_M2M = 1, OP_M2L = 2, OP_L2L = 3, OP_L2P = 4, OP_EVAL = 5, OP_DERIV = 6 };
}  // namespace fmmb
