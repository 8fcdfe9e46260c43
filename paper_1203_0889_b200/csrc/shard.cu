// shard.cu — multi-GPU sharding of the FMM step.
//
// Every rank holds all bodies, the (deterministic, bit-identical) tree and the interaction
// lists. Target leaves are split into `world` contiguous body (Morton) ranges balanced by cost
// (P2P body pairs + an M2L flop weight per list entry). A cell is owned by rank r when its body
// range lies inside rank r's range, and is "shared" (owner -1) when it straddles ranks; leaves
// never straddle because the split points are leaf boundaries. Each rank
//   1. computes the multipoles of its own cells (P2M of its leaves, M2M of its non-leaf cells),
//   2. all-gathers them (NCCL over NVLink, caller side: equal-size chunks of chunk_cells rows),
//   3. unpacks the other ranks' cells and recomputes the shared ancestors (deepest first),
//   4. runs M2L for every target cell meeting its range, P2P and L2P for its own leaves.
// The only data-path exchange is step 2.
#include <algorithm>
#include <vector>

#include <cub/cub.cuh>

#include "context.cuh"

namespace fmmb {
namespace {

// cost per leaf: P2P body pairs + m2l_weight x (M2L list entries of the leaf)
__global__ void k_leaf_costs(const int32_t* __restrict__ leaves, int64_t nleaves, const int64_t* __restrict__ poff,
                             const int32_t* __restrict__ psrc, const int64_t* __restrict__ moff,
                             const int32_t* __restrict__ bb, const int32_t* __restrict__ be, double m2l_weight,
                             double* __restrict__ cost) {
  const int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= nleaves) return;
  const int32_t leaf = leaves[w];
  int64_t s = 0;
  for (int64_t k = poff[leaf] + lane; k < poff[leaf + 1]; k += 32) {
    const int32_t q = psrc[k];
    s += be[q] - bb[q];
  }
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0)
    cost[w] = double(s) * double(be[leaf] - bb[leaf]) + m2l_weight * double(moff[leaf + 1] - moff[leaf]);
}

__global__ void k_pack(const int32_t* __restrict__ cells, int64_t count, int ncoef, const double* __restrict__ M,
                       double* __restrict__ send) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= count * ncoef) return;
  const int64_t k = i / ncoef, e = i - k * ncoef;
  send[i] = M[(int64_t)cells[k] * ncoef + e];
}

__global__ void k_unpack(const int32_t* __restrict__ cells, int64_t count, int ncoef, const double* __restrict__ recv,
                         double* __restrict__ M) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= count * ncoef) return;
  const int64_t k = i / ncoef, e = i - k * ncoef;
  M[(int64_t)cells[k] * ncoef + e] = recv[i];
}

}  // namespace

// Host-only partition plan (also exported as fmm_plan_partition for CPU tests).
void plan_partition_host(int64_t ncells, const int32_t* bb, const int32_t* be, const int32_t* cc,
                         const double* cell_cost, int world, int64_t* bounds, int32_t* owner) {
  std::vector<int32_t> leaves;
  for (int64_t i = 0; i < ncells; ++i)
    if (cc[i] == 0) leaves.push_back(static_cast<int32_t>(i));
  std::sort(leaves.begin(), leaves.end(), [&](int32_t a, int32_t b) { return bb[a] < bb[b]; });
  double total = 0.0;
  for (int32_t l : leaves) total += cell_cost[l];
  const int64_t nbody = ncells > 0 ? be[0] : 0;  // the root covers every body
  bounds[0] = 0;
  double acc = 0.0;
  int r = 1;
  for (size_t k = 0; k < leaves.size() && r < world; ++k) {
    // leaf k starts rank r's range once the running cost reaches r/world of the total
    while (r < world && acc >= total * r / world) bounds[r++] = bb[leaves[k]];
    acc += cell_cost[leaves[k]];
  }
  while (r < world) bounds[r++] = nbody;
  bounds[world] = nbody;
  for (int q = 1; q <= world; ++q) bounds[q] = std::max(bounds[q], bounds[q - 1]);
  for (int64_t i = 0; i < ncells; ++i) {
    owner[i] = -1;
    for (int q = 0; q < world; ++q)
      if (bounds[q] <= bb[i] && be[i] <= bounds[q + 1] && bounds[q] < bounds[q + 1]) {
        owner[i] = q;
        break;
      }
  }
}

namespace {

// owner[i] = the rank whose body range contains cell i, -1 when it straddles ranks (or is empty)
__global__ void k_owner(const int32_t* __restrict__ bb, const int32_t* __restrict__ be, int64_t ncells,
                        const int64_t* __restrict__ bounds, int world, int32_t* __restrict__ owner,
                        uint32_t* __restrict__ okey, int32_t* __restrict__ iota) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= ncells) return;
  int32_t o = -1;
  for (int q = 0; q < world; ++q)
    if (bounds[q] <= bb[i] && be[i] <= bounds[q + 1] && bounds[q] < bounds[q + 1]) {
      o = q;
      break;
    }
  owner[i] = o;
  okey[i] = static_cast<uint32_t>(o + 1);  // 0 = shared, q + 1 = rank q
  iota[i] = static_cast<int32_t>(i);
}

// offsets of each rank's cells in the owner-sorted cell list
__global__ void k_rank_offsets(const uint32_t* __restrict__ skey, int64_t ncells, int world, int64_t* __restrict__ off) {
  const int q = threadIdx.x;
  if (q > world) return;
  int64_t lo = 0, hi = ncells;  // first index with key >= q + 1
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (skey[mid] < static_cast<uint32_t>(q + 1)) lo = mid + 1; else hi = mid;
  }
  off[q] = lo;
}

__global__ void k_flag_own_leaves(const int32_t* __restrict__ leaves, int64_t nleaves, const int32_t* __restrict__ owner,
                                  int rank, int32_t* __restrict__ flag) {
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k < nleaves) flag[k] = owner[leaves[k]] == rank;
}

// Morton boundary keys -> body bounds on this tree: first body whose key reaches the boundary,
// snapped down to the start of its leaf (leaves never straddle ranks)
__global__ void k_plan_bounds(const uint64_t* __restrict__ pk, int world, const uint64_t* __restrict__ keys, int64_t n,
                              const int32_t* __restrict__ leaf_of_body, const int32_t* __restrict__ bb,
                              int64_t* __restrict__ bounds) {
  const int q = threadIdx.x;
  if (q > world) return;
  int64_t b;
  if (q == 0) {
    b = 0;
  } else if (q == world) {
    b = n;
  } else {
    int64_t lo = 0, hi = n;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (keys[mid] < pk[q]) lo = mid + 1; else hi = mid;
    }
    b = lo < n ? bb[leaf_of_body[lo]] : n;
  }
  bounds[q] = b;
}

__global__ void k_bound_keys(const int64_t* __restrict__ bounds, int world, const uint64_t* __restrict__ keys, int64_t n,
                             uint64_t* __restrict__ pk) {
  const int q = threadIdx.x;
  if (q > world) return;
  pk[q] = bounds[q] < n ? keys[bounds[q]] : ~0ull;
}

}  // namespace

// First sharded step: cost-balanced plan from this step's full lists; the bounds are kept as
// Morton keys for the following steps.
void plan_shards(fmm_ctx* c) {
  cudaStream_t s = c->stream;
  const int64_t nl = c->nleaves, nc = c->ncells;
  // 1. leaf costs on the device (all leaves), copied back with the cell ranges
  double* cost = c->small.ensure(std::max<int64_t>(nl, 1) + 64);
  const int p = c->cfg.order;
  const double m2l_weight = (2.0 * n_coef(p) * (p + 3) * (p + 4) * (p + 5) / 120.0) / 20.0;  // ~flops / P2P flops
  k_leaf_costs<<<ceil_div(nl * 32, 256), 256, 0, s>>>(c->leaves.p, nl, c->p2p_off.p, c->p2p_src.p, c->m2l_off.p,
                                                      c->c_body_begin.p, c->c_body_end.p, m2l_weight, cost);
  CK_LAUNCH("k_leaf_costs");
  std::vector<double> hcost(nl);
  std::vector<int32_t> hleaves(nl), bb(nc), be(nc), cc(nc);
  CK(cudaMemcpyAsync(hcost.data(), cost, nl * sizeof(double), cudaMemcpyDeviceToHost, s));
  CK(cudaMemcpyAsync(hleaves.data(), c->leaves.p, nl * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  CK(cudaMemcpyAsync(bb.data(), c->c_body_begin.p, nc * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  CK(cudaMemcpyAsync(be.data(), c->c_body_end.p, nc * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  CK(cudaMemcpyAsync(cc.data(), c->c_child_count.p, nc * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  std::vector<double> cell_cost(nc, 0.0);
  for (int64_t k = 0; k < nl; ++k) cell_cost[hleaves[k]] = hcost[k];
  // 2. host plan (bounds; owners are recomputed on the device by shard_assign)
  std::vector<int64_t> bounds(c->world + 1);
  std::vector<int32_t> owner(nc);
  plan_partition_host(nc, bb.data(), be.data(), cc.data(), cell_cost.data(), c->world, bounds.data(), owner.data());
  int64_t* dbounds = c->shard_bounds.ensure(c->world + 1);
  CK(cudaMemcpyAsync(dbounds, bounds.data(), (c->world + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, s));
  // 3. keep the plan as Morton boundary keys (when this tree has its sorted keys)
  if (c->body_keys_valid) {
    uint64_t* dk = reinterpret_cast<uint64_t*>(c->small.p) + 0;  // cost buffer is consumed
    k_bound_keys<<<1, 128, 0, s>>>(dbounds, c->world, c->body_keys.p, c->N, dk);
    CK_LAUNCH("k_bound_keys");
    c->plan_keys.assign(c->world + 1, 0);
    CK(cudaMemcpyAsync(c->plan_keys.data(), dk, (c->world + 1) * sizeof(uint64_t), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    c->plan_world = c->world;
  }
  c->shard_b0 = bounds[c->rank];
  c->shard_b1 = bounds[c->rank + 1];
  c->kernel_launches += 2;
  shard_assign(c);
}

// Later sharded steps (before the traversal): the kept Morton boundaries mapped onto this tree.
bool shard_bounds_from_plan(fmm_ctx* c) {
  if (c->plan_world != c->world || !c->body_keys_valid || static_cast<int>(c->plan_keys.size()) != c->world + 1)
    return false;
  cudaStream_t s = c->stream;
  uint64_t* dk = reinterpret_cast<uint64_t*>(c->small.ensure(2 * (c->world + 1) + 8));
  CK(cudaMemcpyAsync(dk, c->plan_keys.data(), (c->world + 1) * sizeof(uint64_t), cudaMemcpyHostToDevice, s));
  int64_t* dbounds = c->shard_bounds.ensure(c->world + 1);
  k_plan_bounds<<<1, 128, 0, s>>>(dk, c->world, c->body_keys.p, c->N, c->leaf_of_body.p, c->c_body_begin.p, dbounds);
  CK_LAUNCH("k_plan_bounds");
  int64_t* h = c->hpin;
  CK(cudaMemcpyAsync(h, dbounds + c->rank, 2 * sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  c->shard_b0 = h[0];
  c->shard_b1 = h[1];
  c->kernel_launches += 1;
  return true;
}

// Owners, every rank's owned-cell list (ascending cell index), own leaves and the exchange chunk
// size, all from c->shard_bounds on the device.
void shard_assign(fmm_ctx* c) {
  cudaStream_t s = c->stream;
  const int64_t nc = c->ncells, nl = c->nleaves;
  const int world = c->world;
  int32_t* owner = c->owner.ensure(nc);
  uint32_t* okey = reinterpret_cast<uint32_t*>(c->i32_a.ensure(2 * (nc + 1)));
  uint32_t* okey_s = okey + (nc + 1);
  int32_t* iota = c->i32_b.ensure(nc + 1);
  int32_t* cells = c->rank_cells.ensure(nc + 1);
  k_owner<<<ceil_div(nc, 256), 256, 0, s>>>(c->c_body_begin.p, c->c_body_end.p, nc, c->shard_bounds.p, world, owner,
                                            okey, iota);
  CK_LAUNCH("k_owner");
  int end_bit = 1;
  while ((1 << end_bit) <= world) ++end_bit;
  size_t sb = 0;
  CK(cub::DeviceRadixSort::SortPairs(nullptr, sb, okey, okey_s, iota, cells, (int)nc, 0, end_bit, s));
  CK(cub::DeviceRadixSort::SortPairs(temp_storage(c, sb), sb, okey, okey_s, iota, cells, (int)nc, 0, end_bit, s));
  int64_t* doff = c->scan_a.ensure(world + 2);
  k_rank_offsets<<<1, 128, 0, s>>>(okey_s, nc, world, doff);
  CK_LAUNCH("k_rank_offsets");
  // own leaves (ascending cell index)
  int32_t* flag = c->i32_c.ensure(nl + 1);
  k_flag_own_leaves<<<ceil_div(nl, 256), 256, 0, s>>>(c->leaves.p, nl, owner, c->rank, flag);
  CK_LAUNCH("k_flag_own_leaves");
  int32_t* own = c->own_leaves.ensure(nl + 1);
  int64_t* nsel = c->d_counters.ensure(32) + 2;
  sb = 0;
  CK(cub::DeviceSelect::Flagged(nullptr, sb, c->leaves.p, flag, own, nsel, (int)nl, s));
  CK(cub::DeviceSelect::Flagged(temp_storage(c, sb), sb, c->leaves.p, flag, own, nsel, (int)nl, s));
  int64_t* h = c->hpin;
  CK(cudaMemcpyAsync(h, doff, (world + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  CK(cudaMemcpyAsync(h + world + 1, nsel, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  // rank_cells_off[q] = start of rank q's cells in the owner-sorted list (shared cells sort first)
  c->rank_cells_off.assign(world + 1, 0);
  for (int q = 0; q <= world; ++q) c->rank_cells_off[q] = h[q];
  c->chunk_cells = 0;
  for (int q = 0; q < world; ++q)
    c->chunk_cells = std::max(c->chunk_cells, c->rank_cells_off[q + 1] - c->rank_cells_off[q]);
  c->wl = own;
  c->nwl = h[world + 1];
  c->shard_planned = true;
  c->kernel_launches += 5;
}

void shard_pack(fmm_ctx* c, double* d_send, cudaStream_t s) {
  const int64_t b = c->rank_cells_off[c->rank], n = c->rank_cells_off[c->rank + 1] - b;
  if (n > 0)
    k_pack<<<ceil_div(n * c->ncoef, 256), 256, 0, s>>>(c->rank_cells.p + b, n, c->ncoef, c->M.p, d_send);
  CK_LAUNCH("k_pack");
  c->kernel_launches += 1;
}

void shard_unpack(fmm_ctx* c, const double* d_recv, cudaStream_t s) {
  for (int q = 0; q < c->world; ++q) {
    if (q == c->rank) continue;
    const int64_t b = c->rank_cells_off[q], n = c->rank_cells_off[q + 1] - b;
    if (n > 0)
      k_unpack<<<ceil_div(n * c->ncoef, 256), 256, 0, s>>>(c->rank_cells.p + b, n, c->ncoef,
                                                          d_recv + (int64_t)q * c->chunk_cells * c->ncoef, c->M.p);
    CK_LAUNCH("k_unpack");
    c->kernel_launches += 1;
  }
}

}  // namespace fmmb
