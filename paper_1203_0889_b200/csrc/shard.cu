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
  // 2. host plan
  std::vector<int64_t> bounds(c->world + 1);
  std::vector<int32_t> owner(nc);
  plan_partition_host(nc, bb.data(), be.data(), cc.data(), cell_cost.data(), c->world, bounds.data(), owner.data());
  // 3. own leaves, per-rank owned cell lists, chunk size
  std::vector<int32_t> own_leaves;
  for (int64_t k = 0; k < nl; ++k)
    if (owner[hleaves[k]] == c->rank) own_leaves.push_back(hleaves[k]);
  std::vector<int32_t> cells;
  c->rank_cells_off.assign(c->world + 1, 0);
  for (int q = 0; q < c->world; ++q) {
    c->rank_cells_off[q] = static_cast<int64_t>(cells.size());
    for (int64_t i = 0; i < nc; ++i)
      if (owner[i] == q) cells.push_back(static_cast<int32_t>(i));
  }
  c->rank_cells_off[c->world] = static_cast<int64_t>(cells.size());
  c->chunk_cells = 0;
  for (int q = 0; q < c->world; ++q)
    c->chunk_cells = std::max(c->chunk_cells, c->rank_cells_off[q + 1] - c->rank_cells_off[q]);
  CK(cudaMemcpyAsync(c->owner.ensure(nc), owner.data(), nc * sizeof(int32_t), cudaMemcpyHostToDevice, s));
  CK(cudaMemcpyAsync(c->own_leaves.ensure(own_leaves.size() + 1), own_leaves.data(),
                     own_leaves.size() * sizeof(int32_t), cudaMemcpyHostToDevice, s));
  CK(cudaMemcpyAsync(c->rank_cells.ensure(cells.size() + 1), cells.data(), cells.size() * sizeof(int32_t),
                     cudaMemcpyHostToDevice, s));
  CK(cudaStreamSynchronize(s));  // host vectors leave scope
  c->wl = c->own_leaves.p;
  c->nwl = static_cast<int64_t>(own_leaves.size());
  c->shard_b0 = bounds[c->rank];
  c->shard_b1 = bounds[c->rank + 1];
  c->shard_planned = true;
  c->kernel_launches += 1;
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
