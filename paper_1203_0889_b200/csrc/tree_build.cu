// tree_build.cu — bit-exact adaptive octree build on the GPU (reference: build_tree,
// tree.cpp:52-119; compute_bounds, tree.cpp:10-23).
//
// Design: instead of the reference's per-cell BFS counting sort, every body descends the
// octree once with the SAME recursively computed FP64 centres the reference uses
// (octant_of, tree.cpp:45-48; child centre = parent + child_radius*(+-1), tree.cpp:102-103)
// and records its 21-level path as a 63-bit key. One stable radix sort of (key, input
// index) orders bodies by path; cells are then materialised level by level from key-digit
// boundaries (binary searches inside each splitting cell's sorted range), which reproduces
// the reference's BFS numbering (level-contiguous, children in octant order, empty octants
// skipped). A second sort by (leaf, input index) restores the reference's within-leaf order
// (stable counting sorts keep input order inside a leaf, tree.cpp:82-93).
// All FP64 arithmetic uses explicit __dadd_rn/__dmul_rn so nothing is contracted to FMA.
#include <cooperative_groups.h>
#include <cub/cub.cuh>

#include "context.cuh"

namespace fmmb {
namespace {

constexpr int kLevels = FMM_MAX_LEVEL;  // 21 levels -> 63 key bits
constexpr double kMarginFactor = 1.0 + 1e-6;  // tree.cpp:21 (evaluated exactly at compile time)
constexpr double kMinHalfSide = 0.5;          // tree.hpp:17

__device__ __forceinline__ double dmin_ref(double a, double b) { return b < a ? b : a; }  // cwiseMin
__device__ __forceinline__ double dmax_ref(double a, double b) { return a < b ? b : a; }  // cwiseMax

// ---- compute_bounds: block partials then one finishing block ----------------------------
__global__ void k_bounds_partial(const double4* __restrict__ xyzq, int64_t n, double* __restrict__ part) {
  double lo[3] = {xyzq[0].x, xyzq[0].y, xyzq[0].z};
  double hi[3] = {lo[0], lo[1], lo[2]};
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double4 b = xyzq[i];
    lo[0] = dmin_ref(lo[0], b.x); lo[1] = dmin_ref(lo[1], b.y); lo[2] = dmin_ref(lo[2], b.z);
    hi[0] = dmax_ref(hi[0], b.x); hi[1] = dmax_ref(hi[1], b.y); hi[2] = dmax_ref(hi[2], b.z);
  }
  __shared__ double s[6][32];
  for (int d = 0; d < 3; ++d) {
    for (int o = 16; o > 0; o >>= 1) {
      lo[d] = dmin_ref(lo[d], __shfl_xor_sync(0xffffffffu, lo[d], o));
      hi[d] = dmax_ref(hi[d], __shfl_xor_sync(0xffffffffu, hi[d], o));
    }
  }
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0)
    for (int d = 0; d < 3; ++d) { s[d][w] = lo[d]; s[3 + d][w] = hi[d]; }
  __syncthreads();
  if (threadIdx.x == 0) {
    const int nw = blockDim.x >> 5;
    for (int k = 1; k < nw; ++k)
      for (int d = 0; d < 3; ++d) {
        s[d][0] = dmin_ref(s[d][0], s[d][k]);
        s[3 + d][0] = dmax_ref(s[3 + d][0], s[3 + d][k]);
      }
    for (int d = 0; d < 6; ++d) part[blockIdx.x * 6 + d] = s[d][0];
  }
}

// Finishes the reduction (one block) and evaluates the Domain formula of tree.cpp:19-21.
__global__ void k_bounds_final(const double* __restrict__ part, int nparts, double* __restrict__ dom) {
  __shared__ double s[6][256];
  double lo[3] = {part[0], part[1], part[2]}, hi[3] = {part[3], part[4], part[5]};
  for (int k = threadIdx.x; k < nparts; k += blockDim.x)
    for (int d = 0; d < 3; ++d) {
      lo[d] = dmin_ref(lo[d], part[6 * k + d]);
      hi[d] = dmax_ref(hi[d], part[6 * k + 3 + d]);
    }
  for (int d = 0; d < 3; ++d) {
    s[d][threadIdx.x] = lo[d];
    s[3 + d][threadIdx.x] = hi[d];
  }
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o)
      for (int d = 0; d < 3; ++d) {
        s[d][threadIdx.x] = dmin_ref(s[d][threadIdx.x], s[d][threadIdx.x + o]);
        s[3 + d][threadIdx.x] = dmax_ref(s[3 + d][threadIdx.x], s[3 + d][threadIdx.x + o]);
      }
    __syncthreads();
  }
  if (threadIdx.x != 0) return;
  for (int d = 0; d < 3; ++d) {
    lo[d] = s[d][0];
    hi[d] = s[3 + d][0];
  }
  for (int d = 0; d < 3; ++d) dom[d] = __dmul_rn(0.5, __dadd_rn(lo[d], hi[d]));
  double ext = __dadd_rn(hi[0], -lo[0]);
  ext = dmax_ref(ext, __dadd_rn(hi[1], -lo[1]));  // (hi - lo).maxCoeff()
  ext = dmax_ref(ext, __dadd_rn(hi[2], -lo[2]));
  const double extent_half = __dmul_rn(0.5, ext);
  const double h = __dmul_rn(extent_half, kMarginFactor);
  dom[3] = h < kMinHalfSide ? kMinHalfSide : h;  // std::max(h, kMinHalfSide)
}

// ---- per-body octant descent (octant_of with recursive centres) ------------------------
__global__ void k_keys(const double4* __restrict__ xyzq, int64_t n, const double* __restrict__ dom,
                       uint64_t* __restrict__ keys, int32_t* __restrict__ idx) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double4 b = xyzq[i];
  double cx = dom[0], cy = dom[1], cz = dom[2], r = dom[3];
  uint64_t key = 0;
#pragma unroll 1
  for (int l = 0; l < kLevels; ++l) {
    const double cr = __dmul_rn(0.5, r);
    const int ox = b.x >= cx, oy = b.y >= cy, oz = b.z >= cz;  // tree.cpp:45-48
    key = (key << 3) | (uint64_t)(ox | (oy << 1) | (oz << 2));
    cx = __dadd_rn(cx, ox ? cr : -cr);  // center + child_radius * (+-1), tree.cpp:102-103
    cy = __dadd_rn(cy, oy ? cr : -cr);
    cz = __dadd_rn(cz, oz ? cr : -cr);
    r = cr;
  }
  keys[i] = key;
  idx[i] = static_cast<int32_t>(i);
}

__device__ __forceinline__ int digit_at(uint64_t key, int child_level) {
  return static_cast<int>((key >> (3 * (kLevels - child_level))) & 7u);
}

// First index in [lo, hi) whose digit at child_level is >= d (digits are sorted there).
__device__ __forceinline__ int32_t lower_digit(const uint64_t* __restrict__ k, int32_t lo, int32_t hi,
                                               int child_level, int d) {
  while (lo < hi) {
    const int32_t mid = lo + ((hi - lo) >> 1);
    if (digit_at(k[mid], child_level) < d) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// Children of every cell of one level (warp per cell, grid-stride; the level's cell range is
// read from the device level table, so all levels queue without a host round trip): lanes 1..7
// binary-search the seven octant boundaries in parallel; bnd[9*k + o] = first body of octant o
// (bnd[9*k+8] = end).
__global__ void k_count_children(const int32_t* __restrict__ lev, int level, int n_crit, int sort_levels,
                                 const int32_t* __restrict__ bb, const int32_t* __restrict__ be,
                                 const uint64_t* __restrict__ skeys, int32_t* __restrict__ nchild,
                                 int32_t* __restrict__ bnd, int32_t* __restrict__ deeper) {
  const int32_t cbeg = lev[level], cend = lev[level + 1];
  const int lane = threadIdx.x & 31;
  const int32_t nw = (gridDim.x * blockDim.x) >> 5;
  for (int32_t k = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; cbeg + k < cend; k += nw) {
    const int32_t ci = cbeg + k;
    const int32_t b = bb[ci], e = be[ci];
    bool split = e - b > n_crit && level < kLevels;  // tree.cpp:78
    if (split && level >= sort_levels) {  // digits below the sorted ones: full sort needed
      if (lane == 0) *deeper = 1;
      split = false;
    }
    int32_t pos = e;
    if (split && lane >= 1 && lane <= 7) pos = lower_digit(skeys, b, e, level + 1, lane);
    if (lane == 0) pos = b;
    if (split && lane <= 8) bnd[9 * k + lane] = pos;
    const int32_t nxt = __shfl_down_sync(0xffffffffu, pos, 1);
    const unsigned nonempty = __ballot_sync(0xffffffffu, split && lane < 8 && nxt > pos);
    if (lane == 0) nchild[k] = __popc(nonempty);
  }
}

// next level's range: lev[level + 2] = lev[level + 1] + (children of this level), clamped to
// the cell capacity (overflow flagged; the build is then repeated with larger arrays)
__global__ void k_level_advance(int32_t* __restrict__ lev, int level, const int32_t* __restrict__ offs, int64_t cap,
                                int32_t* __restrict__ overflow) {
  const int32_t m = lev[level + 1] - lev[level];
  int64_t next = static_cast<int64_t>(lev[level + 1]) + offs[m];
  if (next > cap) {
    *overflow = 1;
    next = lev[level + 1];
  }
  lev[level + 2] = static_cast<int32_t>(next);
}

// Materialises the children of one level (grid-stride); offs = exclusive scan of nchild.
__global__ void k_write_children(const int32_t* __restrict__ lev, int level, int64_t cap,
                                 const int32_t* __restrict__ nchild, const int32_t* __restrict__ offs,
                                 const int32_t* __restrict__ bnd, int32_t* __restrict__ c_level,
                                 uint64_t* __restrict__ c_key, double4* __restrict__ c_cr,
                                 int32_t* __restrict__ bb, int32_t* __restrict__ be,
                                 int32_t* __restrict__ cb, int32_t* __restrict__ cc,
                                 int32_t* __restrict__ par) {
  const int32_t cbeg = lev[level], cend = lev[level + 1], next_begin = cend;
  for (int32_t ci = cbeg + blockIdx.x * blockDim.x + threadIdx.x; ci < cend; ci += gridDim.x * blockDim.x) {
  const int k = ci - cbeg;
  if (nchild[k] == 0) continue;
  if (static_cast<int64_t>(next_begin) + offs[k] + nchild[k] > cap) continue;  // overflow: flagged
  const double4 pc = c_cr[ci];
  const uint64_t pkey = c_key[ci];
  const double cr = __dmul_rn(0.5, pc.w);
  int32_t out = next_begin + offs[k];
  cb[ci] = out;
  cc[ci] = nchild[k];
  for (int o = 0; o < 8; ++o) {
    const int32_t start = bnd[9 * k + o], stop = bnd[9 * k + o + 1];
    if (stop > start) {
      c_level[out] = level + 1;
      c_key[out] = (pkey << 3) | (uint64_t)o;
      c_cr[out] = make_double4(__dadd_rn(pc.x, (o & 1) ? cr : -cr), __dadd_rn(pc.y, (o & 2) ? cr : -cr),
                               __dadd_rn(pc.z, (o & 4) ? cr : -cr), cr);
      bb[out] = start;
      be[out] = stop;
      cb[out] = 0;
      cc[out] = 0;
      par[out] = ci;
      ++out;
    }
  }
  }
}

// All levels in ONE cooperative launch (grid barriers between the phases of a level) instead of
// six launches per level (memset, count, scan init, scan over the whole cell capacity, write,
// advance: 25-30 us per level whatever its size; C2's 7 levels were half of its 0.43 ms build).
// Per level: each CTA takes a contiguous block of the level's cells, its warps count the children
// of their cells (same octant-boundary searches as k_count_children) and the CTA publishes its
// children total; after the barrier every CTA sums the totals of the CTAs before it, scans its own
// cells and materialises their children (same code as k_write_children), and CTA 0 sets the next
// level's range. The loop ends at the first level without cells.
#ifndef FMM_BUILD_COOP
#define FMM_BUILD_COOP 1
#endif
constexpr int kCoopThreads = 256;
__global__ void __launch_bounds__(kCoopThreads)
k_build_levels(int32_t* __restrict__ lev, int n_crit, int sort_levels, int64_t cap, const uint64_t* __restrict__ skeys,
               int32_t* __restrict__ nchild, int32_t* __restrict__ bnd, int32_t* __restrict__ part,
               int32_t* __restrict__ deeper, int32_t* __restrict__ overflow, int32_t* __restrict__ c_level,
               uint64_t* __restrict__ c_key, double4* __restrict__ c_cr, int32_t* __restrict__ bb,
               int32_t* __restrict__ be, int32_t* __restrict__ cb, int32_t* __restrict__ cc, int32_t* __restrict__ par) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  using Reduce = cub::BlockReduce<int, kCoopThreads>;
  using Scan = cub::BlockScan<int, kCoopThreads>;
  __shared__ union {
    typename Reduce::TempStorage red;
    typename Scan::TempStorage scan;
  } tmp;
  __shared__ int s_base, s_total;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  constexpr int kWarps = kCoopThreads / 32;
  int level = 0;
  for (; level <= kLevels; ++level) {
    // plain loads: lev is written inside this kernel (no read-only path)
    const int32_t cbeg = *(volatile int32_t*)&lev[level], cend = *(volatile int32_t*)&lev[level + 1];
    const int32_t m = cend - cbeg;
    if (m <= 0) break;  // uniform over the grid
    const int32_t cpb = (m + static_cast<int32_t>(gridDim.x) - 1) / static_cast<int32_t>(gridDim.x);
    const int32_t k0 = min(m, static_cast<int32_t>(blockIdx.x) * cpb), k1 = min(m, k0 + cpb);
    // ---- phase 1: children of the CTA's cells (warp per cell)
    int mine = 0;
    for (int32_t k = k0 + w; k < k1; k += kWarps) {
      const int32_t ci = cbeg + k;
      const int32_t b = bb[ci], e = be[ci];
      bool split = e - b > n_crit && level < kLevels;  // tree.cpp:78
      if (split && level >= sort_levels) {  // digits below the sorted ones: full sort needed
        if (lane == 0) *deeper = 1;
        split = false;
      }
      int32_t pos = e;
      if (split && lane >= 1 && lane <= 7) pos = lower_digit(skeys, b, e, level + 1, lane);
      if (lane == 0) pos = b;
      if (split && lane <= 8) bnd[9 * k + lane] = pos;
      const int32_t nxt = __shfl_down_sync(0xffffffffu, pos, 1);
      const unsigned nonempty = __ballot_sync(0xffffffffu, split && lane < 8 && nxt > pos);
      if (lane == 0) {
        nchild[k] = __popc(nonempty);
        mine += __popc(nonempty);
      }
    }
    const int btot = Reduce(tmp.red).Sum(mine);
    if (tid == 0) part[blockIdx.x] = btot;
    grid.sync();
    // ---- phase 2: offsets (CTAs before this one + a scan of the own cells), children, next range
    int before = 0, all = 0;
    for (int b = tid; b < static_cast<int>(gridDim.x); b += kCoopThreads) {
      const int v = *(volatile int32_t*)&part[b];
      all += v;
      before += b < static_cast<int>(blockIdx.x) ? v : 0;
    }
    __syncthreads();
    const int rb = Reduce(tmp.red).Sum(before);
    __syncthreads();
    const int ra = Reduce(tmp.red).Sum(all);
    if (tid == 0) {
      s_base = rb;
      s_total = ra;
    }
    __syncthreads();
    int carry = s_base;
    const int32_t next_begin = cend;
    for (int32_t kk = k0; kk < k1; kk += kCoopThreads) {
      const int32_t k = kk + tid;
      const int nc = k < k1 ? nchild[k] : 0;
      int ex, agg;
      Scan(tmp.scan).ExclusiveSum(nc, ex, agg);
      if (nc > 0 && static_cast<int64_t>(next_begin) + carry + ex + nc <= cap) {  // else: overflow, flagged below
        const int32_t ci = cbeg + k;
        const double4 pc = c_cr[ci];
        const uint64_t pkey = c_key[ci];
        const double cr = __dmul_rn(0.5, pc.w);
        int32_t out = next_begin + carry + ex;
        cb[ci] = out;
        cc[ci] = nc;
        for (int o = 0; o < 8; ++o) {
          const int32_t start = bnd[9 * k + o], stop = bnd[9 * k + o + 1];
          if (stop > start) {
            c_level[out] = level + 1;
            c_key[out] = (pkey << 3) | (uint64_t)o;
            c_cr[out] = make_double4(__dadd_rn(pc.x, (o & 1) ? cr : -cr), __dadd_rn(pc.y, (o & 2) ? cr : -cr),
                                     __dadd_rn(pc.z, (o & 4) ? cr : -cr), cr);
            bb[out] = start;
            be[out] = stop;
            cb[out] = 0;
            cc[out] = 0;
            par[out] = ci;
            ++out;
          }
        }
      }
      carry += agg;
      __syncthreads();
    }
    if (blockIdx.x == 0 && tid == 0) {
      int64_t next = static_cast<int64_t>(cend) + s_total;
      if (next > cap) {
        *overflow = 1;
        next = cend;
      }
      lev[level + 2] = static_cast<int32_t>(next);
    }
    grid.sync();
  }
  // the levels after the last one are empty (the host looks for the first level without children)
  if (blockIdx.x == 0 && tid == 0)
    for (int l = level; l <= kLevels; ++l) lev[l + 2] = lev[level + 1];
}

__global__ void k_init_root(const double* __restrict__ dom, int32_t n, int32_t* c_level, uint64_t* c_key,
                            double4* c_cr, int32_t* bb, int32_t* be, int32_t* cb, int32_t* cc, int32_t* par) {
  c_level[0] = 0;
  c_key[0] = 0;
  c_cr[0] = make_double4(dom[0], dom[1], dom[2], dom[3]);
  bb[0] = 0;
  be[0] = n;
  cb[0] = 0;
  cc[0] = 0;
  par[0] = -1;
}

// Leaf-of-body map (warp per leaf) and, optionally, the (leaf begin, input index) composite
// key of the global fallback sort.
__global__ void k_leaf_map(const int32_t* __restrict__ leaves, int64_t nleaves, const int32_t* __restrict__ bb,
                           const int32_t* __restrict__ be, const int32_t* __restrict__ sidx,
                           int32_t* __restrict__ leaf_of_body, uint64_t* __restrict__ ckey) {
  const int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= nleaves) return;
  const int32_t leaf = leaves[w];
  const int32_t b = bb[leaf], e = be[leaf];
  for (int32_t i = b + lane; i < e; i += 32) {
    leaf_of_body[i] = leaf;
    if (ckey) ckey[i] = ((uint64_t)(uint32_t)b << 32) | (uint32_t)sidx[i];
  }
}

// Within-leaf input order (tree.cpp:82-93 keeps input order inside every cell): rank sort of
// the leaf's input indices (distinct), warp per leaf, leaves up to kRankMax bodies. Also writes
// leaf_of_body. Larger leaves (level-21 overflow only) raise *big for the global fallback.
constexpr int kRankMax = 1024;
__global__ void __launch_bounds__(128)
k_leaf_sort(const int32_t* __restrict__ leaves, const int64_t* __restrict__ d_nleaves, const int32_t* __restrict__ bb,
            const int32_t* __restrict__ be, const int32_t* __restrict__ sidx, int32_t* __restrict__ perm,
            int32_t* __restrict__ leaf_of_body, int32_t* __restrict__ big) {
  __shared__ int32_t sv[4][kRankMax];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t wid = blockIdx.x * 4ll + w;
  if (wid >= *d_nleaves) return;  // launched for every cell: the leaf count stays on the device
  const int32_t leaf = leaves[wid];
  const int32_t b = bb[leaf], e = be[leaf], n = e - b;
  for (int32_t i = lane; i < n; i += 32) leaf_of_body[b + i] = leaf;
  if (n > kRankMax) {
    if (lane == 0) atomicExch(big, 1);
    return;
  }
  for (int32_t i = lane; i < n; i += 32) sv[w][i] = sidx[b + i];
  __syncwarp();
  for (int32_t i = lane; i < n; i += 32) {
    const int32_t v = sv[w][i];
    int32_t r = 0;
    for (int32_t j = 0; j < n; ++j) r += sv[w][j] < v;
    perm[b + r] = v;
  }
}

__global__ void k_perm_from_ckey(const uint64_t* __restrict__ ckey, int64_t n, int32_t* __restrict__ perm) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) perm[i] = static_cast<int32_t>(ckey[i] & 0xffffffffu);
}

__global__ void k_gather(const double4* __restrict__ in, const int32_t* __restrict__ perm,
                         const int32_t* __restrict__ leaf_of_body, const double4* __restrict__ c_cr,
                         int64_t n, double4* __restrict__ bodies, float4* __restrict__ bodyf,
                         float4* __restrict__ bodyl) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  FMM_CHECK(perm[i] >= 0 && perm[i] < n && leaf_of_body[i] >= 0 && leaf_of_body[i] < FMM_LIM(ncells),
            "k_gather: permutation / leaf index out of range");
  const double4 b = in[perm[i]];
  bodies[i] = b;
  const double4 c = c_cr[leaf_of_body[i]];
  const double dx = b.x - c.x, dy = b.y - c.y, dz = b.z - c.z;
  const float fx = static_cast<float>(dx), fy = static_cast<float>(dy), fz = static_cast<float>(dz);
  bodyf[i] = make_float4(fx, fy, fz, static_cast<float>(b.w));
  // hi + lo carries ~48 bits of the offset: the P2P near tiles form exact close-pair differences
  bodyl[i] = make_float4(static_cast<float>(dx - fx), static_cast<float>(dy - fy), static_cast<float>(dz - fz), 0.f);
}

__global__ void k_flag_leaves(const int32_t* __restrict__ cc, int64_t ncells, int32_t* __restrict__ flag) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < ncells) flag[i] = cc[i] == 0;
}

template <class T>
void grow_preserve(fmm_ctx* c, DBuf<T>& buf, size_t used, size_t need) {
  if (need <= buf.cap) return;  // steady state: no allocation
  T* old = buf.p;
  size_t want = need * 2 + 1024;
  T* fresh = nullptr;
  CK(cudaMalloc(&fresh, want * sizeof(T)));
  if (old && used) CK(cudaMemcpyAsync(fresh, old, used * sizeof(T), cudaMemcpyDeviceToDevice, c->stream));
  if (old) {
    CK(cudaStreamSynchronize(c->stream));
    CK(cudaFree(old));
  }
  buf.p = fresh;
  buf.cap = want;
}

int bits_for(uint64_t v) {
  int b = 1;
  while (b < 64 && (v >> b)) ++b;
  return b;
}

}  // namespace

void* temp_storage(fmm_ctx* c, size_t bytes) { return c->tmp.ensure(bytes > 0 ? bytes : 1); }
void* temp_storage2(fmm_ctx* c, size_t bytes) { return c->tmp2.ensure(bytes > 0 ? bytes : 1); }

void build_tree(fmm_ctx* c) {
  if (!c->have_bodies) fail(FMM_ERR_STATE, "build_tree: no bodies set");
  const int64_t n = c->N;
  if (n <= 0) fail(FMM_ERR_EMPTY_INPUT, "empty input");
  if (c->cfg.n_crit < 1) fail(FMM_ERR_NCRIT, "n_crit must be >= 1");
  if (n >= (int64_t(1) << 31)) fail(FMM_ERR_UNSUPPORTED, "more than 2^31-1 bodies");
  cudaStream_t s = c->stream;
  int64_t* hp = c->hpin;

  // 1. compute_bounds
  const int nparts = 592;  // 4 x 148 SMs
  double* part = c->small.ensure(nparts * 6 + 8);
  double* dom = part + nparts * 6;
  k_bounds_partial<<<nparts, 256, 0, s>>>(c->xyzq_in.p, n, part);
  k_bounds_final<<<1, 256, 0, s>>>(part, nparts, dom);
  CK_LAUNCH("k_bounds");
  CK(cudaMemcpyAsync(hp + 32, dom, 4 * sizeof(double), cudaMemcpyDeviceToHost, s));

  // 2. keys by octant descent, 3. stable radix sort (key, index)
  uint64_t* keys = c->keys_a.ensure(n);
  int32_t* idx = c->idx_a.ensure(n);
  k_keys<<<ceil_div(n, 256), 256, 0, s>>>(c->xyzq_in.p, n, dom, keys, idx);
  CK_LAUNCH("k_keys");
  uint64_t* skeys = c->keys_b.ensure(n);
  int32_t* sidx = c->idx_b.ensure(n);
  // The stable sort only needs the digits of the levels the tree will have: with the previous
  // build's depth D known, sort the top 3(D+1) key bits (C2: 18 bits, 3 passes instead of 8);
  // bodies with equal top digits keep input order, which is the reference's order inside a leaf
  // (stable partitions, tree.cpp:80-98). A cell that would need a deeper split triggers a full
  // sort and rebuild. Sharded runs keep the full sort (their partition keys compare full keys).
  int sort_levels = (c->world > 1 || !c->depth_known) ? kLevels : std::min(kLevels, c->last_depth + 1);
  auto sort_keys = [&]() {
    const int begin_bit = 3 * (kLevels - sort_levels);
    size_t tbytes = 0;
    CK(cub::DeviceRadixSort::SortPairs(nullptr, tbytes, keys, skeys, idx, sidx, (int)n, begin_bit, 3 * kLevels, s));
    CK(cub::DeviceRadixSort::SortPairs(temp_storage(c, tbytes), tbytes, keys, skeys, idx, sidx, (int)n, begin_bit,
                                       3 * kLevels, s));
    c->kernel_launches += 1;
  };
  sort_keys();
  if (c->world > 1) {  // partition reuse maps Morton boundaries onto this tree (shard.cu)
    CK(cudaMemcpyAsync(c->body_keys.ensure(n), skeys, n * sizeof(uint64_t), cudaMemcpyDeviceToDevice, s));
    c->body_keys_valid = true;
  } else {
    c->body_keys_valid = false;
  }

  // 4. level-by-level cell materialisation, queued in batches without host round trips: the
  // level ranges live in a device table; the host reads it once per batch (one batch covers the
  // previous build's depth + 2 levels, so a steady sequence of steps syncs once).
  const int64_t want_cap = std::max<int64_t>(4096, 16 * n / std::max(1, c->cfg.n_crit) + 1024);
  int32_t* dlev = reinterpret_cast<int32_t*>(c->bnd_lev.ensure(FMM_MAX_LEVEL + 5));
  int32_t* overflow = dlev + FMM_MAX_LEVEL + 3;
  int32_t* deeper = dlev + FMM_MAX_LEVEL + 4;
  int level = 0;
  int64_t ncells = 1;
  int launches = 4;
  for (int attempt = 0;; ++attempt) {
    const int64_t cap = std::max<int64_t>(want_cap, static_cast<int64_t>(c->c_level.cap));
    auto ensure_cells = [&](size_t need) {
      grow_preserve(c, c->c_level, 0, need);
      grow_preserve(c, c->c_key, 0, need);
      grow_preserve(c, c->c_cr, 0, need);
      grow_preserve(c, c->c_body_begin, 0, need);
      grow_preserve(c, c->c_body_end, 0, need);
      grow_preserve(c, c->c_child_begin, 0, need);
      grow_preserve(c, c->c_child_count, 0, need);
      grow_preserve(c, c->c_parent, 0, need);
    };
    ensure_cells(cap);
    const int64_t ccap = std::min<int64_t>(static_cast<int64_t>(c->c_level.cap), static_cast<int64_t>(c->c_parent.cap));
    int32_t* nchild = c->i32_a.ensure(ccap + 1);
    int32_t* offs = c->i32_b.ensure(ccap + 1);
    int32_t* bnd = c->bnd.ensure(9 * (size_t)ccap + 9);
    size_t sb = 0;
    CK(cub::DeviceScan::ExclusiveSum(nullptr, sb, nchild, offs, (int)(ccap + 1), s));
    void* scan_tmp = temp_storage(c, sb);
    {
      int32_t h0[3] = {0, 1, 0};
      CK(cudaMemcpyAsync(dlev, h0, 2 * sizeof(int32_t), cudaMemcpyHostToDevice, s));
      CK(cudaMemsetAsync(overflow, 0, 2 * sizeof(int32_t), s));
    }
    k_init_root<<<1, 1, 0, s>>>(dom, (int32_t)n, c->c_level.p, c->c_key.p, c->c_cr.p, c->c_body_begin.p,
                                c->c_body_end.p, c->c_child_begin.p, c->c_child_count.p, c->c_parent.p);
    CK_LAUNCH("k_init_root");
    int32_t hlev[FMM_MAX_LEVEL + 5];
    int done_level = -1;  // last level whose children have been counted
    bool finished = false, over = false;
    int batch = std::max(2, c->last_depth + 2);
    bool coop = FMM_BUILD_COOP && c->build_coop_ok;
    if (coop) {
      static std::atomic<int> coop_blocks{0};  // CTAs per SM of k_build_levels (same on every B200)
      if (coop_blocks.load() == 0) {
        int nb = 0, supported = 0;
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_build_levels, kCoopThreads, 0));
        CK(cudaDeviceGetAttribute(&supported, cudaDevAttrCooperativeLaunch, c->cfg.device));
        coop_blocks.store(supported && nb > 0 ? std::min(nb, 4) : -1);
      }
      if (coop_blocks.load() < 0) {
        coop = false;
        c->build_coop_ok = false;
      } else {
        int sms = 148;
        CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->cfg.device));
        const int grid = sms * coop_blocks.load();
        int32_t* part = c->i32_b.p;  // offs is unused on this path: per-CTA children totals
        int32_t* lev_p = dlev;
        int n_crit = c->cfg.n_crit, sl = sort_levels;
        int64_t cap64 = ccap;
        const uint64_t* skeys_p = skeys;
        int32_t *cl = c->c_level.p, *bbp = c->c_body_begin.p, *bep = c->c_body_end.p, *cbp = c->c_child_begin.p,
                *ccp = c->c_child_count.p, *parp = c->c_parent.p;
        uint64_t* ck = c->c_key.p;
        double4* ccr = c->c_cr.p;
        void* args[] = {&lev_p, &n_crit, &sl, &cap64, &skeys_p, &nchild, &bnd, &part, &deeper, &overflow, &cl, &ck,
                        &ccr, &bbp, &bep, &cbp, &ccp, &parp};
        const cudaError_t le = cudaLaunchCooperativeKernel((const void*)k_build_levels, dim3(grid), dim3(kCoopThreads),
                                                           args, 0, s);
        if (le != cudaSuccess) {  // e.g. the device cannot hold the grid right now: the per-level path
          cudaGetLastError();
          coop = false;
          c->build_coop_ok = false;
        } else {
          launches += 1;
        }
      }
    }
    if (coop) batch = kLevels + 1;  // every level is done: one read of the level table
    while (!finished) {
      const int l_end = std::min(done_level + batch, kLevels);
      for (int L = done_level + 1; L <= l_end && !coop; ++L) {
        CK(cudaMemsetAsync(nchild, 0, (ccap + 1) * sizeof(int32_t), s));
        k_count_children<<<148 * 16, 128, 0, s>>>(dlev, L, c->cfg.n_crit, sort_levels, c->c_body_begin.p,
                                                  c->c_body_end.p, skeys, nchild, bnd, deeper);
        CK_LAUNCH("k_count_children");
        CK(cub::DeviceScan::ExclusiveSum(scan_tmp, sb, nchild, offs, (int)(ccap + 1), s));
        k_write_children<<<148 * 8, 128, 0, s>>>(dlev, L, ccap, nchild, offs, bnd, c->c_level.p, c->c_key.p,
                                                 c->c_cr.p, c->c_body_begin.p, c->c_body_end.p, c->c_child_begin.p,
                                                 c->c_child_count.p, c->c_parent.p);
        CK_LAUNCH("k_write_children");
        k_level_advance<<<1, 1, 0, s>>>(dlev, L, offs, ccap, overflow);
        CK_LAUNCH("k_level_advance");
        launches += 5;
      }
      CK(cudaMemcpyAsync(hlev, dlev, (FMM_MAX_LEVEL + 5) * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
      CK(cudaStreamSynchronize(s));
      over = hlev[FMM_MAX_LEVEL + 3] != 0;
      if (over || hlev[FMM_MAX_LEVEL + 4] != 0) break;
      // the tree ends at the first level that has no children (or at kLevels)
      for (int L = done_level + 1; L <= l_end; ++L) {
        if (hlev[L + 2] == hlev[L + 1] || L == kLevels) {
          finished = true;
          level = L;
          break;
        }
      }
      done_level = l_end;
    }
    if (!over && hlev[FMM_MAX_LEVEL + 4] != 0) {  // deeper than the partial sort: full sort, rebuild
      sort_levels = kLevels;
      sort_keys();
      --attempt;
      continue;
    }
    if (!over) {
      // cells exist at levels 0..level (level = the first level without children)
      for (int l = 0; l <= level + 1; ++l) c->level_start[l] = hlev[l];
      ncells = hlev[level + 1];
      while (level > 0 && hlev[level + 1] == hlev[level]) --level;  // deepest non-empty level
      break;
    }
    if (attempt > 0) fail(FMM_ERR_CUDA, "tree build: cell overflow after regrow");
    ensure_cells(static_cast<size_t>(ccap) * 4);  // regrow and rebuild
  }
  c->last_depth = level;
  c->depth_known = true;
  if (ncells >= (int64_t(1) << 31) - 16) fail(FMM_ERR_UNSUPPORTED, "too many cells");
  for (int l = level + 2; l < FMM_MAX_LEVEL + 2; ++l) c->level_start[l] = static_cast<int32_t>(ncells);
  c->ncells = ncells;
  c->depth = level;
  const double* hdom = reinterpret_cast<const double*>(hp + 32);
  c->center[0] = hdom[0];
  c->center[1] = hdom[1];
  c->center[2] = hdom[2];
  c->half_side = hdom[3];

  // 5. leaves (ascending cell index)
  int32_t* flag = c->i32_a.ensure(ncells);
  k_flag_leaves<<<ceil_div(ncells, 256), 256, 0, s>>>(c->c_child_count.p, ncells, flag);
  int32_t* leaves = c->leaves.ensure(ncells);
  int64_t* nsel = c->d_counters.ensure(4);
  {
    size_t sb = 0;
    cub::CountingInputIterator<int32_t> it(0);
    CK(cub::DeviceSelect::Flagged(nullptr, sb, it, flag, leaves, nsel, (int)ncells, s));
    CK(cub::DeviceSelect::Flagged(temp_storage(c, sb), sb, it, flag, leaves, nsel, (int)ncells, s));
  }
  int32_t* big = reinterpret_cast<int32_t*>(nsel + 1);
  CK(cudaMemsetAsync(big, 0, sizeof(int32_t), s));
  c->wl = leaves;
  c->shard_planned = false;

  // 6. within-leaf input order: rank sort per leaf (grid over the cells, the leaf count read on
  //    the device, so the leaf count and the big-leaf flag come back in one host read); global
  //    (leaf, index) sort only when a level-21 leaf exceeds kRankMax bodies
  int32_t* leaf_of_body = c->leaf_of_body.ensure(n);
  int32_t* perm = c->perm.ensure(n);
  k_leaf_sort<<<ceil_div(ncells, 4), 128, 0, s>>>(leaves, nsel, c->c_body_begin.p, c->c_body_end.p, sidx, perm,
                                                  leaf_of_body, big);
  CK_LAUNCH("k_leaf_sort");
  CK(cudaMemcpyAsync(hp, nsel, sizeof(int64_t) + sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  c->nleaves = hp[0];
  c->nwl = c->nleaves;
  launches += 3;
  if (*reinterpret_cast<int32_t*>(hp + 1)) {
    uint64_t* ckey = c->keys_a.ensure(n);
    k_leaf_map<<<ceil_div(c->nleaves * 32, 256), 256, 0, s>>>(leaves, c->nleaves, c->c_body_begin.p,
                                                                c->c_body_end.p, sidx, leaf_of_body, ckey);
    uint64_t* ckey2 = c->keys_b.ensure(n);  // sorted keys are no longer needed
    const int end_bit = 32 + bits_for(static_cast<uint64_t>(n));
    size_t sb = 0;
    CK(cub::DeviceRadixSort::SortKeys(nullptr, sb, ckey, ckey2, (int)n, 0, end_bit, s));
    CK(cub::DeviceRadixSort::SortKeys(temp_storage(c, sb), sb, ckey, ckey2, (int)n, 0, end_bit, s));
    k_perm_from_ckey<<<ceil_div(n, 256), 256, 0, s>>>(ckey2, n, perm);
    CK_LAUNCH("k_perm_from_ckey");
    launches += 3;
  }
  c->kernel_launches += launches;
  c->have_tree = true;
  set_check_limits(c, s);
  k_gather<<<ceil_div(n, 256), 256, 0, s>>>(c->xyzq_in.p, perm, leaf_of_body, c->c_cr.p, n, c->bodies.ensure(n),
                                            c->bodyf.ensure(n), c->bodyl.ensure(n));
  CK_LAUNCH("k_gather");
  c->kernel_launches += 1;
}

namespace {
__global__ void k_unpermute(const int32_t* __restrict__ perm, int64_t n, const double* __restrict__ phi,
                            const double* __restrict__ acc, double* __restrict__ phi_in, double* __restrict__ acc_in) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int64_t j = perm[i];
  phi_in[j] = phi[i];
  if (acc_in) {
    acc_in[3 * j] = acc[3 * i];
    acc_in[3 * j + 1] = acc[3 * i + 1];
    acc_in[3 * j + 2] = acc[3 * i + 2];
  }
}
}  // namespace

void unpermute_results(fmm_ctx* c, double* phi_in, double* acc_in) {
  k_unpermute<<<ceil_div(c->N, 256), 256, 0, c->stream>>>(c->perm.p, c->N, c->phi.p, c->acc.p, phi_in, acc_in);
  CK_LAUNCH("k_unpermute");
}

namespace {
// tree reuse: every body (new position, kept permutation) must lie in its leaf's closed cube
__global__ void k_check_inside(const double4* __restrict__ in, const int32_t* __restrict__ perm,
                               const int32_t* __restrict__ leaf_of_body, const double4* __restrict__ cr, int64_t n,
                               int* __restrict__ outside) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double4 b = in[perm[i]], c = cr[leaf_of_body[i]];
  if (!(fabs(b.x - c.x) <= c.w && fabs(b.y - c.y) <= c.w && fabs(b.z - c.z) <= c.w)) *outside = 1;
}
}  // namespace

bool refit_bodies(fmm_ctx* c) {
  cudaStream_t s = c->stream;
  const int64_t n = c->N;
  int* flag = reinterpret_cast<int*>(c->d_counters.p + 8);
  CK(cudaMemsetAsync(flag, 0, sizeof(int), s));
  k_check_inside<<<ceil_div(n, 256), 256, 0, s>>>(c->xyzq_in.p, c->perm.p, c->leaf_of_body.p, c->c_cr.p, n, flag);
  CK_LAUNCH("k_check_inside");
  int* h = reinterpret_cast<int*>(c->hpin + 8);
  CK(cudaMemcpyAsync(h, flag, sizeof(int), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  c->kernel_launches += 1;
  if (*h) return false;
  k_gather<<<ceil_div(n, 256), 256, 0, s>>>(c->xyzq_in.p, c->perm.p, c->leaf_of_body.p, c->c_cr.p, n, c->bodies.p,
                                            c->bodyf.p, c->bodyl.p);
  CK_LAUNCH("k_gather");
  c->kernel_launches += 1;
  return true;
}

void gather_bodies(fmm_ctx* c) {
  cudaStream_t s = c->stream;
  const int64_t n = c->N;
  int32_t* leaf_of_body = c->leaf_of_body.ensure(n);
  k_leaf_map<<<ceil_div(c->nleaves * 32, 256), 256, 0, s>>>(c->leaves.p, c->nleaves, c->c_body_begin.p,
                                                              c->c_body_end.p, nullptr, leaf_of_body, nullptr);
  set_check_limits(c, s);
  k_gather<<<ceil_div(n, 256), 256, 0, s>>>(c->xyzq_in.p, c->perm.p, leaf_of_body, c->c_cr.p, n,
                                            c->bodies.ensure(n), c->bodyf.ensure(n), c->bodyl.ensure(n));
  CK_LAUNCH("k_gather");
  c->kernel_launches += 2;
}

}  // namespace fmmb

// ---- single-operator entry points ---------------------------------------------------------
namespace fmmb {
namespace {
// morton_key (tree.cpp:25-39): floor-based interleave (tests-only API of the reference).
__global__ void k_morton(int64_t count, const double* __restrict__ p3, double cx, double cy, double cz,
                         double half, int level, uint64_t* __restrict__ out) {
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= count) return;
  const uint64_t cells = uint64_t(1) << level;
  const double inv_cell = __ddiv_rn(static_cast<double>(cells), __dmul_rn(2.0, half));
  const double c[3] = {cx, cy, cz};
  uint64_t key = 0;
  for (int axis = 0; axis < 3; ++axis) {
    const double offset = __dadd_rn(p3[3 * k + axis], -__dadd_rn(c[axis], -half));
    long long idx = static_cast<long long>(floor(__dmul_rn(offset, inv_cell)));
    if (idx < 0) idx = 0;
    if (idx > static_cast<long long>(cells) - 1) idx = static_cast<long long>(cells) - 1;
    for (int bit = 0; bit < level; ++bit) key |= ((static_cast<uint64_t>(idx) >> bit) & 1u) << (3 * bit + axis);
  }
  out[k] = key;
}
}  // namespace

void op_bounds(const double* xyzq, int64_t n, double* center3, double* half_side) {
  if (n <= 0) fail(FMM_ERR_EMPTY_INPUT, "empty input");
  double4* d = nullptr;
  double* part = nullptr;
  CK(cudaMalloc(&d, n * sizeof(double4)));
  CK(cudaMalloc(&part, (592 * 6 + 8) * sizeof(double)));
  CK(cudaMemcpy(d, xyzq, n * sizeof(double4), cudaMemcpyHostToDevice));
  k_bounds_partial<<<592, 256>>>(d, n, part);
  k_bounds_final<<<1, 32>>>(part, 592, part + 592 * 6);
  CK_LAUNCH("op_bounds");
  double h[4];
  CK(cudaMemcpy(h, part + 592 * 6, sizeof(h), cudaMemcpyDeviceToHost));
  cudaFree(d);
  cudaFree(part);
  center3[0] = h[0];
  center3[1] = h[1];
  center3[2] = h[2];
  *half_side = h[3];
}

void op_morton(int64_t count, const double* p3, const double* center3, double half_side, int level,
               uint64_t* out) {
  if (level < 0 || level > FMM_MAX_LEVEL) fail(FMM_ERR_LEVEL_OVERFLOW, "level overflow");
  if (count <= 0) return;
  double* d = nullptr;
  uint64_t* o = nullptr;
  CK(cudaMalloc(&d, count * 3 * sizeof(double)));
  CK(cudaMalloc(&o, count * sizeof(uint64_t)));
  CK(cudaMemcpy(d, p3, count * 3 * sizeof(double), cudaMemcpyHostToDevice));
  k_morton<<<ceil_div(count, 128), 128>>>(count, d, center3[0], center3[1], center3[2], half_side, level, o);
  CK_LAUNCH("op_morton");
  CK(cudaMemcpy(out, o, count * sizeof(uint64_t), cudaMemcpyDeviceToHost));
  cudaFree(d);
  cudaFree(o);
}
}  // namespace fmmb
