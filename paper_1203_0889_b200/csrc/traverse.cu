// traverse.cu — dual tree traversal on the GPU emitting the reference's M2L / P2P lists
// bit-exactly (reference: mac, traversal.cpp:8-13; split_target_side / process_pair,
// traversal.hpp:49-94; dual_tree_traverse, traversal.hpp:118-133).
//
// The reference's emitted multiset is a pure function of (tree, theta, mutual) and is
// independent of queue order and of the drain threshold Q (acceptance.cpp:99-123). The GPU
// therefore replaces the FIFO queue by level-synchronous frontier expansion: every pair of
// the frontier is examined by one thread (process_pair), emits an M2L or P2P pair or pushes
// its child pairs to the next frontier. Output slots come from exclusive scans, so the
// emission order is deterministic. The lists are then grouped into CSR by target with a
// radix sort on (target, source), i.e. ascending sources within each target.
// The MAC is evaluated with __dmul_rn/__dadd_rn/__dsqrt_rn: no FMA contraction, exactly
// std::sqrt(3.0)*(rt+rs) < theta*sqrt((dx*dx+dy*dy)+dz*dz).
#include <cub/cub.cuh>

#include "context.cuh"
#include "tma.cuh"

namespace fmmb {
namespace {

constexpr double kSqrt3 = 1.7320508075688772;  // std::sqrt(3.0), correctly rounded

__device__ __forceinline__ bool mac_exact(const double4 t, const double4 s, double theta) {
  const double sum_r = __dmul_rn(kSqrt3, __dadd_rn(t.w, s.w));
  const double dx = __dadd_rn(t.x, -s.x), dy = __dadd_rn(t.y, -s.y), dz = __dadd_rn(t.z, -s.z);
  const double d2 = __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
  return sum_r < __dmul_rn(theta, __dsqrt_rn(d2));
}

// Same decision without the FP64 square root whenever it is unambiguous: both sides are
// compared squared with a 1e-12 relative guard band (the rounding of sqrt and of the products
// is below 1e-15), and only pairs inside the band take the exact path above.
__device__ __forceinline__ bool mac_fast(const double4 t, const double4 s, double theta, double theta2) {
  const double sum_r = __dmul_rn(kSqrt3, __dadd_rn(t.w, s.w));
  const double dx = __dadd_rn(t.x, -s.x), dy = __dadd_rn(t.y, -s.y), dz = __dadd_rn(t.z, -s.z);
  const double d2 = __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
  const double a2 = sum_r * sum_r, q = theta2 * d2;
  if (a2 < q * (1.0 - 1e-12)) return true;
  if (a2 > q * (1.0 + 1e-12)) return false;
  return sum_r < __dmul_rn(theta, __dsqrt_rn(d2));
}

// Outcome of process_pair: kind 0 = M2L, 1 = P2P, 2 = split target, 3 = split source,
// 4 = mutual self split. nchild = number of pushed pairs.
__device__ __forceinline__ void classify(const int2 pr, const double4* __restrict__ cr,
                                         const int32_t* __restrict__ cc, double theta, double theta2,
                                         int mutual, int& kind, int& nchild) {
  const double4 t = cr[pr.x], s = cr[pr.y];
  const int tc = cc[pr.x], sc = cc[pr.y];
  if (mac_fast(t, s, theta, theta2)) { kind = 0; nchild = 0; return; }
  if (tc == 0 && sc == 0) { kind = 1; nchild = 0; return; }
  if (mutual && pr.x == pr.y) { kind = 4; nchild = tc * (tc + 1) / 2; return; }
  bool split_t;
  if (tc == 0) split_t = false;            // traversal.hpp:53-57
  else if (sc == 0) split_t = true;
  else if (t.w != s.w) split_t = t.w > s.w;
  else split_t = pr.x <= pr.y;
  kind = split_t ? 2 : 3;
  nchild = split_t ? tc : sc;
}

// One frontier step (frontier level L): every pair is classified (process_pair) and emits an
// M2L or P2P key or pushes its child pairs to level L+1. The launch does not know the frontier
// size: it reads it from the level counters written by the previous launch, so all levels are
// queued back to back without a host round trip. A persistent grid takes chunks of pairs in
// ticket order. Each chunk's output offsets come from a chained (decoupled look-back, warp-wide)
// scan over the chunks of the level, so the emission order is a pure function of the frontier
// order: deterministic, level by level, and the lists only need a STABLE sort on the target bits
// to become deterministic CSR (64-bit keys, more than 2^16 cells or mutual mode: 3 instead of 5
// radix passes; 32-bit keys: 2 instead of 4). The look-back state of a chunk is one 16-byte word
// (values and state together), so a hop is one load. FMM_TRAV_ORDERED32/64 = 0 select the older
// scheme instead: slots reserved by one atomic per chunk and counter and a full (target, source)
// sort (it was the cheaper one for 32-bit keys while a hop cost two dependent loads: C2 traversal
// 1.11 against 1.03 ms now). Output that would exceed a buffer's capacity is dropped and flagged;
// the host then grows the buffers and reruns the traversal.
// Counters (ctr): [0] M2L total, [1] P2P total, [2] overflow flag, [4 + L] frontier size of
// level L (level 0 = the root pair), [64 + L] chunk tickets of level L.
constexpr int kStepThreads = 256;
// pairs per thread: 2 (512-pair chunks; with the one-load look-back hop larger chunks no longer
// pay: 4 pairs per thread C3 traversal 2.89 ms, 2 -> 2.80, 1 -> 3.09); 8 CTAs of 256 threads per
// SM: the kernel is latency bound (ncu at C3's heavy levels: issue 32-40 %, stalls: the CTA barrier
// behind the look-back warp ~40 %, cell / spill loads ~40 %), so occupancy beats the register
// spill it costs (tools/trav_ab.sh: 6 / 5 / 4 CTAs/SM are within +-2 % at C3 / C5 and 3-18 % slower at C2)
#ifndef FMM_TRAV_ORDERED64  // 64-bit keys: ordered look-back emission (1) or atomic slots + full sort (0)
#define FMM_TRAV_ORDERED64 1
#endif
#ifndef FMM_TRAV_ORDERED32  // 32-bit keys: ordered look-back emission + target-only sort (1) or atomic slots + full sort (0)
#define FMM_TRAV_ORDERED32 1
#endif
#ifndef FMM_STEP_PER64
#define FMM_STEP_PER64 2
#endif
#ifndef FMM_STEP_PER32
#define FMM_STEP_PER32 2
#endif
#ifndef FMM_STEP_MINB
#define FMM_STEP_MINB 8
#endif
template <class KeyT>
constexpr int step_per() { return sizeof(KeyT) == 8 ? FMM_STEP_PER64 : FMM_STEP_PER32; }
template <class KeyT>
constexpr int step_chunk() { return kStepThreads * step_per<KeyT>(); }
constexpr int kTicketBase = 64;

__device__ __forceinline__ uint32_t ld_acquire(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}
#ifndef FMM_TRAV_PACKED_LB
#define FMM_TRAV_PACKED_LB 1
#endif
// 16-byte relaxed loads / stores of an aligned {u64, u64} (a single transaction: the two halves
// are always observed together, as CUB's decoupled look-back tile status relies on)
__device__ __forceinline__ void ld_relaxed16(const ulonglong2* p, unsigned long long& x, unsigned long long& y) {
  asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];\n" : "=l"(x), "=l"(y) : "l"(p) : "memory");
}
__device__ __forceinline__ void st_relaxed16(ulonglong2* p, unsigned long long x, unsigned long long y) {
  asm volatile("st.relaxed.gpu.global.v2.u64 [%0], {%1, %2};\n" ::"l"(p), "l"(x), "l"(y) : "memory");
}
__device__ __forceinline__ void st_release(uint32_t* p, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
}

// One frontier pair: load, classify, (sharded) filter the kept target children; returns the packed
// per-pair counts M2L (bits 0..20) | P2P (21..41) | children (42..63)
__device__ __forceinline__ unsigned long long step_classify(bool in_range, const int2* __restrict__ fr, int64_t i,
                                                            const double4* __restrict__ cr,
                                                            const int32_t* __restrict__ cc,
                                                            const int32_t* __restrict__ cb, double theta, double theta2,
                                                            int mutual, int filter, const int32_t* __restrict__ bb,
                                                            const int32_t* __restrict__ be, int32_t tb0, int32_t tb1,
                                                            int2& pr, int& kind, int& nch) {
  kind = -1;
  nch = 0;
  pr = make_int2(0, 0);
  if (!in_range) return 0ull;
  pr = fr[i];
  FMM_CHECK(pr.x >= 0 && pr.x < FMM_LIM(ncells) && pr.y >= 0 && pr.y < FMM_LIM(ncells),
            "k_step: frontier pair outside the cell array");
  classify(pr, cr, cc, theta, theta2, mutual, kind, nch);
  if (filter && kind == 2) {  // sharded: keep only target children meeting [tb0, tb1)
    const int32_t b = cb[pr.x];
    int kept = 0;
    for (int q = 0; q < nch; ++q) kept += (bb[b + q] < tb1 && be[b + q] > tb0) ? 1 : 0;
    nch = kept;
  }
  return kind == 0 ? 1ull : kind == 1 ? (1ull << 21) : (static_cast<unsigned long long>(nch) << 42);
}

// Emits one classified pair at the running offsets (om, op, oc), which it advances; returns true
// if an output would pass its buffer's capacity (dropped; the run is then flagged and repeated).
template <class KeyT>
__device__ __forceinline__ bool step_scatter(const int2 pr, int kind, int nch, int64_t& om, int64_t& op, int64_t& oc,
                                             int sbits, KeyT* __restrict__ m2l_keys, KeyT* __restrict__ p2p_keys,
                                             int2* __restrict__ next, int64_t cap_m, int64_t cap_p, int64_t cap_f,
                                             const int32_t* __restrict__ cb, const int32_t* __restrict__ cc, int filter,
                                             const int32_t* __restrict__ bb, const int32_t* __restrict__ be, int32_t tb0,
                                             int32_t tb1) {
  bool over = false;
  const KeyT key = static_cast<KeyT>(((uint64_t)(uint32_t)pr.x << sbits) | (uint32_t)pr.y);
  if (kind == 0) {
    if (om < cap_m) m2l_keys[om] = key; else over = true;
    ++om;
  } else if (kind == 1) {
    if (op < cap_p) p2p_keys[op] = key; else over = true;
    ++op;
  } else if (kind >= 2) {
    // children past the frontier capacity are dropped (and the run flagged), but every slot
    // below the capacity is written, so a truncated frontier still holds only valid pairs
    if (oc + nch > cap_f) over = true;
    if (kind == 2) {
      const int32_t b = cb[pr.x];
      if (filter) {
        int64_t q = oc;
        for (int k = 0; k < cc[pr.x]; ++k)
          if (bb[b + k] < tb1 && be[b + k] > tb0) {
            if (q < cap_f) next[q] = make_int2(b + k, pr.y);
            ++q;
          }
      } else {
        for (int k = 0; k < nch; ++k)
          if (oc + k < cap_f) next[oc + k] = make_int2(b + k, pr.y);
      }
    } else if (kind == 3) {
      const int32_t b = cb[pr.y];
      for (int k = 0; k < nch; ++k)
        if (oc + k < cap_f) next[oc + k] = make_int2(pr.x, b + k);
    } else {
      const int32_t b = cb[pr.x], m = cc[pr.x];
      int64_t q = oc;
      for (int a = 0; a < m; ++a)
        for (int c = a; c < m; ++c) {
          if (q < cap_f) next[q] = make_int2(b + a, b + c);
          ++q;
        }
    }
    oc += nch;
  }
  return over;
}

template <class KeyT>
__global__ void __launch_bounds__(kStepThreads, FMM_STEP_MINB)
k_step(int level, const int2* __restrict__ fr, const double4* __restrict__ cr, const int32_t* __restrict__ cc,
       const int32_t* __restrict__ cb, double theta, double theta2, int mutual, int sbits, KeyT* __restrict__ m2l_keys,
       KeyT* __restrict__ p2p_keys, int2* __restrict__ next, unsigned long long* __restrict__ ctr, int64_t cap_m,
       int64_t cap_p, int64_t cap_f, const int32_t* __restrict__ bb, const int32_t* __restrict__ be, int32_t tb0,
       int32_t tb1, int filter, uint32_t epoch, uint32_t* __restrict__ lb_flag,
       unsigned long long* __restrict__ lb_val) {
  using Scan = cub::BlockScan<unsigned long long, kStepThreads>;
  // 64-bit keys (more than 2^16 cells, or mutual mode): ordered emission by look-back, and the
  // lists only need a stable sort on the target bits; 32-bit keys: atomic slot reservation (the
  // full (target, source) sort canonicalises them; measured cheaper at C2)
  constexpr bool kOrdered = sizeof(KeyT) == 8 ? FMM_TRAV_ORDERED64 != 0 : FMM_TRAV_ORDERED32 != 0;
  constexpr int kStepPer = step_per<KeyT>();
  constexpr int kStepChunk = step_chunk<KeyT>();
  __shared__ typename Scan::TempStorage scan_tmp;
  __shared__ unsigned long long sbase[3];
  __shared__ int64_t s_chunk;
  // a frontier that overflowed its buffer is only partially written (the run is flagged and
  // repeated with larger buffers): read no further than the capacity
  const int64_t n = min(static_cast<int64_t>(ctr[4 + level]), cap_f);
  const unsigned long long base_m = ctr[0], base_p = ctr[1];  // totals of the previous levels
  const uint32_t f_agg = 2u * epoch, f_inc = 2u * epoch + 1u;
  // CTAs beyond the level's chunk count leave without taking a ticket: a small frontier (the
  // first and last levels hold a few thousand pairs) otherwise pays ~1 200 serialised atomics on
  // one counter, 5-8 us per level
  if (static_cast<int64_t>(blockIdx.x) * kStepChunk >= n) return;
  for (;;) {
    if (threadIdx.x == 0) s_chunk = static_cast<int64_t>(atomicAdd(&ctr[kTicketBase + level], 1ull));
    __syncthreads();
    const int64_t ch = s_chunk;
    const int64_t c0 = ch * kStepChunk;
    if (c0 >= n) break;  // uniform over the block
    int kind[kStepPer], nch[kStepPer];
    int2 pr[kStepPer];
    // packed per-thread counts: M2L (bits 0..20) | P2P (21..41) | children (42..63)
    unsigned long long mine = 0;
#pragma unroll
    for (int j = 0; j < kStepPer; ++j) {
      const int64_t i = c0 + j * kStepThreads + threadIdx.x;
      mine += step_classify(i < n, fr, i, cr, cc, cb, theta, theta2, mutual, filter, bb, be, tb0, tb1, pr[j], kind[j],
                            nch[j]);
    }
    unsigned long long excl, tot;
    Scan(scan_tmp).ExclusiveSum(mine, excl, tot);
    if (!kOrdered) {
      if (threadIdx.x == 0) {
        const unsigned long long tm = tot & 0x1fffffull, tp = (tot >> 21) & 0x1fffffull, tc = tot >> 42;
        sbase[0] = tm ? atomicAdd(&ctr[0], tm) : 0ull;
        sbase[1] = tp ? atomicAdd(&ctr[1], tp) : 0ull;
        sbase[2] = tc ? atomicAdd(&ctr[4 + level + 1], tc) : 0ull;
      }
    } else if (threadIdx.x < 32) {
      // chunk aggregate: (M2L | P2P << 32) and children; the exclusive prefix over the earlier
      // chunks of this level by a warp-wide decoupled look-back, 32 predecessors per step
      // (chunk ch only waits for chunks with lower tickets, all running or done: no deadlock)
      const int lane = threadIdx.x;
      unsigned long long tot_b = __shfl_sync(0xffffffffu, tot, 0);
      const unsigned long long a01 = (tot_b & 0x1fffffull) | (((tot_b >> 21) & 0x1fffffull) << 32);
      const unsigned long long a2 = tot_b >> 42;
      unsigned long long p01 = 0, p2 = 0;
#if FMM_TRAV_PACKED_LB
      // One 16-byte word per chunk, {M2L | P2P << 32, children | state << 40}, read and written
      // whole: a hop of the look-back is ONE load per lane (the state tags the values it travels
      // with), where separate flag and value arrays cost two dependent L2 round trips per hop;
      // the first wave of a large level resolves its ~1 200 chunks 32 per hop.
      ulonglong2* lb = reinterpret_cast<ulonglong2*>(lb_val);
      const unsigned long long t_agg = f_agg & 0xffffffu, t_inc = f_inc & 0xffffffu;
      if (ch > 0) {
        if (lane == 0) st_relaxed16(&lb[ch], a01, a2 | (t_agg << 40));
        for (int64_t top = ch - 1;; top -= 32) {
          const int64_t j = top - lane;
          unsigned long long x = 0, y = t_inc << 40;  // lanes before chunk 0: an empty inclusive prefix
          if (j >= 0) {
            do {
              ld_relaxed16(&lb[j], x, y);
            } while ((y >> 40) != t_agg && (y >> 40) != t_inc);
          }
          const unsigned inc = __ballot_sync(0xffffffffu, (y >> 40) == t_inc);
          const int stop = inc ? __ffs(inc) - 1 : 31;  // nearest lane holding an inclusive prefix
          unsigned long long v01 = 0, v2 = 0;
          if (j >= 0 && lane <= stop) {
            v01 = x;
            v2 = y & 0xffffffffffull;
          }
#pragma unroll
          for (int d = 16; d > 0; d >>= 1) {
            v01 += __shfl_xor_sync(0xffffffffu, v01, d);
            v2 += __shfl_xor_sync(0xffffffffu, v2, d);
          }
          p01 += v01;
          p2 += v2;
          if (inc) break;
        }
      }
      if (lane == 0) {
        st_relaxed16(&lb[ch], p01 + a01, (p2 + a2) | (t_inc << 40));
#else
      if (ch > 0) {
        if (lane == 0) {
          lb_val[4 * ch + 0] = a01;
          lb_val[4 * ch + 1] = a2;
          st_release(&lb_flag[ch], f_agg);
        }
        for (int64_t top = ch - 1;; top -= 32) {
          const int64_t j = top - lane;
          uint32_t f = f_inc;  // lanes before chunk 0 count as an empty inclusive prefix
          if (j >= 0) {
            do {
              f = ld_acquire(&lb_flag[j]);
            } while (f != f_agg && f != f_inc);
          }
          const unsigned inc = __ballot_sync(0xffffffffu, f == f_inc);
          const int stop = inc ? __ffs(inc) - 1 : 31;  // nearest lane holding an inclusive prefix
          unsigned long long v01 = 0, v2 = 0;
          if (j >= 0 && lane <= stop) {
            const int o = f == f_inc ? 2 : 0;
            v01 = __ldcg(&lb_val[4 * j + o]);
            v2 = __ldcg(&lb_val[4 * j + o + 1]);
          }
#pragma unroll
          for (int d = 16; d > 0; d >>= 1) {
            v01 += __shfl_xor_sync(0xffffffffu, v01, d);
            v2 += __shfl_xor_sync(0xffffffffu, v2, d);
          }
          p01 += v01;
          p2 += v2;
          if (inc) break;
        }
      }
      if (lane == 0) {
        lb_val[4 * ch + 2] = p01 + a01;
        lb_val[4 * ch + 3] = p2 + a2;
        st_release(&lb_flag[ch], f_inc);
#endif
        sbase[0] = base_m + (p01 & 0xffffffffull);
        sbase[1] = base_p + (p01 >> 32);
        sbase[2] = p2;
        if (c0 + kStepChunk >= n) {  // the level's last chunk: totals for the next launch
          const unsigned long long i01 = p01 + a01;
          ctr[0] = base_m + (i01 & 0xffffffffull);
          ctr[1] = base_p + (i01 >> 32);
          ctr[4 + level + 1] = p2 + a2;
        }
      }
    }
    __syncthreads();
    int64_t om = static_cast<int64_t>(sbase[0] + (excl & 0x1fffffull));
    int64_t op = static_cast<int64_t>(sbase[1] + ((excl >> 21) & 0x1fffffull));
    int64_t oc = static_cast<int64_t>(sbase[2] + (excl >> 42));
    bool over = false;
#pragma unroll
    for (int j = 0; j < kStepPer; ++j)
      over |= step_scatter<KeyT>(pr[j], kind[j], nch[j], om, op, oc, sbits, m2l_keys, p2p_keys, next, cap_m, cap_p, cap_f,
                                 cb, cc, filter, bb, be, tb0, tb1);
    if (over) ctr[2] = 1ull;
    __syncthreads();  // sbase / scan storage / s_chunk reuse
  }
}


// Pipelined frontier step (ordered emission only): eight worker warps and one RESOLVER warp per
// CTA. The workers classify chunk k into a shared-memory stage, scan their counts and hand the
// chunk total to the resolver, which runs the look-back for chunk k while the workers classify
// chunk k + 1; the workers then scatter chunk k from its stage. In k_step all eight warps wait at
// a CTA barrier behind the look-back warp (ncu, C3's heavy levels: ~40 % of the stall samples);
// here the look-back of a chunk overlaps the next chunk's classification and still starts right
// after the chunk's scan, so the prefixes of later chunks are not delayed. Two stages; mbarriers
// scanned[s] (workers -> resolver) and resolved[s] (resolver -> workers); named barrier 1 among
// the 256 worker threads.
#ifndef FMM_STEP_PIPE
#define FMM_STEP_PIPE 1
#endif
#ifndef FMM_STEP_PIPE_MINB
#define FMM_STEP_PIPE_MINB 7
#endif
constexpr int kPipeWorkers = 256;
constexpr int kPipeThreads = kPipeWorkers + 32;
__device__ __forceinline__ void bar_workers() { asm volatile("bar.sync 1, %0;\n" ::"r"(kPipeWorkers) : "memory"); }

template <class KeyT>
__global__ void __launch_bounds__(kPipeThreads, FMM_STEP_PIPE_MINB)
k_step_pipe(int level, const int2* __restrict__ fr, const double4* __restrict__ cr, const int32_t* __restrict__ cc,
            const int32_t* __restrict__ cb, double theta, double theta2, int mutual, int sbits,
            KeyT* __restrict__ m2l_keys, KeyT* __restrict__ p2p_keys, int2* __restrict__ next,
            unsigned long long* __restrict__ ctr, int64_t cap_m, int64_t cap_p, int64_t cap_f,
            const int32_t* __restrict__ bb, const int32_t* __restrict__ be, int32_t tb0, int32_t tb1, int filter,
            uint32_t epoch, unsigned long long* __restrict__ lb_val) {
  constexpr int kPer = step_per<KeyT>();
  constexpr int kChunk = kPipeWorkers * kPer;
  struct Stage {
    int2 pr[kChunk];
    int16_t kn[kChunk];                  // kind (low 4 bits, -1 -> 15) | children << 4
    unsigned long long excl[kPipeWorkers];
    unsigned long long tot;
    long long ch;                        // ticket (workers)
    long long rch;                       // chunk index for the resolver, -1 = no more chunks
  };
  __shared__ Stage st[2];
  __shared__ unsigned long long sbase[2][3];
  __shared__ unsigned long long wsum[kPipeWorkers / 32];
  __shared__ __align__(8) uint64_t scanned[2], resolved[2];
  const int tid = threadIdx.x, lane = tid & 31;
  const int64_t n = min(static_cast<int64_t>(ctr[4 + level]), cap_f);
  const unsigned long long base_m = ctr[0], base_p = ctr[1];  // totals of the previous levels
  if (static_cast<int64_t>(blockIdx.x) * kChunk >= n) return;
  if (tid == 0) {
    for (int b = 0; b < 2; ++b) {
      mbar_init(&scanned[b], 1);
      mbar_init(&resolved[b], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();

  if (tid >= kPipeWorkers) {  // ---- resolver warp
    ulonglong2* lb = reinterpret_cast<ulonglong2*>(lb_val);
    const unsigned long long t_agg = (2u * epoch) & 0xffffffu, t_inc = (2u * epoch + 1u) & 0xffffffu;
    for (unsigned k = 0;; ++k) {
      const int s = k & 1;
      mbar_wait(&scanned[s], (k >> 1) & 1u);
      const int64_t ch = st[s].rch;
      if (ch < 0) return;
      const unsigned long long tot = st[s].tot;
      const unsigned long long a01 = (tot & 0x1fffffull) | (((tot >> 21) & 0x1fffffull) << 32);
      const unsigned long long a2 = tot >> 42;
      unsigned long long p01 = 0, p2 = 0;
      if (ch > 0) {
        if (lane == 0) st_relaxed16(&lb[ch], a01, a2 | (t_agg << 40));
        for (int64_t top = ch - 1;; top -= 32) {
          const int64_t j = top - lane;
          unsigned long long x = 0, y = t_inc << 40;  // lanes before chunk 0: an empty inclusive prefix
          if (j >= 0) {
            do {
              ld_relaxed16(&lb[j], x, y);
            } while ((y >> 40) != t_agg && (y >> 40) != t_inc);
          }
          const unsigned inc = __ballot_sync(0xffffffffu, (y >> 40) == t_inc);
          const int stop = inc ? __ffs(inc) - 1 : 31;
          unsigned long long v01 = 0, v2 = 0;
          if (j >= 0 && lane <= stop) {
            v01 = x;
            v2 = y & 0xffffffffffull;
          }
#pragma unroll
          for (int d = 16; d > 0; d >>= 1) {
            v01 += __shfl_xor_sync(0xffffffffu, v01, d);
            v2 += __shfl_xor_sync(0xffffffffu, v2, d);
          }
          p01 += v01;
          p2 += v2;
          if (inc) break;
        }
      }
      if (lane == 0) {
        st_relaxed16(&lb[ch], p01 + a01, (p2 + a2) | (t_inc << 40));
        sbase[s][0] = base_m + (p01 & 0xffffffffull);
        sbase[s][1] = base_p + (p01 >> 32);
        sbase[s][2] = p2;
        if (ch * kChunk + kChunk >= n) {  // the level's last chunk: totals for the next launch
          const unsigned long long i01 = p01 + a01;
          ctr[0] = base_m + (i01 & 0xffffffffull);
          ctr[1] = base_p + (i01 >> 32);
          ctr[4 + level + 1] = p2 + a2;
        }
        mbar_arrive(&resolved[s]);
      }
      __syncwarp();
    }
  }

  // ---- worker warps
  const int w = tid >> 5;
  bool over = false, have_prev = false;
  for (unsigned k = 0;; ++k) {
    const int s = k & 1;
    // stage s was scattered in iteration k - 1 (as chunk k - 2) and the barrier closed it
    if (tid == 0) st[s].ch = static_cast<long long>(atomicAdd(&ctr[kTicketBase + level], 1ull));
    bar_workers();
    const int64_t ch = st[s].ch;
    const int64_t c0 = ch * kChunk;
    const bool active = c0 < n;  // uniform over the workers
    if (active) {
      unsigned long long mine = 0;
#pragma unroll
      for (int j = 0; j < kPer; ++j) {
        const int64_t i = c0 + j * kPipeWorkers + tid;
        int2 pr;
        int kind, nch;
        mine += step_classify(i < n, fr, i, cr, cc, cb, theta, theta2, mutual, filter, bb, be, tb0, tb1, pr, kind, nch);
        st[s].pr[j * kPipeWorkers + tid] = pr;
        st[s].kn[j * kPipeWorkers + tid] = static_cast<int16_t>((kind & 15) | (nch << 4));
      }
      // exclusive scan over the 256 workers: warp scan, warp totals through shared memory
      unsigned long long incl = mine;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const unsigned long long v = __shfl_up_sync(0xffffffffu, incl, d);
        if (lane >= d) incl += v;
      }
      if (lane == 31) wsum[w] = incl;
      bar_workers();
      unsigned long long before = 0, total = 0;
#pragma unroll
      for (int q = 0; q < kPipeWorkers / 32; ++q) {
        const unsigned long long v = wsum[q];
        before += q < w ? v : 0ull;
        total += v;
      }
      st[s].excl[tid] = before + incl - mine;
      if (tid == 0) {
        st[s].tot = total;
        st[s].rch = ch;
      }
    } else if (tid == 0) {
      st[s].rch = -1;  // tells the resolver to leave
    }
    bar_workers();  // the stage is complete (and wsum may be rewritten)
    if (tid == 0) mbar_arrive(&scanned[s]);
    if (have_prev) {  // scatter chunk k - 1 once its prefix is resolved
      const int sp = s ^ 1;
      mbar_wait(&resolved[sp], ((k - 1) >> 1) & 1u);
      const unsigned long long excl = st[sp].excl[tid];
      int64_t om = static_cast<int64_t>(sbase[sp][0] + (excl & 0x1fffffull));
      int64_t op = static_cast<int64_t>(sbase[sp][1] + ((excl >> 21) & 0x1fffffull));
      int64_t oc = static_cast<int64_t>(sbase[sp][2] + (excl >> 42));
#pragma unroll
      for (int j = 0; j < kPer; ++j) {
        const int2 pr = st[sp].pr[j * kPipeWorkers + tid];
        const int kn = st[sp].kn[j * kPipeWorkers + tid];
        int kind = kn & 15;
        if (kind == 15) kind = -1;
        over |= step_scatter<KeyT>(pr, kind, kn >> 4, om, op, oc, sbits, m2l_keys, p2p_keys, next, cap_m, cap_p, cap_f,
                                   cb, cc, filter, bb, be, tb0, tb1);
      }
    }
    if (!active) break;
    have_prev = true;
    bar_workers();  // every worker is done with stage s ^ 1 before the next iteration refills it
  }
  if (over) ctr[2] = 1ull;
}

template <class KeyT>
__global__ void k_pair_keys(const int2* __restrict__ pr, int64_t n, int sbits, KeyT* __restrict__ keys) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) keys[i] = static_cast<KeyT>(((uint64_t)(uint32_t)pr[i].x << sbits) | (uint32_t)pr[i].y);
}

// CSR from sorted (target, source) keys: sources, and offsets (targets tp+1..t start at i).
// Mutual mode: bit 63 marks a mirrored key (outside the sorted bit range, so carried along) and
// is written to `mir`; the all-ones key of the sorted range is a dropped slot (a self pair has
// no mirror) and sorts past every cell, so off[ncells] = the number of real entries.
constexpr uint64_t kMirrorBit = 1ull << 63;

// Four keys per thread: vector loads / stores and one neighbour load per four keys (one key per
// thread was issue-bound: 55 us for C2's 15.7 M M2L keys).
constexpr int kCsrPer = 4;
template <class KeyT>
__global__ void __launch_bounds__(256)
k_csr_from_keys(const KeyT* __restrict__ keys, int64_t n, int sbits, int64_t ncells,
                int64_t* __restrict__ off, int32_t* __restrict__ src, uint8_t* __restrict__ mir,
                int32_t* __restrict__ tgt) {
  const int64_t i0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) * kCsrPer;
  if (i0 > n) return;
  const uint64_t mask = (1ull << sbits) - 1, range = (1ull << (2 * sbits)) - 1;
  auto target_of = [&](uint64_t key) -> int64_t {
    const uint64_t k = key & range;
    return k == range ? ncells : static_cast<int64_t>(k >> sbits);
  };
  KeyT k[kCsrPer];
  if (i0 + kCsrPer <= n) {  // aligned: 16 or 32 bytes
    using V = std::conditional_t<sizeof(KeyT) == 4, uint4, ulonglong2>;
    constexpr int kPerV = sizeof(V) / sizeof(KeyT);
    const V* kv = reinterpret_cast<const V*>(keys + i0);
#pragma unroll
    for (int q = 0; q < kCsrPer / kPerV; ++q) reinterpret_cast<V*>(k)[q] = kv[q];
  } else {
#pragma unroll
    for (int j = 0; j < kCsrPer; ++j) k[j] = i0 + j < n ? keys[i0 + j] : KeyT(0);
  }
  int64_t tp = i0 > 0 ? target_of(static_cast<uint64_t>(keys[i0 - 1])) : -1;
  int32_t sv[kCsrPer], tv[kCsrPer];
#pragma unroll
  for (int j = 0; j < kCsrPer; ++j) {
    const int64_t i = i0 + j;
    if (i > n) break;
    const int64_t t = i < n ? target_of(static_cast<uint64_t>(k[j])) : ncells;
    sv[j] = static_cast<int32_t>(static_cast<uint64_t>(k[j]) & mask);
    tv[j] = static_cast<int32_t>(t);  // ncells for a dropped slot (past off[ncells])
    for (int64_t c = tp + 1; c <= t; ++c) off[c] = i;
    tp = t;
  }
  if (i0 + kCsrPer <= n) {
    *reinterpret_cast<int4*>(src + i0) = make_int4(sv[0], sv[1], sv[2], sv[3]);
    if (tgt) *reinterpret_cast<int4*>(tgt + i0) = make_int4(tv[0], tv[1], tv[2], tv[3]);
    if (mir) {
      uint32_t m = 0;
#pragma unroll
      for (int j = 0; j < kCsrPer; ++j) m |= static_cast<uint32_t>(static_cast<uint64_t>(k[j]) >> 63) << (8 * j);
      *reinterpret_cast<uint32_t*>(mir + i0) = m;
    }
  } else {
    for (int j = 0; j < kCsrPer && i0 + j < n; ++j) {
      src[i0 + j] = sv[j];
      if (tgt) tgt[i0 + j] = tv[j];
      if (mir) mir[i0 + j] = static_cast<uint8_t>(static_cast<uint64_t>(k[j]) >> 63);
    }
  }
}

// Mutual mode (traversal.hpp:76-84 emits each unordered pair once): out[0, n) = the emitted
// keys, out[n, 2n) = their mirrors (s, t) flagged with kMirrorBit, or the dropped-slot key for
// a self pair. The symmetrised list equals the non-mutual emission (test_traversal.cpp:182-210),
// so the target-owned M2L / P2P kernels run unchanged on it.
__global__ void k_mirror_keys(const uint64_t* __restrict__ in, int64_t n, int sbits, uint64_t* __restrict__ out) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint64_t mask = (1ull << sbits) - 1, k = in[i];
  const uint64_t t = k >> sbits, s = k & mask;
  out[i] = k;
  out[n + i] = t == s ? (1ull << (2 * sbits)) - 1 : ((s << sbits) | t | kMirrorBit);
}

// cells with a non-empty M2L list whose body range meets [b0, b1) (the rank's targets)
__global__ void k_flag_nonempty(const int64_t* __restrict__ off, int64_t ncells, const int32_t* __restrict__ bb,
                                const int32_t* __restrict__ be, int64_t b0, int64_t b1, int32_t* __restrict__ flag) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < ncells) flag[i] = off[i + 1] > off[i] && bb[i] < b1 && be[i] > b0;
}

int bits_for(uint64_t v) {
  int b = 1;
  while (b < 63 && (v >> b)) ++b;
  return b;
}

// Sorts packed (target, source) keys (2 * ceil(log2 ncells) bits) and splits them into CSR by
// target with ascending sources: the canonical form of the emitted multiset.
// Keys are 32-bit when 2 * ceil(log2 ncells) <= 32 (half the sort traffic), else 64-bit.
inline bool small_keys(int64_t ncells) { return 2 * bits_for(static_cast<uint64_t>(ncells)) <= 32; }
// mutual mode carries the mirror flag in bit 63: always 64-bit keys
inline bool keys32(const fmm_ctx* c) { return !c->cfg.mutual && !c->dbg_keys64 && small_keys(c->ncells); }

template <class KeyT>
void keys_to_csr(fmm_ctx* c, KeyT* keys, int64_t n, DBuf<int64_t>& off, DBuf<int32_t>& src, uint8_t* mir,
                 int32_t* tgt = nullptr, bool p2p_path = false) {
  // the P2P list uses the P2P preparation stream and scratch (it may overlap the M2L path)
  cudaStream_t s = p2p_path ? c->pstream : c->stream;
  const int64_t nc = c->ncells;
  off.ensure(nc + 1);
  src.ensure(n > 0 ? n : 1);
  if (n == 0) {
    CK(cudaMemsetAsync(off.p, 0, sizeof(int64_t) * (nc + 1), s));
    return;
  }
  const int sbits = bits_for(static_cast<uint64_t>(nc));
  KeyT* kb = reinterpret_cast<KeyT*>(p2p_path ? c->p2p_keys_b2.ensure(n) : c->keys_b.ensure(n));
  size_t sb = 0;
  // 64-bit keys come in a deterministic order (ordered emission / given pairs): a stable sort on
  // the target bits keeps it within each target; 32-bit keys: the full (target, source) sort
  const int b0 = (sizeof(KeyT) == 8 ? FMM_TRAV_ORDERED64 != 0 : FMM_TRAV_ORDERED32 != 0) ? sbits : 0;
  CK(cub::DeviceRadixSort::SortKeys(nullptr, sb, keys, kb, (int)n, b0, 2 * sbits, s));
  CK(cub::DeviceRadixSort::SortKeys(p2p_path ? temp_storage2(c, sb) : temp_storage(c, sb), sb, keys, kb, (int)n, b0,
                                    2 * sbits, s));
  k_csr_from_keys<<<ceil_div(ceil_div(n + 1, kCsrPer), 256), 256, 0, s>>>(kb, n, sbits, nc, off.p, src.p, mir, tgt);
  CK_LAUNCH("keys_to_csr");
  c->kernel_launches += 3;
}

}  // namespace

void lists_from_pairs(fmm_ctx* c, const int2* d_m2l, int64_t n_m2l, const int2* d_p2p, int64_t n_p2p) {
  const int sbits = bits_for(static_cast<uint64_t>(c->ncells));
  uint64_t* mk = c->m2l_keys.ensure(n_m2l + 1);
  uint64_t* pk = c->p2p_keys.ensure(n_p2p + 1);
  if (keys32(c)) {
    if (n_m2l) k_pair_keys<<<ceil_div(n_m2l, 256), 256, 0, c->stream>>>(d_m2l, n_m2l, sbits, (uint32_t*)mk);
    if (n_p2p) k_pair_keys<<<ceil_div(n_p2p, 256), 256, 0, c->stream>>>(d_p2p, n_p2p, sbits, (uint32_t*)pk);
  } else {
    if (n_m2l) k_pair_keys<<<ceil_div(n_m2l, 256), 256, 0, c->stream>>>(d_m2l, n_m2l, sbits, mk);
    if (n_p2p) k_pair_keys<<<ceil_div(n_p2p, 256), 256, 0, c->stream>>>(d_p2p, n_p2p, sbits, pk);
  }
  CK_LAUNCH("k_pair_keys");
  finish_lists(c, n_m2l, n_p2p);
}

void finish_lists(fmm_ctx* c, int64_t n_m2l, int64_t n_p2p) {
  cudaStream_t s = c->stream;
  c->n_m2l_emit = n_m2l;
  c->n_p2p_emit = n_p2p;
  // The P2P list and work list may be prepared on the second stream, concurrently with the M2L
  // list and kernel (evaluate with overlap, single rank, non-mutual: c->p2p_overlap). Sharded
  // runs plan from both lists and mutual runs read both lengths back: one stream.
  const bool split = c->p2p_overlap && c->world == 1 && !c->cfg.mutual;
  c->pstream = split ? c->stream3 : c->stream;
  if (split) {
    CK(cudaEventRecord(c->ev_lists, s));  // the emitted keys are complete
    CK(cudaStreamWaitEvent(c->pstream, c->ev_lists, 0));
  }
  if (c->cfg.mutual) {
    // symmetrise (emitted + mirrored), then the same canonical CSR; off[ncells] of each list is
    // its executed length (self pairs have no mirror), read back with the M2L target count
    const int sbits = bits_for(static_cast<uint64_t>(c->ncells));
    uint64_t* dm = c->mut_keys.ensure(2 * (n_m2l + n_p2p) + 2);
    uint64_t* dp = dm + 2 * n_m2l;
    if (n_m2l) k_mirror_keys<<<ceil_div(n_m2l, 256), 256, 0, s>>>(c->m2l_keys.p, n_m2l, sbits, dm);
    if (n_p2p) k_mirror_keys<<<ceil_div(n_p2p, 256), 256, 0, s>>>(c->p2p_keys.p, n_p2p, sbits, dp);
    CK_LAUNCH("k_mirror_keys");
    keys_to_csr(c, dm, 2 * n_m2l, c->m2l_off, c->m2l_src, c->m2l_mir.ensure(2 * n_m2l + 1));
    keys_to_csr(c, dp, 2 * n_p2p, c->p2p_off, c->p2p_src, c->p2p_mir.ensure(2 * n_p2p + 1),
                c->p2p_tgt.ensure(2 * n_p2p + 1), true);
    CK(cudaMemcpyAsync(c->hpin + 2, c->m2l_off.p + c->ncells, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(c->hpin + 3, c->p2p_off.p + c->ncells, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    n_m2l = c->hpin[2];
    n_p2p = c->hpin[3];
  } else if (keys32(c)) {
    keys_to_csr(c, reinterpret_cast<uint32_t*>(c->p2p_keys.p), n_p2p, c->p2p_off, c->p2p_src, nullptr,
                c->p2p_tgt.ensure(n_p2p + 1), true);
    keys_to_csr(c, reinterpret_cast<uint32_t*>(c->m2l_keys.p), n_m2l, c->m2l_off, c->m2l_src, nullptr);
  } else {
    keys_to_csr(c, c->p2p_keys.p, n_p2p, c->p2p_off, c->p2p_src, nullptr, c->p2p_tgt.ensure(n_p2p + 1), true);
    keys_to_csr(c, c->m2l_keys.p, n_m2l, c->m2l_off, c->m2l_src, nullptr);
  }
  c->n_m2l = n_m2l;
  c->n_p2p = n_p2p;
  // partition (sharded runs), then the M2L target list of this rank
  if (c->world > 1) {
    if (c->shard_from_plan) shard_assign(c);  // bounds already mapped from the kept plan
    else plan_shards(c);                      // full lists: plan from this step's costs
  } else {
    c->shard_b0 = 0;
    c->shard_b1 = c->N;
  }
  if (split) p2p_worklist_begin(c);  // queued on the second stream before the M2L host sync
  // p <= 6, one rank: the register M2L kernel takes a warp per CELL and leaves at once on an empty
  // list (nearly every cell has one: 37 440 of C2's 37 449), so the target list, its select and
  // the host read of its length are skipped (n_m2l_targets = -1: every cell)
  if (c->world == 1 && c->cfg.order <= 6) {
    c->n_m2l_targets = n_m2l > 0 ? -1 : 0;
    c->have_lists = true;
    if (!split) build_p2p_worklist(c);
    return;
  }
  int32_t* flag = c->i32_c.ensure(c->ncells);
  k_flag_nonempty<<<ceil_div(c->ncells, 256), 256, 0, s>>>(c->m2l_off.p, c->ncells, c->c_body_begin.p,
                                                           c->c_body_end.p, c->shard_b0, c->shard_b1, flag);
  CK_LAUNCH("k_flag_nonempty");
  int32_t* targets = c->m2l_targets.ensure(c->ncells);
  int64_t* nsel = c->d_counters.p + 1;
  size_t sb = 0;
  cub::CountingInputIterator<int32_t> it(0);
  CK(cub::DeviceSelect::Flagged(nullptr, sb, it, flag, targets, nsel, (int)c->ncells, s));
  CK(cub::DeviceSelect::Flagged(temp_storage(c, sb), sb, it, flag, targets, nsel, (int)c->ncells, s));
  int64_t* h = c->hpin;
  CK(cudaMemcpyAsync(h, nsel, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  c->n_m2l_targets = h[0];
  c->kernel_launches += 3;
  c->have_lists = true;
  if (!split) build_p2p_worklist(c);  // else finished by the caller (p2p_worklist_end)
}

void traverse(fmm_ctx* c) {
  if (!c->have_tree) fail(FMM_ERR_STATE, "traverse: no tree");
  set_check_limits(c, c->stream);
  const double theta = c->cfg.theta;
  if (!(theta > 0.0 && theta < 1.0)) fail(FMM_ERR_THETA, "theta must be in (0,1)");
  cudaStream_t s = c->stream;
  const int mutual = c->cfg.mutual ? 1 : 0;
  const int sbits = bits_for(static_cast<uint64_t>(c->ncells));
  const bool small = keys32(c);
  if (mutual && c->world > 1) fail(FMM_ERR_UNSUPPORTED, "mutual mode is not supported by the sharded traversal");
  // Every split descends the target or the source by one level (a mutual self split both), so
  // the frontier is empty after at most 2 * depth + 1 levels.
  const int nlev = 2 * c->depth + 2;
  if (4 + nlev + 1 > 60) fail(FMM_ERR_UNSUPPORTED, "traverse: tree too deep");
  unsigned long long* ctr = reinterpret_cast<unsigned long long*>(c->trav_ctr.ensure(128));
  unsigned long long* h = reinterpret_cast<unsigned long long*>(c->hpin);
  // first call: capacities from the cell count; afterwards the buffers keep their size
  const int64_t want_f = c->dbg_cap > 0 ? c->dbg_cap : std::max<int64_t>(c->ncells * 256, 1 << 16);
  const int64_t want_m = c->dbg_cap > 0 ? c->dbg_cap : std::max<int64_t>(c->ncells * 512, 1 << 16);
  const int64_t want_p = c->dbg_cap > 0 ? c->dbg_cap : std::max<int64_t>(c->nleaves * 256, 1 << 16);
  if (c->pairs_a.cap < static_cast<size_t>(want_f)) c->pairs_a.ensure(want_f);
  if (c->pairs_d.cap < static_cast<size_t>(want_f)) c->pairs_d.ensure(want_f);
  if (c->m2l_keys.cap < static_cast<size_t>(want_m)) c->m2l_keys.ensure(want_m);
  if (c->p2p_keys.cap < static_cast<size_t>(want_p)) c->p2p_keys.ensure(want_p);
  const int grid = 148 * (2048 / kStepThreads);
  const int2 root = make_int2(0, 0);
  // sharded steps after the first: targets restricted to the rank's range (kept plan)
  c->shard_from_plan = c->world > 1 && shard_bounds_from_plan(c);
  const int filter = c->shard_from_plan ? 1 : 0;
  const int32_t tb0 = static_cast<int32_t>(filter ? c->shard_b0 : 0);
  const int32_t tb1 = static_cast<int32_t>(filter ? c->shard_b1 : c->N);
  for (int attempt = 0;; ++attempt) {
    c->trav_regrows = attempt;
    const int64_t cap_f = static_cast<int64_t>(std::min(c->pairs_a.cap, c->pairs_d.cap));
    // KeyT buffers are uint64_t arrays; 32-bit keys use twice the count
    const int64_t cap_m = static_cast<int64_t>(c->m2l_keys.cap) * (small ? 2 : 1);
    const int64_t cap_p = static_cast<int64_t>(c->p2p_keys.cap) * (small ? 2 : 1);
    CK(cudaMemsetAsync(ctr, 0, 128 * sizeof(unsigned long long), s));
    // look-back state: one flag + 4 values per chunk of the largest frontier (flags zeroed on
    // (re)allocation only: every launch uses a fresh epoch)
    const int64_t nchunk = cap_f / std::min(step_chunk<uint32_t>(), step_chunk<uint64_t>()) + 2;
    if (c->lb_flag.cap < static_cast<size_t>(nchunk)) {
      c->lb_flag.ensure(nchunk);
      CK(cudaMemsetAsync(c->lb_flag.p, 0, sizeof(uint32_t) * c->lb_flag.cap, s));
    }
    // the packed words carry a 24-bit state (2 * epoch + {0, 1}): zeroed on (re)allocation and
    // when the epoch counter would wrap within this traversal
    const bool lb_grow = c->lb_val.cap < static_cast<size_t>(4 * nchunk);
    unsigned long long* lbv = reinterpret_cast<unsigned long long*>(c->lb_val.ensure(4 * nchunk));
    const bool lb_wrap = ((c->trav_epoch + nlev + 2) & 0x7fffffu) < static_cast<uint32_t>(nlev + 2);
    if (lb_grow || lb_wrap) {
      CK(cudaMemsetAsync(lbv, 0, sizeof(unsigned long long) * c->lb_val.cap, s));
      CK(cudaMemsetAsync(c->lb_flag.p, 0, sizeof(uint32_t) * c->lb_flag.cap, s));
      if (lb_wrap) c->trav_epoch = 0;  // the epochs of this traversal are 1 .. nlev: never state 0
    }
    const unsigned long long one = 1;
    CK(cudaMemcpyAsync(ctr + 4, &one, sizeof(one), cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(c->pairs_a.p, &root, sizeof(int2), cudaMemcpyHostToDevice, s));
    for (int L = 0; L < nlev; ++L) {
      const int2* fr = (L & 1) ? c->pairs_d.p : c->pairs_a.p;
      int2* nx = (L & 1) ? c->pairs_a.p : c->pairs_d.p;
      const uint32_t epoch = ++c->trav_epoch;
      constexpr bool kPipe32 = FMM_STEP_PIPE && FMM_TRAV_ORDERED32, kPipe64 = FMM_STEP_PIPE && FMM_TRAV_ORDERED64;
      const int pgrid = 148 * FMM_STEP_PIPE_MINB;
      if (small && kPipe32)
        k_step_pipe<<<pgrid, kPipeThreads, 0, s>>>(L, fr, c->c_cr.p, c->c_child_count.p, c->c_child_begin.p, theta,
                                                   theta * theta, mutual, sbits, (uint32_t*)c->m2l_keys.p,
                                                   (uint32_t*)c->p2p_keys.p, nx, ctr, cap_m, cap_p, cap_f,
                                                   c->c_body_begin.p, c->c_body_end.p, tb0, tb1, filter, epoch, lbv);
      else if (!small && kPipe64)
        k_step_pipe<<<pgrid, kPipeThreads, 0, s>>>(L, fr, c->c_cr.p, c->c_child_count.p, c->c_child_begin.p, theta,
                                                   theta * theta, mutual, sbits, c->m2l_keys.p, c->p2p_keys.p, nx, ctr,
                                                   cap_m, cap_p, cap_f, c->c_body_begin.p, c->c_body_end.p, tb0, tb1,
                                                   filter, epoch, lbv);
      else if (small)
        k_step<<<grid, kStepThreads, 0, s>>>(L, fr, c->c_cr.p, c->c_child_count.p, c->c_child_begin.p, theta,
                                             theta * theta, mutual, sbits, (uint32_t*)c->m2l_keys.p,
                                             (uint32_t*)c->p2p_keys.p, nx, ctr, cap_m, cap_p, cap_f,
                                             c->c_body_begin.p, c->c_body_end.p, tb0, tb1, filter, epoch,
                                             c->lb_flag.p, lbv);
      else
        k_step<<<grid, kStepThreads, 0, s>>>(L, fr, c->c_cr.p, c->c_child_count.p, c->c_child_begin.p, theta,
                                             theta * theta, mutual, sbits, c->m2l_keys.p, c->p2p_keys.p, nx, ctr,
                                             cap_m, cap_p, cap_f, c->c_body_begin.p, c->c_body_end.p, tb0, tb1,
                                             filter, epoch, c->lb_flag.p, lbv);
      CK_LAUNCH("k_step");
    }
    CK(cudaMemcpyAsync(h, ctr, (4 + nlev + 1) * sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    c->kernel_launches += nlev;
    const int64_t nm = static_cast<int64_t>(h[0]), np = static_cast<int64_t>(h[1]);
    if (h[2] == 0) {  // no overflow: the lists are complete
      if (h[4 + nlev] != 0) fail(FMM_ERR_CUDA, "traverse: frontier not empty after 2*depth+2 levels");
      finish_lists(c, nm, np);
      return;
    }
    // Counters keep counting past a full buffer, so every count is exact up to the first level
    // whose frontier was truncated; the levels after it saw a partial frontier and their counts
    // are lower bounds. Grow each buffer to its count (+ slack), and at least double the ones
    // that may be underestimated; every attempt completes at least one more level.
    if (attempt >= 24) fail(FMM_ERR_CUDA, "traverse: output overflow after regrow");
    bool trunc = false;
    int64_t fgrow = 0;
    for (int L = 0; L <= nlev; ++L) {
      const int64_t f = static_cast<int64_t>(h[4 + L]);
      fgrow = std::max(fgrow, trunc ? std::max(f, 2 * cap_f) : f);
      if (f > cap_f) trunc = true;
    }
    auto grow = [&](int64_t count, int64_t cap) {
      const int64_t want = count + count / 8 + 1024;
      return trunc ? std::max(want, 2 * cap) : want;
    };
    const int64_t newf = fgrow + fgrow / 8 + 1024;
    if (newf > cap_f) {
      c->pairs_a.ensure(newf);
      c->pairs_d.ensure(newf);
    }
    const int64_t div = small ? 2 : 1;
    if (nm > cap_m || trunc) c->m2l_keys.ensure(grow(nm, cap_m) / div + 1);
    if (np > cap_p || trunc) c->p2p_keys.ensure(grow(np, cap_p) / div + 1);
  }
}

}  // namespace fmmb

namespace fmmb {
namespace {
__global__ void k_op_mac(int64_t count, const double* __restrict__ tc, const double* __restrict__ tr,
                         const double* __restrict__ sc, const double* __restrict__ sr, double theta,
                         int32_t* __restrict__ out) {
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= count) return;
  out[k] = mac_exact(make_double4(tc[3 * k], tc[3 * k + 1], tc[3 * k + 2], tr[k]),
                     make_double4(sc[3 * k], sc[3 * k + 1], sc[3 * k + 2], sr[k]), theta) ? 1 : 0;
}
}  // namespace

void op_mac(int64_t count, const double* tc3, const double* tr, const double* sc3, const double* sr,
            double theta, int32_t* out) {
  if (count <= 0) return;
  double* d = nullptr;
  int32_t* o = nullptr;
  CK(cudaMalloc(&d, count * 8 * sizeof(double)));
  CK(cudaMalloc(&o, count * sizeof(int32_t)));
  CK(cudaMemcpy(d, tc3, count * 3 * sizeof(double), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(d + 3 * count, tr, count * sizeof(double), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(d + 4 * count, sc3, count * 3 * sizeof(double), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(d + 7 * count, sr, count * sizeof(double), cudaMemcpyHostToDevice));
  k_op_mac<<<ceil_div(count, 128), 128>>>(count, d, d + 3 * count, d + 4 * count, d + 7 * count, theta, o);
  CK_LAUNCH("op_mac");
  CK(cudaMemcpy(out, o, count * sizeof(int32_t), cudaMemcpyDeviceToHost));
  cudaFree(d);
  cudaFree(o);
}
}  // namespace fmmb
