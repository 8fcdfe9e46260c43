// m2l.cu — the FP64 M2L kernel (reference: m2l, kernels.cpp:98-111, applied over the M2L list
// by KernelVisitor::m2l_pair, traversal.hpp:143-152). See expansions.cu for the conventions.
#include <algorithm>
#include <atomic>

#include <cub/cub.cuh>

#include "expansions.cuh"
#include "tma.cuh"

// A/B switches (tools/m2l_ab.sh): split recurrence sums, next-chunk centre prefetch, volatile
// source-row reads in k_m2l_big2
#ifndef FMM_BIG2_VOLATILE
#define FMM_BIG2_VOLATILE 0
#endif
#ifndef FMM_M2L_TWOACC
#define FMM_M2L_TWOACC 0
#endif
#ifndef FMM_M2L_PREFETCH
#define FMM_M2L_PREFETCH 0
#endif
#ifndef FMM_M2L_SPLIT_EPILOGUE  // p >= 7: compact Lambda to global, expanded by k_m2l_expand
#define FMM_M2L_SPLIT_EPILOGUE 1
#endif

namespace fmmb {
namespace {

// kernel attributes are per device: set them once for each device a context runs on (marked
// only after the attribute is set: a concurrent first use just sets it twice)
template <class F>
inline void once_per_device(std::atomic<uint64_t>& mask, int device, F&& set) {
  const uint64_t bit = 1ull << (device & 63);
  if (mask.load() & bit) return;
  set();
  mask.fetch_or(bit);
}

// ---------------------------------------------------------------- register M2L (p <= 6) ----
// Harmonic (traceless) reduction. Dt_g = g! D_g = d^g(1/|R|) is harmonic, so
//   Dt_{g+2ex} + Dt_{g+2ey} + Dt_{g+2ez} = 0   (R != 0),
// which makes every index with c >= 2 a combination of same-degree indices with smaller c.
//  * Source side: M_a Dt_{a+b} with a_c >= 2 equals -M_a Dt_{(a-2ez+2ex)+b} - M_a Dt_{(a-2ez+2ey)+b}
//    for every b, so each multipole is folded once ("detraced", k_detrace) onto the p^2
//    indices with a_c <= 1, exactly (the fold is linear and independent of b and R).
//  * Target side: Lambda_b = sum_a M'_a Dt_{a+b} inherits the identity in b (the truncation
//    |a| + |b| <= p-1 depends on |b| only), so Lambda is contracted for b_c <= 1 and the c >= 2
//    entries are filled afterwards: Lambda_{a,b,c} = -Lambda_{a+2,b,c-2} - Lambda_{a,b+2,c-2}.
//  * Only Dt_g with g_c <= 2 then appear (the recurrence for them never leaves that set).
// p = 6: 301 contraction terms instead of 462, 46 derivatives instead of 56, 36 accumulators
// instead of 56 (the register budget limits this kernel's occupancy). The folded arithmetic
// differs from the reference's only by rounding.
template <int P>
struct HM {
  static constexpr int N = n_coef(P);
  struct Tab {
    int na, ng;
    int a_full[N], a_of[N], g_of[N];
  };
  static constexpr Tab make() {
    Tab t{};
    t.na = 0;
    t.ng = 0;
    for (int i = 0; i < N; ++i) {
      t.a_of[i] = -1;
      t.g_of[i] = -1;
      const int c = MI<P>::ec(i);
      if (c <= 1) {
        t.a_of[i] = t.na;
        t.a_full[t.na++] = i;
      }
      if (c <= 2) t.g_of[i] = t.ng++;
    }
    return t;
  }
  static constexpr Tab tab = make();
  static constexpr int NA = tab.na, NG = tab.ng;
  static constexpr int a_full(int k) { return tab.a_full[k]; }
  static constexpr int a_of(int i) { return tab.a_of[i]; }
  static constexpr int g_of(int i) { return tab.g_of[i]; }
};

// Row stride (doubles) of the staged rows: even (16-B aligned rows) with an odd half, so a
// quarter-warp's LDS.128 of 8 distinct rows hits 8 distinct bank groups.
constexpr int m2l_row_stride(int n) {
  int s = n + (n & 1);
  return (s / 2) % 2 == 1 ? s : s + 2;
}

// One bulk copy per RUN of consecutive source cells instead of one per lane. A per-lane bulk copy
// compiles to a serial loop over the active lanes (R2UR / ELECT / UBLKCP: the instruction takes
// uniform operands): 32 steps per chunk, 20 % of the p = 10 kernel's and 48 % of the p = 6 kernel's
// stall samples (ncu, C5 / C2). The sources of a list ascend and siblings are adjacent cells, so
// most chunks are a handful of runs. The detraced rows are stored with the staged stride (padded)
// in global memory, so a run is contiguous on both sides. Valid lanes are a prefix [0, nv).
__device__ __forceinline__ void stage_runs(int lane, bool valid, int nv, int32_t s, double* rows, const double* Mt,
                                           int S, uint64_t* bar) {
  const int32_t sp = __shfl_up_sync(0xffffffffu, s, 1);
  const bool head = valid && (lane == 0 || s != sp + 1);
  const unsigned heads = __ballot_sync(0xffffffffu, head);
  if (head) {
    const unsigned above = (heads >> 1) >> lane;  // run heads above this lane
    const int next = above ? lane + __ffs(above) : nv;
    FMM_CHECK(next > lane && next <= 32 && s >= 0 && s + (next - lane) <= FMM_LIM(ncells), "stage_runs: run of source rows");
    bulk_g2s(rows + lane * S, Mt + (int64_t)s * S, static_cast<unsigned>(next - lane) * S * 8u, bar);
  }
}

// M' = detraced multipoles (HM<P>::NA per cell, compact a_c <= 1 order); thread per cell, the
// row in a per-thread shared-memory slice (odd stride: the lanes always touch the same entry, so
// the accesses are conflict-free). Fold c >= 2 onto c - 2, highest c first.
constexpr int kDetraceThreads = 64;
template <int P>
__global__ void __launch_bounds__(kDetraceThreads) k_detrace(const double* __restrict__ M, int64_t ncells,
                                                             double* __restrict__ Mt) {
  using T = MI<P>;
  using H = HM<P>;
  constexpr int N = T::N, S = odd_stride(N);
  extern __shared__ double dsm[];
  const int64_t cell = blockIdx.x * (int64_t)kDetraceThreads + threadIdx.x;
  if (cell >= ncells) return;
  double* m = dsm + threadIdx.x * S;
  for (int i = 0; i < N; ++i) m[i] = M[cell * N + i];
  static_for<P>([&](auto K) {
    constexpr int c = P - 1 - decltype(K)::value;
    if constexpr (c >= 2) {
      static_for<N>([&](auto I) {
        constexpr int i = decltype(I)::value;
        if constexpr (T::ec(i) == c) {
          constexpr int a = T::ea(i), b = T::eb(i);
          const double v = m[i];
          m[index_of(a + 2, b, c - 2)] -= v;
          m[index_of(a, b + 2, c - 2)] -= v;
        }
      });
    }
  });
  constexpr int MS = m2l_row_stride(H::NA);  // rows padded to the staged stride
  static_for<H::NA>([&](auto K) {
    constexpr int k = decltype(K)::value;
    Mt[cell * MS + k] = m[H::a_full(k)];
  });
  for (int k = H::NA; k < MS; ++k) Mt[cell * MS + k] = 0.0;
}

template <int P>
void launch_detrace(fmm_ctx* c, double* Mt, cudaStream_t s) {
  const size_t smem = sizeof(double) * kDetraceThreads * odd_stride(MI<P>::N);
  static std::atomic<uint64_t> attr{0};  // per device: the attribute is a per-device setting
  once_per_device(attr, c->cfg.device, [&] {
    CK(cudaFuncSetAttribute(k_detrace<P>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  });
  k_detrace<P><<<ceil_div(c->ncells, kDetraceThreads), kDetraceThreads, smem, s>>>(c->M.p, c->ncells, Mt);
  CK_LAUNCH("k_detrace");
}

// The detraced rows of the current multipoles (built once per upward pass: fmm_evaluate builds them
// on the upward stream, under the traversal; a stand-alone fmm_m2l builds them here)
template <int P>
double* detraced_rows(fmm_ctx* c, cudaStream_t s) {
  const size_t need = c->ncells * m2l_row_stride(HM<P>::NA) + 1;
  if (c->mt_version != c->M_version || c->m2l_mt.cap < need) {
    launch_detrace<P>(c, c->m2l_mt.ensure(need), s);
    c->mt_version = c->M_version;
    c->kernel_launches += 1;
  }
  return c->m2l_mt.p;
}
template <int P>
struct Detrace {
  static void run(fmm_ctx* c, cudaStream_t s) { detraced_rows<P>(c, s); }
};

// Dt_g for g_c <= 2 (compact HM::g_of order) by the reference's degree recurrence
// (multi_index.cpp:64-83) rescaled by g!:
//   n r^2 Dt_g = -(2n-1) sum_d g_d r_d Dt_{g-e_d} - (n-1) sum_d g_d (g_d - 1) Dt_{g-2e_d},
// every index and coefficient a compile-time constant, all in registers.
template <int P>
__device__ __forceinline__ void derivs_reg(double rx, double ry, double rz, double (&D)[HM<P>::NG]) {
  using T = MI<P>;
  using H = HM<P>;
  const double r2 = (rx * rx + ry * ry) + rz * rz;
  D[0] = rsqrt(r2);
  const double inv_r2 = D[0] * D[0];
  double an[P];  // -(2n-1)/(n r^2); the s2 weight -(n-1)/(n r^2) = an * (n-1)/(2n-1) is folded
#pragma unroll
  for (int n = 1; n < P; ++n) an[n] = (-double(2 * n - 1) / double(n)) * inv_r2;
  static_for<T::N>([&](auto I) {
    constexpr int i = decltype(I)::value;
    constexpr int a = T::ea(i), b = T::eb(i), c = T::ec(i), n = T::deg(i);
    if constexpr (i > 0 && c <= 2) {
      constexpr double cn = double(n - 1) / double(2 * n - 1);
      // two independent partial sums (first- and second-order terms): half the dependent-FMA
      // chain of the degree recurrence (it is latency-bound at the register kernels' occupancy)
      double acc1 = 0.0;
#if FMM_M2L_TWOACC
      double acc2 = 0.0;
#else
      double& acc2 = acc1;
#endif
      if constexpr (a >= 1) acc1 = fma(double(a) * rx, D[H::g_of(index_of(a - 1, b, c))], acc1);
      if constexpr (b >= 1) acc1 = fma(double(b) * ry, D[H::g_of(index_of(a, b - 1, c))], acc1);
      if constexpr (c >= 1) acc1 = fma(double(c) * rz, D[H::g_of(index_of(a, b, c - 1))], acc1);
      if constexpr (a >= 2) acc2 = fma(double(a * (a - 1)) * cn, D[H::g_of(index_of(a - 2, b, c))], acc2);
      if constexpr (b >= 2) acc2 = fma(double(b * (b - 1)) * cn, D[H::g_of(index_of(a, b - 2, c))], acc2);
      if constexpr (c >= 2) acc2 = fma(double(c * (c - 1)) * cn, D[H::g_of(index_of(a, b, c - 2))], acc2);
#if FMM_M2L_TWOACC
      D[H::g_of(i)] = an[n] * (acc1 + acc2);
#else
      D[H::g_of(i)] = an[n] * acc1;
#endif
    }
  });
}

// Same recurrence restricted to g_c <= 1 (the compact a-order HM::a_of, NA values): the set is
// closed under the recurrence. Used when the g_c = 2 entries are folded by the trace identity
// Dt_{x,y,2} = -Dt_{x+2,y,0} - Dt_{x,y+2,0} (k_m2l_big2 at p = 10: 100 registers instead of 136).
template <int P>
__device__ __forceinline__ void derivs_reg1(double rx, double ry, double rz, double (&D)[HM<P>::NA]) {
  using T = MI<P>;
  using H = HM<P>;
  const double r2 = (rx * rx + ry * ry) + rz * rz;
  D[0] = rsqrt(r2);
  const double inv_r2 = D[0] * D[0];
  double an[P];
#pragma unroll
  for (int n = 1; n < P; ++n) an[n] = (-double(2 * n - 1) / double(n)) * inv_r2;
  static_for<T::N>([&](auto I) {
    constexpr int i = decltype(I)::value;
    constexpr int a = T::ea(i), b = T::eb(i), c = T::ec(i), n = T::deg(i);
    if constexpr (i > 0 && c <= 1) {
      constexpr double cn = double(n - 1) / double(2 * n - 1);
      double acc = 0.0;
      if constexpr (a >= 1) acc = fma(double(a) * rx, D[H::a_of(index_of(a - 1, b, c))], acc);
      if constexpr (b >= 1) acc = fma(double(b) * ry, D[H::a_of(index_of(a, b - 1, c))], acc);
      if constexpr (c >= 1) acc = fma(double(c) * rz, D[H::a_of(index_of(a, b, c - 1))], acc);
      if constexpr (a >= 2) acc = fma(double(a * (a - 1)) * cn, D[H::a_of(index_of(a - 2, b, c))], acc);
      if constexpr (b >= 2) acc = fma(double(b * (b - 1)) * cn, D[H::a_of(index_of(a, b - 2, c))], acc);
      D[H::a_of(i)] = an[n] * acc;
    }
  });
}

// Lambda epilogue driven by tables in constant memory: lanes take the coefficients lane,
// lane + 32, ... with runtime indices, instead of one predicated static branch per coefficient
// (p = 10: 320 branches per target; ncu C5: ~15 % of the kernel's stall samples were
// branch_resolving in that epilogue, with ~3 source chunks per target).
template <int P>
struct TraceTab {
  static constexpr int N = n_coef(P), NA = HM<P>::NA;
  int16_t a_full[NA];      // compact index -> full index
  int16_t fill[N][3];      // c >= 2 entries in increasing c: target, j1, j2 (full = -full[j1] - full[j2])
  int16_t cstart[P + 1];   // fill entries of c are [cstart[c], cstart[c + 1])
  double w[N];             // (-1)^|b| / b!
};
template <int P>
constexpr TraceTab<P> make_trace_tab() {
  using T = MI<P>;
  TraceTab<P> t{};
  for (int k = 0; k < HM<P>::NA; ++k) t.a_full[k] = static_cast<int16_t>(HM<P>::a_full(k));
  int m = 0;
  for (int c = 0; c <= P; ++c) {
    t.cstart[c] = static_cast<int16_t>(m);
    if (c >= 2 && c < P)
      for (int i = 0; i < T::N; ++i)
        if (T::ec(i) == c) {
          t.fill[m][0] = static_cast<int16_t>(i);
          t.fill[m][1] = static_cast<int16_t>(index_of(T::ea(i) + 2, T::eb(i), c - 2));
          t.fill[m][2] = static_cast<int16_t>(index_of(T::ea(i), T::eb(i) + 2, c - 2));
          ++m;
        }
  }
  for (int i = 0; i < T::N; ++i) t.w[i] = ((T::deg(i) & 1) ? -1.0 : 1.0) / T::fact(i);
  return t;
}
template <int P>
__constant__ TraceTab<P> g_trace = make_trace_tab<P>();

template <int P>
__device__ __forceinline__ void trace_fill_store_tab(int lane, const double* cmp, double* full, double* Lt) {
  const TraceTab<P>& tt = g_trace<P>;
  for (int k = lane; k < TraceTab<P>::NA; k += 32) full[tt.a_full[k]] = cmp[k];
  __syncwarp();
  for (int c = 2; c < P; ++c) {
    for (int m = tt.cstart[c] + lane; m < tt.cstart[c + 1]; m += 32)
      full[tt.fill[m][0]] = -full[tt.fill[m][1]] - full[tt.fill[m][2]];
    __syncwarp();
  }
  for (int i = lane; i < TraceTab<P>::N; i += 32) Lt[i] += tt.w[i] * full[i];
}

// Split epilogue (p >= 7): the M2L kernel stores each target's compact Lambda (b_c <= 1) and a
// second, fully parallel kernel expands it: iterating the trace identity gives the closed form
//   Lambda_{a,b,c} = (-1)^k sum_j C(k,j) Lambda_{a+2j, b+2(k-j), c-2k},  k = c div 2,
// at most 5 compact terms per coefficient at p = 10. The serial, table-driven fill (8 warp
// barriers and ~900 dependent constant/shared loads per target) took 17 % of the p = 10 kernel's
// stall samples on a 7-warp SM (ncu, C5); here it runs one thread per (target, coefficient).
template <int P>
struct ExpandTab {
  static constexpr int N = n_coef(P), K = (P + 1) / 2;
  int8_t n[N];
  int16_t idx[N][K];  // compact index of each term
  double w[N][K];     // (-1)^k C(k,j) * (-1)^{|b|} / b!
};
template <int P>
constexpr ExpandTab<P> make_expand_tab() {
  using T = MI<P>;
  ExpandTab<P> t{};
  for (int i = 0; i < T::N; ++i) {
    const int a = T::ea(i), b = T::eb(i), c = T::ec(i), k = c / 2;
    const double w = ((T::deg(i) & 1) ? -1.0 : 1.0) / T::fact(i);
    t.n[i] = static_cast<int8_t>(k + 1);
    double binom = 1.0;
    for (int j = 0; j <= k; ++j) {
      t.idx[i][j] = static_cast<int16_t>(HM<P>::a_of(index_of(a + 2 * j, b + 2 * (k - j), c - 2 * k)));
      t.w[i][j] = ((k & 1) ? -binom : binom) * w;
      binom = binom * double(k - j) / double(j + 1);
    }
  }
  return t;
}
// global (not constant) memory: the lanes of a warp read different entries
template <int P>
__device__ const ExpandTab<P> g_expand = make_expand_tab<P>();

// Block = one coefficient per thread (its table row in registers), looping over a range of
// targets; each target's compact row is staged in shared memory (double-buffered: one barrier
// per target) and the RMW of L is coalesced. (One thread per (target, coefficient) with the table
// read from global memory per element took 1.2 ms at C5, 5x its memory time.)
constexpr int kExpandTargets = 32;  // targets per block
template <int P, class RowFn>
__device__ __forceinline__ void expand_rows(const int32_t* __restrict__ targets, int64_t nt, double* __restrict__ L,
                                            RowFn&& compact) {
  constexpr int N = n_coef(P), NA = HM<P>::NA, K = ExpandTab<P>::K;
  static_assert(N <= 256, "one coefficient per thread");
  __shared__ double row[2][NA];
  const int i = threadIdx.x;
  const ExpandTab<P>& et = g_expand<P>;
  int idx[K];
  double w[K];
#pragma unroll
  for (int j = 0; j < K; ++j) {  // unused terms: weight 0 on entry 0
    idx[j] = 0;
    w[j] = 0.0;
  }
  if (i < N) {
    const int n = et.n[i];
#pragma unroll
    for (int j = 0; j < K; ++j)
      if (j < n) {
        idx[j] = et.idx[i][j];
        w[j] = et.w[i][j];
      }
  }
  const int64_t r0 = blockIdx.x * (int64_t)kExpandTargets;
  const int64_t r1 = r0 + kExpandTargets < nt ? r0 + kExpandTargets : nt;
  for (int64_t r = r0; r < r1; ++r) {
    double* rw = row[(r - r0) & 1];
    if (i < NA) rw[i] = compact(r, i);
    __syncthreads();  // the readers of this buffer's previous row passed the barrier in between
    if (i < N) {
      double v = 0.0;
#pragma unroll
      for (int j = 0; j < K; ++j) v = fma(w[j], rw[idx[j]], v);
      FMM_CHECK(targets[r] >= 0 && targets[r] < FMM_LIM(ncells), "k_m2l_expand: target index");
      L[(int64_t)targets[r] * N + i] += v;
    }
  }
}

template <int P>
__global__ void __launch_bounds__(256) k_m2l_expand(const int32_t* __restrict__ targets, int64_t ntargets,
                                                    const double* __restrict__ Lc, double* __restrict__ L) {
  constexpr int NA = HM<P>::NA;
  expand_rows<P>(targets, ntargets, L, [&](int64_t r, int i) { return Lc[r * NA + i]; });
}

// Lane = source, warp = target. Dt (g_c <= 2) in registers; the contraction
// Lambda_b += M'_a Dt_{a+b} over a_c, b_c <= 1 (one FMA per term) with Lambda in registers. Each
// lane's detraced source row arrives by one TMA bulk copy (8-byte cp.async when the row is not
// a 16-byte multiple) on a per-warp mbarrier while the recurrence runs; one shared-memory
// transpose reduction per target, then the c >= 2 entries of Lambda by the trace identity.
#ifndef FMM_M2L_DB
#define FMM_M2L_DB 0  // measured slower at p = 6 (1.07 -> 1.14 ms): register pressure
#endif
#ifndef FMM_M2L_MINB
#define FMM_M2L_MINB 10
#endif
#ifndef FMM_M2L_WARPS
#define FMM_M2L_WARPS 1
#endif
constexpr int kM2LWarps = FMM_M2L_WARPS;  // warps (targets) per CTA
template <int P>
__global__ void __launch_bounds__(32 * kM2LWarps, FMM_M2L_MINB)
k_m2l_reg(const int32_t* __restrict__ targets, int64_t ntargets, const int64_t* __restrict__ off,
          const int32_t* __restrict__ src, const double4* __restrict__ cr, const double* __restrict__ Mt,
          double* __restrict__ L) {
  using T = MI<P>;
  using H = HM<P>;
  constexpr int N = T::N, NA = H::NA, NG = H::NG, S = m2l_row_stride(NA);
#ifndef FMM_M2L_COOP
#define FMM_M2L_COOP 0
#endif
  // kCoop: the warp stages its 32 source rows cooperatively with 16-B cp.async (lane-strided
  // pieces of every row). A bulk copy per lane serialises: the bulk-copy instruction takes
  // uniform operands, so 32 per-lane copies become a 32-step loop of R2UR / ELECT / UBLKCP
  // (ncu, C2: a quarter of the kernel's instructions).
  constexpr bool kCoop = FMM_M2L_COOP && (NA % 2) == 0;
#ifndef FMM_M2L_REG_C1
#define FMM_M2L_REG_C1 1
#endif
  constexpr bool kRegC1 = FMM_M2L_REG_C1 != 0;
  constexpr bool kBulk = !kCoop;  // rows are padded to S doubles (16-B multiples) in global memory too
  // kBulk: the rows of chunk k+1 are copied (TMA) into the other buffer while chunk k computes
  constexpr int kBufs = kBulk && FMM_M2L_DB ? 2 : 1;
  extern __shared__ double smem[];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* sR = smem + (size_t)w * kBufs * 32 * S;  // per-warp source rows, then reduction rows
  __shared__ __align__(8) uint64_t bars[kM2LWarps][2];
  if (kBulk && lane == 0) {
    mbar_init(&bars[w][0], 1);
    mbar_init(&bars[w][1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncwarp();
  const int64_t wid = blockIdx.x * (int64_t)kM2LWarps + w;
  if (wid >= ntargets) return;
  const int32_t t = targets ? targets[wid] : static_cast<int32_t>(wid);  // no target list: warp per cell
  FMM_CHECK(t >= 0 && t < FMM_LIM(ncells), "k_m2l_reg: target index");
  const int64_t l0 = off[t], l1 = off[t + 1];
  FMM_CHECK(l0 >= 0 && l0 <= l1 && l1 <= FMM_LIM(n_m2l), "k_m2l_reg: list range");
  if (l0 >= l1) return;
  const double4 ct = cr[t];
  double lam[NA];
#pragma unroll
  for (int i = 0; i < NA; ++i) lam[i] = 0.0;
  // stage the lane's detraced source row of chunk `cbase` into buffer b (async)
  auto stage = [&](int b, int64_t cbase, int32_t s_lane) {
    double* row = sR + (size_t)b * 32 * S + lane * S;
    if constexpr (kCoop) {
      constexpr int PC = NA / 2;  // 16-B pieces per row
      const int nv = l1 - cbase < 32 ? static_cast<int>(l1 - cbase) : 32;
      double* rows = sR + (size_t)b * 32 * S;
#pragma unroll 2
      for (int idx = lane; idx < 32 * PC; idx += 32) {
        const int r = idx / PC, pc = idx - r * PC;
        const int32_t sr = __shfl_sync(0xffffffffu, s_lane, r);
        double* d = rows + r * S + 2 * pc;
        if (r < nv) {
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(d)),
                       "l"(Mt + (int64_t)sr * S + 2 * pc));
        } else {
          *reinterpret_cast<double2*>(d) = make_double2(0.0, 0.0);  // tail rows contribute nothing
        }
      }
      asm volatile("cp.async.commit_group;\n" ::: "memory");
      return;
    }
    const bool valid_l = cbase + lane < l1;
    if (!valid_l)
      for (int e = 0; e < NA; ++e) row[e] = 0.0;  // tail lanes contribute nothing
    if constexpr (kBulk) {
      fence_proxy_async_smem();  // earlier generic reads of this row before the async write
      const int nvl = l1 - cbase < 32 ? static_cast<int>(l1 - cbase) : 32;
      stage_runs(lane, valid_l, nvl, s_lane, sR + (size_t)b * 32 * S, Mt, S, &bars[w][b]);
    } else if (valid_l) {
      const char* g = reinterpret_cast<const char*>(Mt + (int64_t)s_lane * S);
      const unsigned dst = static_cast<unsigned>(__cvta_generic_to_shared(row));
#pragma unroll
      for (int e = 0; e < NA * 8; e += 8)
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(dst + e), "l"(g + e));
    }
    if constexpr (kBulk) {
      if (lane == 0) {
        const int64_t nv = l1 - cbase < 32 ? l1 - cbase : 32;
        mbar_arrive_expect_tx(&bars[w][b], static_cast<unsigned>(nv * S * 8));
      }
    } else {
      asm volatile("cp.async.commit_group;\n" ::: "memory");
    }
  };
  int32_t s_cur = (l0 + lane < l1) ? src[l0 + lane] : t;
  int32_t s_nxt = (l0 + 32 + lane < l1) ? src[l0 + 32 + lane] : t;
  if (kBufs == 2) stage(0, l0, s_cur);
#ifndef FMM_M2L_REG_PF
#define FMM_M2L_REG_PF 1  // A/B at C2: 0.806 -> 0.801 ms, with 10 CTAs/SM 0.793
#endif
#if FMM_M2L_REG_PF
  // next chunk's source centre one chunk ahead (its L2 latency behind this chunk's contraction)
  double cnx = ct.x, cny = ct.y, cnz = ct.z;
  if (l0 + lane < l1) {
    const double4 c0 = cr[s_cur];
    cnx = c0.x; cny = c0.y; cnz = c0.z;
  }
#endif
  unsigned k = 0;
  for (int64_t base = l0; base < l1; base += 32, ++k) {
    const int b = kBufs == 2 ? (k & 1) : 0;
    const bool valid = base + lane < l1;
    if (kBufs == 2) {
      if (base + 32 < l1) stage(b ^ 1, base + 32, s_nxt);  // next chunk, behind this one
    } else {
      stage(0, base, s_cur);  // hidden behind the Dt recurrence only
    }
    const int32_t s_nn = (base + 64 + lane < l1) ? src[base + 64 + lane] : t;
    FMM_CHECK(s_cur >= 0 && s_cur < FMM_LIM(ncells), "k_m2l_reg: source index");
#if FMM_M2L_REG_PF
    double rx = 1.0, ry = 0.0, rz = 0.0;
    if (valid) {
      rx = cnx - ct.x;
      ry = cny - ct.y;
      rz = cnz - ct.z;
    }
    if (base + 32 + lane < l1) {
      const double4 c1 = cr[s_nxt];
      cnx = c1.x; cny = c1.y; cnz = c1.z;
    }
#else
    const double4 cs = valid ? cr[s_cur] : ct;
    double rx = 1.0, ry = 0.0, rz = 0.0;
    if (valid) {
      rx = cs.x - ct.x;  // R = source centre - target centre (traversal.hpp:146)
      ry = cs.y - ct.y;
      rz = cs.z - ct.z;
    }
#endif
    // kRegC1: Dt over g_c <= 1 only (NA values instead of NG), the g_c = 2 entries from the trace
    // identity in the contraction: fewer registers (occupancy) for a few more FMAs
    double D[kRegC1 ? NA : NG];
    if constexpr (kRegC1) derivs_reg1<P>(rx, ry, rz, D);
    else derivs_reg<P>(rx, ry, rz, D);
    if constexpr (kBulk) {
      mbar_wait(&bars[w][b], kBufs == 2 ? ((k >> 1) & 1u) : (k & 1u));
    } else {
      asm volatile("cp.async.wait_all;\n" ::: "memory");
    }
    __syncwarp();
    const double* Ms = sR + (size_t)b * 32 * S + lane * S;
    auto contract = [&](auto KA, const double m) {
      constexpr int ia = H::a_full(decltype(KA)::value);
      constexpr int aa = T::ea(ia), ab = T::eb(ia), ac = T::ec(ia), da = T::deg(ia);
      static_for<NA>([&](auto KB) {
        constexpr int kb = decltype(KB)::value;
        constexpr int ib = H::a_full(kb);
        if constexpr (da + T::deg(ib) <= P - 1) {
          constexpr int gx = aa + T::ea(ib), gy = ab + T::eb(ib), gz = ac + T::ec(ib);
          if constexpr (!kRegC1) {
            lam[kb] = fma(m, D[H::g_of(index_of(gx, gy, gz))], lam[kb]);
          } else if constexpr (gz <= 1) {
            lam[kb] = fma(m, D[H::a_of(index_of(gx, gy, gz))], lam[kb]);
          } else {  // gz == 2: Dt_{x,y,2} = -Dt_{x+2,y,0} - Dt_{x,y+2,0}
            lam[kb] = fma(-m, D[H::a_of(index_of(gx + 2, gy, 0))], lam[kb]);
            lam[kb] = fma(-m, D[H::a_of(index_of(gx, gy + 2, 0))], lam[kb]);
          }
        }
      });
    };
    // 16-B loads of the staged row (conflict-free: S/2 is odd), two coefficients at a time
    static_for<NA / 2>([&](auto IP) {
      constexpr int i0 = 2 * decltype(IP)::value;
      const double2 mm = *reinterpret_cast<const double2*>(Ms + i0);
      contract(std::integral_constant<int, i0>{}, mm.x);
      contract(std::integral_constant<int, i0 + 1>{}, mm.y);
    });
    if constexpr (NA & 1) contract(std::integral_constant<int, NA - 1>{}, Ms[NA - 1]);
    __syncwarp();  // every lane done reading this buffer before it is refilled
    s_cur = s_nxt;
    s_nxt = s_nn;
  }
  // reduce the 32 lane partials (shared-memory transpose) ...
#pragma unroll
  for (int i = 0; i < NA; ++i) sR[lane * S + i] = lam[i];
  __syncwarp();
  constexpr int R = (NA + 31) / 32;
  double red[R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int kk = lane + 32 * r;
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;  // four chains of 8 dependent adds
    if (kk < NA) {
#pragma unroll
      for (int j = 0; j < 32; j += 4) {
        a0 += sR[j * S + kk];
        a1 += sR[(j + 1) * S + kk];
        a2 += sR[(j + 2) * S + kk];
        a3 += sR[(j + 3) * S + kk];
      }
    }
    red[r] = (a0 + a1) + (a2 + a3);
  }
  __syncwarp();
  // ... place at the full (reference-order) index, fill c >= 2 by the trace identity, then
  // L_b += (-1)^{|b|}/b! Lambda_b (table-driven epilogue: trace_fill_store_tab below)
  double* full = sR;             // N doubles
  double* cmp = sR + 2 * N + 2;  // NA reduced values (32 * S >= 2N + 2 + NA)
#pragma unroll
  for (int r = 0; r < R; ++r)
    if (lane + 32 * r < NA) cmp[lane + 32 * r] = red[r];
  __syncwarp();
  trace_fill_store_tab<P>(lane, cmp, full, L + (int64_t)t * N);
}

// Lambda (compact, lanes reduced) -> full reference-order Lambda by the trace identity, then
// L_b += (-1)^{|b|}/b! Lambda_b. cmp: NA reduced values, full: N doubles of scratch (smem).
template <int P>
__device__ __forceinline__ void trace_fill_store(int lane, const double* cmp, double* full, double* Lt) {
  using T = MI<P>;
  using H = HM<P>;
  constexpr int N = T::N;
  static_for<H::NA>([&](auto K) {
    constexpr int kk = decltype(K)::value;
    if (lane == kk % 32) full[H::a_full(kk)] = cmp[kk];
  });
  __syncwarp();
  static_for<P>([&](auto C) {
    constexpr int c = decltype(C)::value;
    if constexpr (c >= 2) {
      static_for<N>([&](auto I) {
        constexpr int i = decltype(I)::value;
        if constexpr (T::ec(i) == c) {
          constexpr int a = T::ea(i), b = T::eb(i);
          if (lane == i % 32) full[i] = -full[index_of(a + 2, b, c - 2)] - full[index_of(a, b + 2, c - 2)];
        }
      });
      __syncwarp();
    }
  });
  static_for<N>([&](auto I) {
    constexpr int i = decltype(I)::value;
    constexpr double w = ((T::deg(i) & 1) ? -1.0 : 1.0) / T::fact(i);
    if (lane == i % 32) Lt[i] += w * full[i];
  });
}

// ------------------------------------------------- staged-row M2L (p >= 7), v2 ----
// Lane = source, warp = target, like k_m2l_reg, with the per-lane state split by size:
//  * Dt (g_c <= 2; p = 10: 136 values) in registers (derivs_reg, no shared-memory row);
//  * the detraced source row M' (100 values) staged in the warp's shared memory by one TMA
//    bulk copy per lane, read back as broadcast-free own-row loads (16-B stride with an odd
//    half: conflict-free);
//  * the lane's partial Lambda (100 values) in a shared-memory row (odd stride), streamed
//    through registers in blocks of kBlk coefficients: per block and source, kBlk loads and
//    stores against ~2035 / (NA / kBlk) FMAs.
// No L2 scratch, no global gathers inside the contraction. The 32 Lambda rows are reduced
// once per target, then the c >= 2 entries follow from the trace identity.
template <int P>
struct BigCfg2 {
  static constexpr int NA = HM<P>::NA, NG = HM<P>::NG;
  static constexpr int SA = m2l_row_stride(NA);  // staged M' rows (TMA: 16-B multiples)
  static constexpr int SL = odd_stride(NA);      // Lambda rows
#ifndef FMM_BIG2_BLK
#define FMM_BIG2_BLK 25
#endif
  static constexpr int kBlk = FMM_BIG2_BLK;
  static constexpr int kBlocks = (NA + kBlk - 1) / kBlk;
#ifndef FMM_BIG2_C1_MIN_P
#define FMM_BIG2_C1_MIN_P 10
#endif
  static constexpr bool kC1 = P >= FMM_BIG2_C1_MIN_P;  // Dt over g_c <= 1 only (register budget)
#ifndef FMM_BIG2_LR_MIN_P
#define FMM_BIG2_LR_MIN_P 10
#endif
  // kLR: the lanes' block partials are reduced after every block (transpose through a 32 x kBlk
  // buffer) into lane-owned target accumulators, instead of a Lambda row per lane: 5 KB instead
  // of 26 KB of shared memory per warp (p = 10), so 7 instead of 4 warps per SM (C5 M2L
  // 24.5 -> 19.6 ms; at p = 8 the extra reductions cost more than the occupancy gains)
  static constexpr bool kLR = P >= FMM_BIG2_LR_MIN_P;
  static constexpr int SB = odd_stride(kBlk);
#ifndef FMM_BIG2_SHFL
#define FMM_BIG2_SHFL 0
#endif
  // kShfl: the per-block lane reduction as a register butterfly (reduce-scatter by shuffles: lane
  // j ends with the sum of value j) instead of a transpose through shared memory: no block
  // buffer (26 instead of 32.5 KB per warp at p = 10: 8 warps per SM), no warp barriers, and the
  // shuffles are free to interleave with the next block's FMAs
  static constexpr bool kShfl = kLR && FMM_BIG2_SHFL && kBlk <= 32;
  static constexpr size_t kSmemPerWarp = sizeof(double) * 32 * (SA + (kLR ? (kShfl ? 0 : SB) : SL));
#ifndef FMM_BIG2_WARPS
#define FMM_BIG2_WARPS 1
#endif
#ifndef FMM_BIG2_WARPS_P10
#define FMM_BIG2_WARPS_P10 7
#endif
  // warps (targets) per CTA, advancing chunk by chunk in lockstep (a CTA barrier per chunk):
  // the fully unrolled contraction (p = 10: ~45 KB of SASS per chunk) is then fetched once per
  // SM position instead of once per warp (ncu at 1 warp/CTA: 40 % no_instruction stalls)
  static constexpr int kWarps = P >= 10 ? FMM_BIG2_WARPS_P10 : FMM_BIG2_WARPS;
#ifndef FMM_BIG2_MINB_P10
#define FMM_BIG2_MINB_P10 1
#endif
  static constexpr int kMinBlocks = P >= 10 ? FMM_BIG2_MINB_P10 : 1;
};

template <int P>
__global__ void __launch_bounds__(32 * BigCfg2<P>::kWarps, BigCfg2<P>::kMinBlocks)
k_m2l_big2(const int32_t* __restrict__ targets, int64_t ntargets, const int64_t* __restrict__ off,
           const int32_t* __restrict__ src, const double4* __restrict__ cr, const double* __restrict__ Mt,
           double* __restrict__ L, double* __restrict__ Lc) {
  using T = MI<P>;
  using H = HM<P>;
  using C = BigCfg2<P>;
  constexpr int N = T::N, NA = C::NA, NG = C::NG, SA = C::SA, SL = C::SL;
  // warp-cooperative 16-B cp.async staging of the 32 source rows (a bulk copy per lane compiles
  // to a 32-step R2UR / ELECT / UBLKCP loop: ncu C5, ~9 % of the stall samples)
  constexpr bool kCoop = FMM_M2L_COOP && (NA % 2) == 0;
  constexpr bool kBulk = !kCoop;  // padded rows: always 16-B multiples
  constexpr int W = C::kWarps;
  extern __shared__ __align__(16) double smem[];
  __shared__ __align__(8) uint64_t bars[W];
  __shared__ int64_t cta_chunks;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  double* wsm = smem + (size_t)w * (C::kSmemPerWarp / sizeof(double));
  double* rowsM = wsm;            // [32][SA]
  double* rowsL = wsm + 32 * SA;  // [32][SL] (kLR: [32][SB] block buffer)
  double* myM = rowsM + lane * SA;
  double* myL = rowsL + lane * SL;
  uint64_t& bar = bars[w];
  if (kBulk && lane == 0) {
    mbar_init(&bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (threadIdx.x == 0) cta_chunks = 0;
  __syncthreads();
  unsigned phase = 0;
  const int64_t wid = blockIdx.x * (int64_t)W + w;
  const bool have = wid < ntargets;
  const int32_t t = have ? targets[wid] : 0;
  FMM_CHECK(t >= 0 && t < FMM_LIM(ncells), "k_m2l_big2: target index");
  const double4 ct = cr[t];
  const int64_t l0 = have ? off[t] : 0, l1 = have ? off[t + 1] : 0;
  FMM_CHECK(l0 >= 0 && l0 <= l1 && l1 <= FMM_LIM(n_m2l), "k_m2l_big2: list range");
  if (W > 1 && lane == 0) atomicMax(reinterpret_cast<unsigned long long*>(&cta_chunks),
                                    static_cast<unsigned long long>((l1 - l0 + 31) / 32));
  if (W > 1) __syncthreads();
  const int64_t lockstep_end = W > 1 ? l0 + 32 * cta_chunks : l1;
  constexpr bool kLR = C::kLR;
  double accT[C::kBlocks];  // kLR: Lambda_{q kBlk + lane} of the target (lanes < block width)
#pragma unroll
  for (int q = 0; q < C::kBlocks; ++q) accT[q] = 0.0;
  if constexpr (!kLR)
    for (int i = 0; i < NA; ++i) myL[i] = 0.0;
  int32_t s_next = (l0 + lane < l1) ? src[l0 + lane] : t;
#if FMM_M2L_PREFETCH
  double4 cs_next = cr[s_next];
#endif
  for (int64_t base = l0; base < lockstep_end; base += 32) {
    if (base >= l1) {  // this warp's target is done: keep the CTA's chunk barriers
      __syncthreads();
      continue;
    }
    const int64_t k = base + lane;
    const bool valid = k < l1;
    const int32_t s = s_next;
    FMM_CHECK(!valid || (s >= 0 && s < FMM_LIM(ncells)), "k_m2l_big2: source index");
    if constexpr (kCoop) {  // committed below with the other cp.async paths
      constexpr int PC = NA / 2;  // 16-B pieces per row
      const int nv = l1 - base < 32 ? static_cast<int>(l1 - base) : 32;
#pragma unroll 2
      for (int idx = lane; idx < 32 * PC; idx += 32) {
        const int r = idx / PC, pc = idx - r * PC;
        const int32_t sr = __shfl_sync(0xffffffffu, s, r);
        double* d = rowsM + r * SA + 2 * pc;
        if (r < nv) {
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(d)),
                       "l"(Mt + (int64_t)sr * SA + 2 * pc));
        } else {
          *reinterpret_cast<double2*>(d) = make_double2(0.0, 0.0);  // tail rows contribute nothing
        }
      }
    } else if constexpr (kBulk) {
      if (!valid)
        for (int e = 0; e < NA; ++e) myM[e] = 0.0;  // tail lanes contribute nothing
      fence_proxy_async_smem();
      stage_runs(lane, valid, l1 - base < 32 ? static_cast<int>(l1 - base) : 32, s, rowsM, Mt, SA, &bar);
    } else if (!valid) {
      for (int e = 0; e < NA; ++e) myM[e] = 0.0;
    } else {
      const char* row = reinterpret_cast<const char*>(Mt + (int64_t)s * SA);
      const unsigned dst = static_cast<unsigned>(__cvta_generic_to_shared(myM));
#pragma unroll 1
      for (int e = 0; e < NA * 8; e += 8)
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(dst + e), "l"(row + e));
    }
    if constexpr (kBulk) {
      if (lane == 0) {
        const int64_t nv = l1 - base < 32 ? l1 - base : 32;
        mbar_arrive_expect_tx(&bar, static_cast<unsigned>(nv * SA * 8));
      }
    } else {
      asm volatile("cp.async.commit_group;\n" ::: "memory");
    }
#if FMM_M2L_PREFETCH
    const double4 cs = cs_next;
    if (base + 32 + lane < l1) {
      s_next = src[base + 32 + lane];
      cs_next = cr[s_next];  // next chunk's centre: its L2 latency hides behind this chunk
    }
#else
    if (base + 32 + lane < l1) s_next = src[base + 32 + lane];
    const double4 cs = valid ? cr[s] : ct;
#endif
    double rx = 1.0, ry = 0.0, rz = 0.0;
    if (valid) {
      rx = cs.x - ct.x;  // R = source centre - target centre (traversal.hpp:146)
      ry = cs.y - ct.y;
      rz = cs.z - ct.z;
    }
    constexpr bool kC1 = C::kC1;
    double D[kC1 ? NA : NG];
    if constexpr (kC1) derivs_reg1<P>(rx, ry, rz, D);
    else derivs_reg<P>(rx, ry, rz, D);
    if constexpr (kBulk) {
      mbar_wait_sleep(&bar, phase);
      phase ^= 1u;
    } else {
      asm volatile("cp.async.wait_all;\n" ::: "memory");
    }
    __syncwarp();
    // the source row is re-read in every block: a compiler memory barrier between blocks keeps
    // the loads from being merged across blocks (all NA values live: the Dt registers spill)
    // while leaving them free to be scheduled early within a block
#if FMM_BIG2_VOLATILE
    const volatile double* vM = myM;
#else
    const double* vM = myM;
#endif
    static_for<C::kBlocks>([&](auto BI) {
      constexpr int b0 = decltype(BI)::value * C::kBlk;
      asm volatile("" ::: "memory");
      constexpr int b1 = (b0 + C::kBlk < NA) ? b0 + C::kBlk : NA;
      double lam[b1 - b0];
#pragma unroll
      for (int j = 0; j < b1 - b0; ++j) lam[j] = kLR ? 0.0 : myL[b0 + j];
      static_for<NA>([&](auto KA) {
        constexpr int ka = decltype(KA)::value;
        constexpr int ia = H::a_full(ka);
        constexpr int aa = T::ea(ia), ab = T::eb(ia), ac = T::ec(ia), da = T::deg(ia);
        if constexpr (da + T::deg(H::a_full(b0)) <= P - 1) {
          const double m = vM[ka];
          static_for<b1 - b0>([&](auto J) {
            constexpr int ib = H::a_full(b0 + decltype(J)::value);
            if constexpr (da + T::deg(ib) <= P - 1) {
              constexpr int gx = aa + T::ea(ib), gy = ab + T::eb(ib), gz = ac + T::ec(ib);
              if constexpr (!kC1) {
                constexpr int ig = H::g_of(index_of(gx, gy, gz));
                lam[decltype(J)::value] = fma(m, D[ig], lam[decltype(J)::value]);
              } else if constexpr (gz <= 1) {
                lam[decltype(J)::value] = fma(m, D[H::a_of(index_of(gx, gy, gz))], lam[decltype(J)::value]);
              } else {  // gz == 2: trace identity
                lam[decltype(J)::value] = fma(-m, D[H::a_of(index_of(gx + 2, gy, 0))], lam[decltype(J)::value]);
                lam[decltype(J)::value] = fma(-m, D[H::a_of(index_of(gx, gy + 2, 0))], lam[decltype(J)::value]);
              }
            }
          });
        }
      });
      if constexpr (C::kShfl) {
        // butterfly reduce-scatter over the 32 lanes: at mask m a lane keeps the half of its values
        // selected by its bit m and receives the partner's partials of that half
        double v[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = j < b1 - b0 ? lam[j] : 0.0;
#pragma unroll
        for (int m = 16; m >= 1; m >>= 1) {
          const bool up = (lane & m) != 0;
#pragma unroll
          for (int i = 0; i < m; ++i) {
            if (i < b1 - b0) {  // v[i + m] may be a structural zero, v[i] never is for i < width
              const double lo = v[i], hi = v[i + m];
              const double send = up ? lo : hi;
              const double keep = up ? hi : lo;
              v[i] = keep + __shfl_xor_sync(0xffffffffu, send, m);
            }
          }
        }
        accT[decltype(BI)::value] += v[0];  // lane j: value j (zero for j >= width)
      } else if constexpr (kLR) {
        double* red = rowsL;  // [32][SB]
#pragma unroll
        for (int j = 0; j < b1 - b0; ++j) red[lane * C::SB + j] = lam[j];
        __syncwarp();
        if (lane < b1 - b0) {  // four interleaved partial sums: a chain of 8 dependent adds, not 32
          double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
#pragma unroll
          for (int j = 0; j < 32; j += 4) {
            s0 += red[j * C::SB + lane];
            s1 += red[(j + 1) * C::SB + lane];
            s2 += red[(j + 2) * C::SB + lane];
            s3 += red[(j + 3) * C::SB + lane];
          }
          accT[decltype(BI)::value] += (s0 + s1) + (s2 + s3);
        }
        __syncwarp();
      } else {
#pragma unroll
        for (int j = 0; j < b1 - b0; ++j) myL[b0 + j] = lam[j];
      }
    });
    __syncwarp();  // every lane done with its M' row before the next chunk's copies land
    if (W > 1) __syncthreads();
  }
  if (!have) return;
  if constexpr (FMM_M2L_SPLIT_EPILOGUE) {
    // the target's compact Lambda row goes to Lc[wid] (k_m2l_expand finishes it)
    double* out = Lc + wid * NA;
    if constexpr (kLR) {
#pragma unroll
      for (int q = 0; q < C::kBlocks; ++q)
        if (q * C::kBlk + lane < NA && lane < C::kBlk) out[q * C::kBlk + lane] = accT[q];
    } else {
      for (int kk = lane; kk < NA; kk += 32) {  // column sums in fixed order
        double acc = 0.0;
        for (int j = 0; j < 32; ++j) acc += rowsL[j * SL + kk];
        out[kk] = acc;
      }
    }
    return;
  }
  // reduce the 32 lane rows (column sums, fixed order) ...
  double* cmp = rowsM;            // NA reduced values
  double* full = rowsM + NA + 1;  // N values (32 * SA >= NA + N + 1)
  if constexpr (kLR) {
#pragma unroll
    for (int q = 0; q < C::kBlocks; ++q)
      if (q * C::kBlk + lane < NA && lane < C::kBlk) cmp[q * C::kBlk + lane] = accT[q];
  } else {
    for (int kk = lane; kk < NA; kk += 32) {
      double acc = 0.0;
      for (int j = 0; j < 32; ++j) acc += rowsL[j * SL + kk];
      cmp[kk] = acc;
    }
  }
  __syncwarp();
#ifndef FMM_M2L_TAB_EPILOGUE
#define FMM_M2L_TAB_EPILOGUE 1
#endif
  if constexpr (FMM_M2L_TAB_EPILOGUE) trace_fill_store_tab<P>(lane, cmp, full, L + (int64_t)t * N);
  else trace_fill_store<P>(lane, cmp, full, L + (int64_t)t * N);
}

// ------------------------------------------- staged-row M2L, flat pair partition (p >= 10) ----
// The CSR source array is one flat sequence of (target, source) pairs ordered by target. Warp wg
// takes the kFlatK * 32 consecutive pairs from position wg * 32 * K, whichever targets they belong
// to: every chunk is full (C5's lists have a median of 70 sources, i.e. 32 + 32 + 6: per-target
// chunks are 85 % full), every warp of a lockstep CTA has the same number of chunks (no sort by
// chunk count), and a chunk may hold the tail of one target and the head of the next. Lane =
// pair: its own target centre, the same Dt recurrence and contraction as k_m2l_big2; the
// per-block lane reduction runs per segment (lanes of one target). A finished target's compact
// Lambda goes to row (t + wg) of Lc; a target cut by a warp boundary leaves one row per warp,
// (t + w) for w = w1..w2 (consecutive, collision-free because targets ascend with the warp id),
// which k_m2l_expand_flat sums in that fixed order: deterministic, no atomics.
// Chunk metadata (one thread per 32-pair chunk): rank of the target holding the chunk's first
// pair (targets = the cells with a non-empty list, ascending), the lanes at which a list starts
// inside the chunk (bit 0 always set), and whether the last target's list ends with the chunk.
// tcr / toff: the targets' centres and list offsets by rank (one dependent load fewer per chunk).
__global__ void k_flat_targets(const int32_t* __restrict__ targets, int64_t nt, const int64_t* __restrict__ off,
                               const double4* __restrict__ cr, int64_t npairs, double4* __restrict__ tcr,
                               int64_t* __restrict__ toff) {
  const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (r > nt) return;
  if (r == nt) {
    toff[r] = npairs;
    return;
  }
  tcr[r] = cr[targets[r]];
  toff[r] = off[targets[r]];
}

__global__ void k_flat_meta(const int64_t* __restrict__ toff, int64_t nt, int64_t nchunks, int4* __restrict__ meta) {
  const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c >= nchunks) return;
  const int64_t pos0 = 32 * c;
  int64_t lo = 0, hi = nt;  // largest r with toff[r] <= pos0 (toff[nt] = npairs > pos0)
  while (hi - lo > 1) {
    const int64_t mid = (lo + hi) >> 1;
    if (toff[mid] <= pos0) lo = mid;
    else hi = mid;
  }
  unsigned heads = 1u;
  int64_t r = lo + 1;
  while (r < nt && toff[r] < pos0 + 32) {
    heads |= 1u << static_cast<int>(toff[r] - pos0);
    ++r;
  }
  // r - 1 = the chunk's last target; its list ends here iff the next list (or the end) starts at pos0 + 32
  // (a final, partly filled chunk ends its target as well)
  const int last_ends = toff[r] <= pos0 + 32 ? 1 : 0;
  meta[c] = make_int4(static_cast<int>(lo), static_cast<int>(heads), last_ends, 0);
}

template <int P>
__global__ void __launch_bounds__(32 * BigCfg2<P>::kWarps, 1)
k_m2l_flat(const int4* __restrict__ meta, int64_t nwarps, int K, int64_t npairs, const double4* __restrict__ tcr,
           const int32_t* __restrict__ src, const double4* __restrict__ cr, const double* __restrict__ Mt,
           double* __restrict__ Lc) {
  using T = MI<P>;
  using H = HM<P>;
  using C = BigCfg2<P>;
  constexpr int NA = C::NA, SA = C::SA, W = C::kWarps;
#ifndef FMM_FLAT_SYNC
#define FMM_FLAT_SYNC 1
#endif
  constexpr bool kSync = FMM_FLAT_SYNC != 0;  // lockstep chunk barriers
  extern __shared__ __align__(16) double smem[];
  __shared__ __align__(8) uint64_t bars[W];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  double* wsm = smem + (size_t)w * (C::kSmemPerWarp / sizeof(double));
  double* rowsM = wsm;            // [32][SA]
  double* red = wsm + 32 * SA;    // [32][SB] block buffer
  double* myM = rowsM + lane * SA;
  uint64_t& bar = bars[w];
  if (lane == 0) {
    mbar_init(&bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  unsigned phase = 0;
  const int64_t wg = blockIdx.x * (int64_t)W + w;
  const bool have = wg < nwarps;
  const int64_t c0 = wg * (int64_t)K;  // first chunk
  const int64_t nchunks = (npairs + 31) >> 5;
  double accT[C::kBlocks];
#pragma unroll
  for (int q = 0; q < C::kBlocks; ++q) accT[q] = 0.0;
  int r_open = -1;  // rank of the unfinished target held in accT, or -1
  int4 mt_next = have && c0 < nchunks ? meta[c0] : make_int4(0, 1, 1, 0);
  int32_t s_next = have && 32 * c0 + lane < npairs ? src[32 * c0 + lane] : 0;
  for (int c = 0; c < K; ++c) {
    const int64_t pos0 = 32 * (c0 + c);
    if (!have || pos0 >= npairs) {  // keep the CTA's chunk barriers
      if (W > 1 && kSync) __syncthreads();
      continue;
    }
    const int4 mt = mt_next;
    const int32_t s = s_next;
    const bool valid = pos0 + lane < npairs;
    FMM_CHECK(!valid || (s >= 0 && s < FMM_LIM(ncells)), "k_m2l_flat: source index");
    const int nv = npairs - pos0 < 32 ? static_cast<int>(npairs - pos0) : 32;
    if (!valid)
      for (int e = 0; e < NA; ++e) myM[e] = 0.0;  // tail lanes contribute nothing
    fence_proxy_async_smem();
    stage_runs(lane, valid, nv, s, rowsM, Mt, SA, &bar);
    if (lane == 0) mbar_arrive_expect_tx(&bar, static_cast<unsigned>(nv * SA * 8));
    if (c + 1 < K && pos0 + 32 < npairs) {  // next chunk's metadata and sources: latency behind this chunk
      mt_next = meta[c0 + c + 1];
      if (pos0 + 32 + lane < npairs) s_next = src[pos0 + 32 + lane];
    }
    const unsigned heads = static_cast<unsigned>(mt.y);
    const int r_lane = mt.x + __popc(heads & (0xffffffffu >> (31 - lane))) - 1;
    FMM_CHECK((heads & 1u) && mt.x >= 0 && r_lane < FMM_LIM(ncells), "k_m2l_flat: chunk metadata / target rank");
    const double4 ct = tcr[r_lane];
    const double4 cs = valid ? cr[s] : ct;
    double rx = 1.0, ry = 0.0, rz = 0.0;
    if (valid) {
      rx = cs.x - ct.x;  // R = source centre - target centre (traversal.hpp:146)
      ry = cs.y - ct.y;
      rz = cs.z - ct.z;
    }
    constexpr bool kC1 = C::kC1;
    double D[kC1 ? NA : C::NG];
    if constexpr (kC1) derivs_reg1<P>(rx, ry, rz, D);
    else derivs_reg<P>(rx, ry, rz, D);
    mbar_wait_sleep(&bar, phase);
    phase ^= 1u;
    __syncwarp();
    const double* vM = myM;
    static_for<C::kBlocks>([&](auto BI) {
      constexpr int b0 = decltype(BI)::value * C::kBlk;
      asm volatile("" ::: "memory");
      constexpr int b1 = (b0 + C::kBlk < NA) ? b0 + C::kBlk : NA;
      double lam[b1 - b0];
#pragma unroll
      for (int j = 0; j < b1 - b0; ++j) lam[j] = 0.0;
      static_for<NA>([&](auto KA) {
        constexpr int ka = decltype(KA)::value;
        constexpr int ia = H::a_full(ka);
        constexpr int aa = T::ea(ia), ab = T::eb(ia), ac = T::ec(ia), da = T::deg(ia);
        if constexpr (da + T::deg(H::a_full(b0)) <= P - 1) {
          const double m = vM[ka];
          static_for<b1 - b0>([&](auto J) {
            constexpr int ib = H::a_full(b0 + decltype(J)::value);
            if constexpr (da + T::deg(ib) <= P - 1) {
              constexpr int gx = aa + T::ea(ib), gy = ab + T::eb(ib), gz = ac + T::ec(ib);
              if constexpr (!kC1) {
                lam[decltype(J)::value] = fma(m, D[H::g_of(index_of(gx, gy, gz))], lam[decltype(J)::value]);
              } else if constexpr (gz <= 1) {
                lam[decltype(J)::value] = fma(m, D[H::a_of(index_of(gx, gy, gz))], lam[decltype(J)::value]);
              } else {  // gz == 2: trace identity
                lam[decltype(J)::value] = fma(-m, D[H::a_of(index_of(gx + 2, gy, 0))], lam[decltype(J)::value]);
                lam[decltype(J)::value] = fma(-m, D[H::a_of(index_of(gx, gy + 2, 0))], lam[decltype(J)::value]);
              }
            }
          });
        }
      });
#pragma unroll
      for (int j = 0; j < b1 - b0; ++j) red[lane * C::SB + j] = lam[j];
      __syncwarp();
      if (heads == 1u) {  // one target in the chunk: four interleaved chains over all lanes
        if (lane < b1 - b0) {
          double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
#pragma unroll
          for (int j = 0; j < 32; j += 4) {
            s0 += red[j * C::SB + lane];
            s1 += red[(j + 1) * C::SB + lane];
            s2 += red[(j + 2) * C::SB + lane];
            s3 += red[(j + 3) * C::SB + lane];
          }
          accT[decltype(BI)::value] += (s0 + s1) + (s2 + s3);
          if (mt.z) {
            Lc[(mt.x + wg) * NA + b0 + lane] = accT[decltype(BI)::value];
            accT[decltype(BI)::value] = 0.0;
          }
        }
      } else if (__popc(heads) == 2) {
        // two targets: the same 32 loads, predicated onto two sets of four chains (the CTA's warps
        // advance in lockstep, so a chunk with a boundary must not cost more than one without)
        const int bnd = 31 - __clz(heads);  // first lane of the second target
        if (lane < b1 - b0) {
          double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0, u0 = 0.0, u1 = 0.0, u2 = 0.0, u3 = 0.0;
#pragma unroll
          for (int j = 0; j < 32; j += 4) {
            const double v0 = red[j * C::SB + lane], v1 = red[(j + 1) * C::SB + lane];
            const double v2 = red[(j + 2) * C::SB + lane], v3 = red[(j + 3) * C::SB + lane];
            if (j < bnd) s0 += v0; else u0 += v0;
            if (j + 1 < bnd) s1 += v1; else u1 += v1;
            if (j + 2 < bnd) s2 += v2; else u2 += v2;
            if (j + 3 < bnd) s3 += v3; else u3 += v3;
          }
          Lc[(mt.x + wg) * NA + b0 + lane] = accT[decltype(BI)::value] + ((s0 + s1) + (s2 + s3));
          accT[decltype(BI)::value] = (u0 + u1) + (u2 + u3);
          if (mt.z) {
            Lc[(mt.x + 1 + wg) * NA + b0 + lane] = accT[decltype(BI)::value];
            accT[decltype(BI)::value] = 0.0;
          }
        }
      } else {  // segments [a, b) of consecutive lanes, one target each, in lane order
        unsigned rest = heads;
        int r_seg = mt.x;
        while (rest) {
          const int a = __ffs(rest) - 1;
          rest &= rest - 1;
          const int b = rest ? __ffs(rest) - 1 : 32;
          if (lane < b1 - b0) {
            double s0 = 0.0, s1 = 0.0;
            for (int j = a; j + 1 < b; j += 2) {
              s0 += red[j * C::SB + lane];
              s1 += red[(j + 1) * C::SB + lane];
            }
            if ((b - a) & 1) s0 += red[(b - 1) * C::SB + lane];
            accT[decltype(BI)::value] += s0 + s1;
            if (rest || mt.z) {  // every segment but the last ends inside the chunk
              Lc[(r_seg + wg) * NA + b0 + lane] = accT[decltype(BI)::value];
              accT[decltype(BI)::value] = 0.0;
            }
          }
          ++r_seg;
        }
      }
      __syncwarp();
    });
    r_open = mt.z ? -1 : mt.x + __popc(heads) - 1;
    __syncwarp();  // every lane done with its M' row before the next chunk's copies land
    if (W > 1 && kSync) __syncthreads();
  }
  if (r_open >= 0) {  // the target cut by the end of this warp's range: its partial row
#pragma unroll
    for (int q = 0; q < C::kBlocks; ++q)
      if (q * C::kBlk + lane < NA && lane < C::kBlk) Lc[(r_open + wg) * NA + q * C::kBlk + lane] = accT[q];
  }
}

// Expansion for the flat partition: the rows of the target of rank r are (r + w), w = w1..w2,
// the warps whose pair ranges meet its list; summed in warp order, then the closed-form trace
// expansion.
template <int P>
__global__ void __launch_bounds__(256) k_m2l_expand_flat(const int32_t* __restrict__ targets, int64_t nt,
                                                         const int64_t* __restrict__ toff, int64_t span,
                                                         const double* __restrict__ Lc, double* __restrict__ L) {
  constexpr int NA = HM<P>::NA;
  expand_rows<P>(targets, nt, L, [&](int64_t r, int i) {
    const int64_t w1 = toff[r] / span, w2 = (toff[r + 1] - 1) / span;
    double acc = 0.0;
    for (int64_t w = w1; w <= w2; ++w) acc += Lc[(r + w) * NA + i];
    return acc;
  });
}

// lockstep CTAs: targets ordered by descending chunk count (stable), so the warps of a CTA carry
// similar list lengths and few idle through the chunk barriers
__global__ void k_target_chunks(const int32_t* __restrict__ targets, int64_t n, const int64_t* __restrict__ off,
                                uint32_t* __restrict__ chunks) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) chunks[i] = static_cast<uint32_t>((off[targets[i] + 1] - off[targets[i]] + 31) / 32);
}

template <int P>
struct M2L {
  static void run(fmm_ctx* c, cudaStream_t s) {
    if constexpr (P <= 6) {
      constexpr int S = m2l_row_stride(HM<P>::NA);
      constexpr int kBufs = FMM_M2L_DB && !(FMM_M2L_COOP && HM<P>::NA % 2 == 0) ? 2 : 1;  // as in the kernel
      const size_t smem = sizeof(double) * kM2LWarps * kBufs * 32 * S;
      static std::atomic<uint64_t> attr{0};
      once_per_device(attr, c->cfg.device, [&] {
        CK(cudaFuncSetAttribute(k_m2l_reg<P>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      });
      if (c->n_m2l_targets == 0) return;
      double* Mt = detraced_rows<P>(c, s);
      const bool all_cells = c->n_m2l_targets < 0;  // finish_lists skipped the target list
      const int64_t nt = all_cells ? c->ncells : c->n_m2l_targets;
      k_m2l_reg<P><<<ceil_div(nt, kM2LWarps), 32 * kM2LWarps, smem, s>>>(all_cells ? nullptr : c->m2l_targets.p, nt,
                                                                    c->m2l_off.p, c->m2l_src.p, c->c_cr.p, Mt, c->L.p);
      CK_LAUNCH("k_m2l_reg");
      c->kernel_launches += 1;
    } else {  // p >= 7 (only these orders instantiate the staged-row kernel)
    using C2 = BigCfg2<P>;
    const size_t smem2 = C2::kSmemPerWarp * C2::kWarps;
    static std::atomic<uint64_t> attr2{0};
    once_per_device(attr2, c->cfg.device, [&] {
      CK(cudaFuncSetAttribute(k_m2l_big2<P>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem2));
    });
    if (c->n_m2l_targets == 0) return;
    double* Mt = detraced_rows<P>(c, s);
#ifndef FMM_BIG2_FLAT
#define FMM_BIG2_FLAT 1
#endif
    if constexpr (C2::kLR && !C2::kShfl && FMM_BIG2_FLAT && FMM_M2L_SPLIT_EPILOGUE) {
      if (c->world == 1) {  // whole lists (the sharded step runs the target list of the rank)
        const int64_t np = c->n_m2l, nt = c->n_m2l_targets;
        // chunks per warp (A/B at C5: 3 -> 10.05 ms, 6 -> 9.92, 12 -> 9.86: fewer CTA prologues)
#ifndef FMM_FLAT_K
#define FMM_FLAT_K 12
#endif
        const int K = FMM_FLAT_K;
        const int64_t span = 32 * (int64_t)K;
        const int64_t nchunks = (np + 31) / 32, nw = (nchunks + K - 1) / K;
        int4* meta = reinterpret_cast<int4*>(c->keys_a.ensure(2 * nchunks + 2));
        double4* tcr = reinterpret_cast<double4*>(c->keys_b.ensure(5 * (nt + 1) + 4));
        int64_t* toff = reinterpret_cast<int64_t*>(tcr + nt + 1);
        double* Lc = c->m2l_scratch.ensure((nt + nw + 1) * C2::NA);
        k_flat_targets<<<ceil_div(nt + 1, 256), 256, 0, s>>>(c->m2l_targets.p, nt, c->m2l_off.p, c->c_cr.p, np, tcr, toff);
        k_flat_meta<<<ceil_div(nchunks, 256), 256, 0, s>>>(toff, nt, nchunks, meta);
        static std::atomic<uint64_t> attr3{0};
        once_per_device(attr3, c->cfg.device, [&] {
          CK(cudaFuncSetAttribute(k_m2l_flat<P>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem2));
        });
        k_m2l_flat<P><<<(unsigned)ceil_div(nw, C2::kWarps), 32 * C2::kWarps, smem2, s>>>(meta, nw, K, np, tcr, c->m2l_src.p,
                                                                                     c->c_cr.p, Mt, Lc);
        CK_LAUNCH("k_m2l_flat");
        k_m2l_expand_flat<P><<<(unsigned)ceil_div(nt, kExpandTargets), 256, 0, s>>>(c->m2l_targets.p, nt, toff, span, Lc,
                                                                                  c->L.p);
        CK_LAUNCH("k_m2l_expand_flat");
        c->kernel_launches += 4;
        return;
      }
    }
    const int32_t* tg = c->m2l_targets.p;
#ifndef FMM_BIG2_SORT
#define FMM_BIG2_SORT 1
#endif
    if (C2::kWarps > 1 && FMM_BIG2_SORT) {
      const int64_t nt = c->n_m2l_targets;
      uint32_t* kin = reinterpret_cast<uint32_t*>(c->keys_a.ensure(nt + 1));
      uint32_t* kout = reinterpret_cast<uint32_t*>(c->keys_b.ensure(nt + 1));
      int32_t* tout = c->i32_b.ensure(nt + 1);
      k_target_chunks<<<ceil_div(nt, 256), 256, 0, s>>>(c->m2l_targets.p, nt, c->m2l_off.p, kin);
      size_t sb = 0;
      CK(cub::DeviceRadixSort::SortPairsDescending(nullptr, sb, kin, kout, c->m2l_targets.p, tout, (int)nt, 0, 16, s));
      CK(cub::DeviceRadixSort::SortPairsDescending(temp_storage(c, sb), sb, kin, kout, c->m2l_targets.p, tout,
                                                   (int)nt, 0, 16, s));
      tg = tout;
      c->kernel_launches += 4;
    }
    double* Lc = FMM_M2L_SPLIT_EPILOGUE ? c->m2l_scratch.ensure(c->n_m2l_targets * C2::NA + 1) : nullptr;
    k_m2l_big2<P><<<(unsigned)ceil_div(c->n_m2l_targets, C2::kWarps), 32 * C2::kWarps, smem2, s>>>(
        tg, c->n_m2l_targets, c->m2l_off.p, c->m2l_src.p, c->c_cr.p, Mt, c->L.p, Lc);
    CK_LAUNCH("k_m2l_big2");
    c->kernel_launches += 1;
    if (FMM_M2L_SPLIT_EPILOGUE) {
      k_m2l_expand<P><<<(unsigned)ceil_div(c->n_m2l_targets, kExpandTargets), 256, 0, s>>>(tg, c->n_m2l_targets, Lc,
                                                                                         c->L.p);
      CK_LAUNCH("k_m2l_expand");
      c->kernel_launches += 1;
    }
    }
  }
};

}  // namespace

void run_detrace(fmm_ctx* c, cudaStream_t s) {
  if (!c->have_M) fail(FMM_ERR_STATE, "detrace: no multipoles (run upward first)");
  dispatch_order<Detrace>(c->cfg.order, c, s);
}

void run_m2l(fmm_ctx* c, cudaStream_t s) {
  if (!c->have_lists) fail(FMM_ERR_STATE, "m2l: no interaction lists");
  set_check_limits(c, s);
  if (!c->have_M) fail(FMM_ERR_STATE, "m2l: no multipoles (run upward first)");
  dispatch_order<M2L>(c->cfg.order, c, s);
  c->have_L = true;
}

}  // namespace fmmb
