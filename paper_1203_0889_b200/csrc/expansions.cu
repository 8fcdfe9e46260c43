// expansions.cu — Cartesian Taylor expansion operators on sm_100a, FP64, in the reference's
// coefficient order and conventions (kernels.hpp:15-23):
//   multipole  M_a = sum_j q_j (y_j - c)^a / a!                  p2m  kernels.cpp:78-86
//   M2M        parent_b += child_a d^{b-a}/(b-a)!                 m2m  kernels.cpp:88-96
//   M2L        L_b += sum_a (-1)^{|b|} (a+b)!/b! M_a D_{a+b}(R)    m2l  kernels.cpp:98-111
//   L2L        child_a += parent_{a+d} ((a+d)!/a!) d^d/d!          l2l  kernels.cpp:128-136
//   L2P        phi += sum_b L_b (x-c)^b  (+ acc = -grad, extension) l2p kernels.cpp:138-148
// with D_g(R) = (1/g!) d^g (1/|R|) from the reference's degree recurrence
// (multi_index.cpp:59-85). The upward/downward passes (traversal.cpp:36-63) become
// level-synchronous launches: all leaves at once for P2M/L2P, one launch per level for
// M2M (deepest first) and L2L (root first). Every cell is written by exactly one warp.
//
// M2L (the FP64 hot kernel) uses the folded form  Lambda_b = sum_a M_a Dt_{a+b},
// Dt_g = g! D_g = d^g(1/|R|), and L_b += (-1)^{|b|}/b! * Lambda_b at the end: one FMA per
// term. One warp per target cell; lane k handles source k of each 32-source chunk of the
// target's list (lane = source), so every lane runs the same fully unrolled, compile-time
// indexed term sequence; Dt rows live in shared memory (odd stride: conflict-free), the
// per-lane partial Lambda in registers, reduced across the warp once per target.
#include <algorithm>

#include "expansions.cuh"

namespace fmmb {
namespace {

// ------------------------------------------------------------------------------ P2M ----
// Warp per leaf; lanes own coefficients; bodies staged 32 at a time as 1-D power lines
// x^k/k!, y^k/k!, z^k/k! (the multi-index power is their product).
template <int P>
__global__ void __launch_bounds__(128)
k_p2m(const int32_t* __restrict__ leaves, int64_t nleaves, const int32_t* __restrict__ bb,
      const int32_t* __restrict__ be, const double4* __restrict__ cr, const double4* __restrict__ bodies,
      double* __restrict__ M) {
  using T = MI<P>;
  constexpr int N = T::N;
  constexpr int LS = 3 * P + 1;  // per-body line storage: X[P], Y[P], Z[P], q
  __shared__ double sP[4][32][LS];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t wid = blockIdx.x * 4ll + w;
  if (wid >= nleaves) return;
  const int32_t leaf = leaves[wid];
  FMM_CHECK(leaf >= 0 && leaf < FMM_LIM(ncells), "k_p2m: leaf index");
  const double4 c = cr[leaf];
  const int32_t b0 = bb[leaf], b1 = be[leaf];
  FMM_CHECK(b0 >= 0 && b0 <= b1 && b1 <= FMM_LIM(nbodies), "k_p2m: body range");
  constexpr int KPL = (N + 31) / 32;  // coefficients per lane
  double acc[KPL];
#pragma unroll
  for (int k = 0; k < KPL; ++k) acc[k] = 0.0;
  for (int32_t base = b0; base < b1; base += 32) {
    const int nb = min(32, b1 - base);
    if (lane < nb) {
      const double4 b = bodies[base + lane];
      const double vx = b.x - c.x, vy = b.y - c.y, vz = b.z - c.z;
      double* L = sP[w][lane];
      L[0] = 1.0;
      L[P] = 1.0;
      L[2 * P] = 1.0;
#pragma unroll
      for (int k = 1; k < P; ++k) {  // v^k/k! (reciprocals are compile-time constants: no DDIV)
        const double rk = 1.0 / k;
        L[k] = L[k - 1] * (vx * rk);
        L[P + k] = L[P + k - 1] * (vy * rk);
        L[2 * P + k] = L[2 * P + k - 1] * (vz * rk);
      }
      L[3 * P] = b.w;
    }
    __syncwarp();
#pragma unroll
    for (int k = 0; k < KPL; ++k) {
      const int i = lane + 32 * k;
      if (i < N) {
        // runtime exponents of coefficient i
        int n = 0;
        while (n_coef(n + 1) <= i) ++n;
        int r = i - n_coef(n), a = 0;
        while (r >= n - a + 1) { r -= n - a + 1; ++a; }
        const int bexp = r, cexp = n - a - r;
        double s = 0.0;
        for (int j = 0; j < nb; ++j) {
          const double* L = sP[w][j];
          s += L[3 * P] * (L[a] * L[P + bexp] * L[2 * P + cexp]);
        }
        acc[k] += s;
      }
    }
    __syncwarp();
  }
#pragma unroll
  for (int k = 0; k < KPL; ++k) {
    const int i = lane + 32 * k;
    if (i < N) M[(int64_t)leaf * N + i] = acc[k];
  }
}

// ------------------------------------------------------------- axis line sweeps ------
// M2M and L2L factorise over the three axes: the 3-D operator is the composition of 1-D
// operators applied along the "lines" of the coefficient triangle (the exponents on the other
// two axes fixed). Lane l owns line l of an axis (P(P+1)/2 lines) in a warp-private
// shared-memory copy of the expansion; the axes are swept in turn with a __syncwarp between.
// The truncation |alpha| <= P-1 of the reference's term lists (kernels.cpp:25-76) is exactly
// the lines' lengths, so the result equals the term-list sums up to rounding (parity 1e-12).
template <int A>
__device__ __forceinline__ int axis_index(int t, int u, int v) {
  return A == 0 ? index_of(t, u, v) : (A == 1 ? index_of(u, t, v) : index_of(u, v, t));
}

template <int P>
__device__ __forceinline__ int line_uv(int l, int& u) {  // line l -> (u, v), u + v <= P-1
  u = 0;
  while (l >= P - u) {
    l -= P - u;
    ++u;
  }
  return l;
}

// Line tables: element t of line l of axis A sits at coefficient tab[(A NL + l) P + t], the line
// has len[l] elements. Built once per (persistent) block in shared memory: the per-element
// index arithmetic otherwise dominated these kernels (ncu, k_l2l<10>: ALU 44 %, IMAD on the FMA
// pipe 40 %, FP64 11 %).
template <int P>
struct Lines {
  static constexpr int NL = P * (P + 1) / 2;
  static constexpr int kTab = 3 * NL * P;
};

template <int P>
__device__ __forceinline__ void build_lines(int16_t* tab, uint8_t* len) {
  using LN = Lines<P>;
  for (int e = threadIdx.x; e < LN::kTab; e += blockDim.x) {
    const int A = e / (LN::NL * P), l = (e / P) % LN::NL, t = e % P;
    int u;
    const int v = line_uv<P>(l, u);
    const int idx = A == 0 ? axis_index<0>(t, u, v) : (A == 1 ? axis_index<1>(t, u, v) : axis_index<2>(t, u, v));
    tab[e] = static_cast<int16_t>(t < P - u - v ? idx : 0);
  }
  for (int l = threadIdx.x; l < LN::NL; l += blockDim.x) {
    int u;
    const int v = line_uv<P>(l, u);
    len[l] = static_cast<uint8_t>(P - u - v);
  }
  __syncthreads();
}

// L2L along axis A (traversal.cpp:55-57 via l2l, kernels.cpp:128-136): the polynomial
// sum_t x_t s^t becomes its Taylor shift sum_t x_t (s + d)^t (repeated synthetic division)
template <int P, int A>
__device__ __forceinline__ void shift_axis(double* s, double d, int lane, const int16_t* tab, const uint8_t* len) {
  constexpr int NL = Lines<P>::NL;
  for (int l = lane; l < NL; l += 32) {
    const int16_t* row = tab + (A * NL + l) * P;
    const int m = len[l];
    double x[P];
#pragma unroll
    for (int t = 0; t < P; ++t) x[t] = t < m ? s[row[t]] : 0.0;
#pragma unroll
    for (int t = 0; t < P - 1; ++t)
#pragma unroll
      for (int i = P - 2; i >= t; --i)
        if (i + 1 < m) x[i] = fma(d, x[i + 1], x[i]);
#pragma unroll
    for (int t = 0; t < P; ++t)
      if (t < m) s[row[t]] = x[t];
  }
}

// M2M along axis A (kernels.cpp:88-96): u_b = sum_{k<=b} x_{b-k} d^k/k!
template <int P, int A>
__device__ __forceinline__ void m2m_axis(double* s, const double* D, int lane, const int16_t* tab, const uint8_t* len) {
  constexpr int NL = Lines<P>::NL;
  for (int l = lane; l < NL; l += 32) {
    const int16_t* row = tab + (A * NL + l) * P;
    const int m = len[l];
    double x[P];
#pragma unroll
    for (int t = 0; t < P; ++t) x[t] = t < m ? s[row[t]] : 0.0;
#pragma unroll
    for (int b = P - 1; b >= 1; --b) {
      if (b < m) {
        double y = x[b];
#pragma unroll
        for (int k = 1; k <= b; ++k) y = fma(x[b - k], D[k], y);
        x[b] = y;
      }
    }
#pragma unroll
    for (int t = 0; t < P; ++t)
      if (t < m) s[row[t]] = x[t];
  }
}

constexpr int kSweepBlocksPerSM = 16;  // persistent grid of the sweep kernels (x SMs)

// ------------------------------------------------------------------------------ M2M ----
// Warp per cell of one level (grid-stride): each child's multipole (in child order k = 0..count-1,
// the reference's accumulation order, traversal.cpp:44-47) is translated by three axis sweeps in
// a warp-private shared-memory copy and added to the lane-owned parent coefficients.
template <int P>
__global__ void __launch_bounds__(128)
k_m2m(int32_t cbeg, int32_t cend, const int32_t* __restrict__ cb, const int32_t* __restrict__ cc,
      const double4* __restrict__ cr, double* __restrict__ M, const int32_t* __restrict__ owner, int32_t want) {
  using T = MI<P>;
  constexpr int N = T::N;
  constexpr int KPL = (N + 31) / 32;
  __shared__ double sM[4][N];
  __shared__ double sD[4][3][P];
  __shared__ int16_t tab[Lines<P>::kTab];
  __shared__ uint8_t len[Lines<P>::NL];
  build_lines<P>(tab, len);
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int32_t ci = cbeg + blockIdx.x * 4 + w; ci < cend; ci += gridDim.x * 4) {
    const int32_t nch = cc[ci];
    if (nch == 0) continue;
    if (owner && owner[ci] != want) continue;  // sharded: only this rank's (or the shared) cells
    const double4 pc = cr[ci];
    double acc[KPL];
#pragma unroll
    for (int k = 0; k < KPL; ++k) acc[k] = 0.0;
    for (int k = 0; k < nch; ++k) {
      const int32_t child = cb[ci] + k;
      const double4 c4 = cr[child];
      if (lane < 3) {
        const double d = lane == 0 ? c4.x - pc.x : (lane == 1 ? c4.y - pc.y : c4.z - pc.z);
        double* D = sD[w][lane];
        D[0] = 1.0;
        for (int q = 1; q < P; ++q) D[q] = D[q - 1] * d / q;
      }
      for (int i = lane; i < N; i += 32) sM[w][i] = M[(int64_t)child * N + i];
      __syncwarp();
      m2m_axis<P, 0>(sM[w], sD[w][0], lane, tab, len);
      __syncwarp();
      m2m_axis<P, 1>(sM[w], sD[w][1], lane, tab, len);
      __syncwarp();
      m2m_axis<P, 2>(sM[w], sD[w][2], lane, tab, len);
      __syncwarp();
#pragma unroll
      for (int q = 0; q < KPL; ++q) {
        const int i = lane + 32 * q;
        if (i < N) acc[q] += sM[w][i];
      }
      __syncwarp();
    }
#pragma unroll
    for (int q = 0; q < KPL; ++q) {
      const int i = lane + 32 * q;
      if (i < N) M[(int64_t)ci * N + i] = acc[q];
    }
  }
}

// ------------------------------------------------------------------------------ L2L ----
// Warp per cell of one level >= 1 (grid-stride): the parent local, Taylor-shifted to the child
// centre by three axis sweeps, is added to the child's local (the M2L result).
template <int P>
__global__ void __launch_bounds__(128)
k_l2l(int32_t cbeg, int32_t cend, const int32_t* __restrict__ par, const double4* __restrict__ cr,
      double* __restrict__ L) {
  using T = MI<P>;
  constexpr int N = T::N;
  __shared__ double sL[4][N];
  __shared__ int16_t tab[Lines<P>::kTab];
  __shared__ uint8_t len[Lines<P>::NL];
  build_lines<P>(tab, len);
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int32_t ci = cbeg + blockIdx.x * 4 + w; ci < cend; ci += gridDim.x * 4) {
    const int32_t pi = par[ci];
    const double4 c = cr[ci], pc = cr[pi];
    for (int i = lane; i < N; i += 32) sL[w][i] = L[(int64_t)pi * N + i];
    __syncwarp();
    shift_axis<P, 0>(sL[w], c.x - pc.x, lane, tab, len);
    __syncwarp();
    shift_axis<P, 1>(sL[w], c.y - pc.y, lane, tab, len);
    __syncwarp();
    shift_axis<P, 2>(sL[w], c.z - pc.z, lane, tab, len);
    __syncwarp();
    double* Lc = L + (int64_t)ci * N;
    for (int i = lane; i < N; i += 32) Lc[i] += sL[w][i];
    __syncwarp();
  }
}

// ------------------------------------------------------------------------------ L2P ----
// Warp per leaf, lane per body; phi_out = phi_near + sum_b L_b (x-c)^b and
// acc_out = acc_near - grad (extension). Leaf L staged in shared memory (broadcast reads).
#ifndef FMM_L2P_MINB
#define FMM_L2P_MINB 6
#endif
template <int P>
__global__ void __launch_bounds__(128, FMM_L2P_MINB)
k_l2p(const int32_t* __restrict__ leaves, int64_t nleaves, const int32_t* __restrict__ bb,
      const int32_t* __restrict__ be, const double4* __restrict__ cr, const double4* __restrict__ bodies,
      const double* __restrict__ L, const double* __restrict__ phi_near, const double* __restrict__ acc_near,
      double* __restrict__ phi_out, double* __restrict__ acc_out, int with_acc) {
  using T = MI<P>;
  constexpr int N = T::N;
  __shared__ double sL[4][N];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t wid = blockIdx.x * 4ll + w;
  if (wid >= nleaves) return;
  const int32_t leaf = leaves[wid];
  for (int i = lane; i < N; i += 32) sL[w][i] = L[(int64_t)leaf * N + i];
  __syncwarp();
  const double4 c = cr[leaf];
  const int32_t b0 = bb[leaf], b1 = be[leaf];
  for (int32_t i = b0 + lane; i < b1; i += 32) {
    const double4 b = bodies[i];
    const double x = b.x - c.x, y = b.y - c.y, z = b.z - c.z;
    // nested Horner: phi = sum_a x^a sum_b y^b sum_c z^c L_abc, derivatives carried along
    // (dp = dp * x + p before p = p * x + coef); registers only, L broadcast from shared memory
    double ph = 0.0, gx = 0.0, gy = 0.0, gz = 0.0;
    // P >= 8: volatile reads keep the unrolled coefficient loads in order (otherwise they are
    // hoisted ahead of the FMAs and spill)
#ifndef FMM_L2P_VOLATILE_MIN_P
#define FMM_L2P_VOLATILE_MIN_P 4
#endif
    using LPtr = std::conditional_t<(P >= FMM_L2P_VOLATILE_MIN_P), const volatile double*, const double*>;
    const LPtr Lw = sL[w];
    static_for<P>([&](auto AI) {
      constexpr int a = P - 1 - decltype(AI)::value;
      double Tv = 0.0, Ty = 0.0, Tz = 0.0;
      static_for<P - a>([&](auto BI) {
        constexpr int bb_ = P - 1 - a - decltype(BI)::value;
        double S = 0.0, Sz = 0.0;
        static_for<P - a - bb_>([&](auto CI) {
          constexpr int cc_ = P - 1 - a - bb_ - decltype(CI)::value;
          Sz = fma(Sz, z, S);
          S = fma(S, z, Lw[index_of(a, bb_, cc_)]);
        });
        Ty = fma(Ty, y, Tv);
        Tv = fma(Tv, y, S);
        Tz = fma(Tz, y, Sz);
      });
      gx = fma(gx, x, ph);
      ph = fma(ph, x, Tv);
      gy = fma(gy, x, Ty);
      gz = fma(gz, x, Tz);
    });
    phi_out[i] = phi_near[i] + ph;
    if (with_acc) {
      acc_out[3 * i] = acc_near[3 * i] - gx;
      acc_out[3 * i + 1] = acc_near[3 * i + 1] - gy;
      acc_out[3 * i + 2] = acc_near[3 * i + 2] - gz;
    }
  }
}


// --------------------------------------------------------------------- launchers ------
template <int P>
struct Upward {
  // mode 0: every cell; 1: P2P leaves + M2M of this rank's cells; 2: M2M of shared cells only
  static void run(fmm_ctx* c, cudaStream_t s, int mode) {
    const int N = MI<P>::N;
    double* M = c->M.ensure((size_t)c->ncells * N);
    int launches = 0;
    if (mode != 2 && c->nwl > 0) {
      k_p2m<P><<<ceil_div(c->nwl, 4), 128, 0, s>>>(c->wl, c->nwl, c->c_body_begin.p, c->c_body_end.p, c->c_cr.p,
                                                   c->bodies.p, M);
      CK_LAUNCH("k_p2m");
      ++launches;
    }
    const int32_t* owner = mode == 0 ? nullptr : c->owner.p;
    const int32_t want = mode == 1 ? c->rank : -1;
    for (int l = c->depth - 1; l >= 0; --l) {
      const int32_t b = c->level_start[l], e = c->level_start[l + 1];
      if (e <= b) continue;
      const int grid = std::min(ceil_div(e - b, 4), 148 * kSweepBlocksPerSM);
      k_m2m<P><<<grid, 128, 0, s>>>(b, e, c->c_child_begin.p, c->c_child_count.p, c->c_cr.p, M, owner, want);
      CK_LAUNCH("k_m2m");
      ++launches;
    }
    c->kernel_launches += launches;
  }
};

template <int P>
struct Downward {
  // part 1: L2L, level by level (needs only the locals: may run beside P2P); part 2: L2P and the
  // near-field combine (needs the P2P result)
  static void run(fmm_ctx* c, cudaStream_t s, int part) {
    int launches = 0;
    if (part & 1)
      for (int l = 1; l <= c->depth; ++l) {
        const int32_t b = c->level_start[l], e = c->level_start[l + 1];
        if (e <= b) continue;
        const int grid = std::min(ceil_div(e - b, 4), 148 * kSweepBlocksPerSM);
        k_l2l<P><<<grid, 128, 0, s>>>(b, e, c->c_parent.p, c->c_cr.p, c->L.p);
        CK_LAUNCH("k_l2l");
        ++launches;
      }
    if ((part & 2) && c->nwl > 0) {
      k_l2p<P><<<ceil_div(c->nwl, 4), 128, 0, s>>>(c->wl, c->nwl, c->c_body_begin.p, c->c_body_end.p, c->c_cr.p,
                                                   c->bodies.p, c->L.p, c->phi_p2p.p, c->acc_p2p.p,
                                                   c->phi.ensure(c->N), c->acc.ensure(3 * c->N),
                                                   c->cfg.with_acc ? 1 : 0);
      CK_LAUNCH("k_l2p");
      ++launches;
    }
    c->kernel_launches += launches;
  }
};

}  // namespace

void run_upward(fmm_ctx* c, cudaStream_t s, int mode) {
  if (!c->have_tree) fail(FMM_ERR_STATE, "upward: no tree");
  set_check_limits(c, s);
  if (mode != 0 && !c->shard_planned) fail(FMM_ERR_STATE, "sharded upward before the partition (run traverse)");
  dispatch_order<Upward>(c->cfg.order, c, s, mode);
  c->have_M = true;
  ++c->M_version;
}

void run_downward(fmm_ctx* c, cudaStream_t s, int part) {
  if (!c->have_tree) fail(FMM_ERR_STATE, "downward: no tree");
  set_check_limits(c, s);
  dispatch_order<Downward>(c->cfg.order, c, s, part);
  if (part & 2) c->have_out = true;
}

}  // namespace fmmb
