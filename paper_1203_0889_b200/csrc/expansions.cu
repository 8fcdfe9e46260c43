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
  const double4 c = cr[leaf];
  const int32_t b0 = bb[leaf], b1 = be[leaf];
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
      for (int k = 1; k < P; ++k) {
        L[k] = L[k - 1] * vx / k;
        L[P + k] = L[P + k - 1] * vy / k;
        L[2 * P + k] = L[2 * P + k - 1] * vz / k;
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

// ------------------------------------------------------------------------------ M2M ----
// One CTA per cell of one level; warp k translates child k (staged multipole + power lines
// d^k/k! of its shift) into a shared-memory partial, and the partials are summed in child
// order k = 0..count-1 (the reference's accumulation order, traversal.cpp:44-47).
template <int P>
__global__ void __launch_bounds__(256)
k_m2m(int32_t cbeg, int32_t cend, const int32_t* __restrict__ cb, const int32_t* __restrict__ cc,
      const double4* __restrict__ cr, double* __restrict__ M, const int32_t* __restrict__ owner, int32_t want) {
  using T = MI<P>;
  constexpr int N = T::N;
  __shared__ double sD[8][3 * P];
  __shared__ double sM[8][N];
  __shared__ double part[8][N];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int32_t ci = cbeg + blockIdx.x;
  if (ci >= cend) return;
  const int32_t nch = cc[ci];
  if (nch == 0) return;  // uniform over the CTA
  if (owner && owner[ci] != want) return;  // sharded: only this rank's (or the shared) cells
  if (w < nch) {
    const double4 pc = cr[ci];
    const int32_t child = cb[ci] + w;
    const double4 c4 = cr[child];
    if (lane < 3) {
      const double d = lane == 0 ? c4.x - pc.x : (lane == 1 ? c4.y - pc.y : c4.z - pc.z);
      double* L = sD[w] + lane * P;
      L[0] = 1.0;
      for (int k = 1; k < P; ++k) L[k] = L[k - 1] * d / k;
    }
    for (int i = lane; i < N; i += 32) sM[w][i] = M[(int64_t)child * N + i];
    __syncwarp();
    for (int i = lane; i < N; i += 32) {
      int n = 0;
      while (n_coef(n + 1) <= i) ++n;
      int r = i - n_coef(n), a = 0;
      while (r >= n - a + 1) { r -= n - a + 1; ++a; }
      const int bb_ = r, cc_ = n - a - r;
      double s = 0.0;
      for (int ax = 0; ax <= a; ++ax)
        for (int ay = 0; ay <= bb_; ++ay) {
          const double xy = sD[w][a - ax] * sD[w][P + bb_ - ay];
          for (int az = 0; az <= cc_; ++az) s += sM[w][index_of(ax, ay, az)] * (xy * sD[w][2 * P + cc_ - az]);
        }
      part[w][i] = s;
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < N; i += blockDim.x) {
    double s = 0.0;
    for (int k = 0; k < nch; ++k) s += part[k][i];
    M[(int64_t)ci * N + i] = s;
  }
}

// ------------------------------------------------------------------------------ L2L ----
// Warp per cell of one level (>= 1): child_a += sum_d parent_{a+d} ((a+d)!/a!) d^d/d!,
// parent local staged in shared memory.
template <int P>
__global__ void __launch_bounds__(128)
k_l2l(int32_t cbeg, int32_t cend, const int32_t* __restrict__ par, const double4* __restrict__ cr,
      double* __restrict__ L) {
  using T = MI<P>;
  constexpr int N = T::N;
  __shared__ double sD[4][3 * P];
  __shared__ double sL[4][N];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int32_t ci = cbeg + blockIdx.x * 4 + w;
  if (ci >= cend) return;
  const int32_t pi = par[ci];
  const double4 c = cr[ci], pc = cr[pi];
  if (lane < 3) {
    const double d = lane == 0 ? c.x - pc.x : (lane == 1 ? c.y - pc.y : c.z - pc.z);
    double* Ld = sD[w] + lane * P;
    Ld[0] = 1.0;
    for (int k = 1; k < P; ++k) Ld[k] = Ld[k - 1] * d / k;
  }
  for (int i = lane; i < N; i += 32) sL[w][i] = L[(int64_t)pi * N + i];
  __syncwarp();
  __shared__ double sCw[4][P][P];  // (a+d)!/a! (per warp)
  for (int k = lane; k < P * P; k += 32) {
    const int a = k / P, d = k % P;
    double v = 1.0;
    for (int q = a + 1; q <= a + d; ++q) v *= q;
    sCw[w][a][d] = v;
  }
  __syncwarp();
  const auto& sC = sCw[w];
  double* Lc = L + (int64_t)ci * N;
  for (int i = lane; i < N; i += 32) {
    int n = 0;
    while (n_coef(n + 1) <= i) ++n;
    int r = i - n_coef(n), a = 0;
    while (r >= n - a + 1) { r -= n - a + 1; ++a; }
    const int b = r, cz = n - a - r;
    double s = 0.0;
    for (int dx = 0; dx + n < P; ++dx)
      for (int dy = 0; dx + dy + n < P; ++dy) {
        const double wxy = sC[a][dx] * sC[b][dy];
        const double pxy = sD[w][dx] * sD[w][P + dy];
        for (int dz = 0; dx + dy + dz + n < P; ++dz)
          s += sL[w][index_of(a + dx, b + dy, cz + dz)] * (wxy * sC[cz][dz]) * (pxy * sD[w][2 * P + dz]);
      }
    Lc[i] += s;
  }
}

// ------------------------------------------------------------------------------ L2P ----
// Warp per leaf, lane per body; phi_out = phi_near + sum_b L_b (x-c)^b and
// acc_out = acc_near - grad (extension). Leaf L staged in shared memory (broadcast reads).
template <int P>
__global__ void __launch_bounds__(128)
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
    double X[P], Y[P], Z[P];
    X[0] = Y[0] = Z[0] = 1.0;
#pragma unroll
    for (int k = 1; k < P; ++k) {
      X[k] = X[k - 1] * (b.x - c.x);
      Y[k] = Y[k - 1] * (b.y - c.y);
      Z[k] = Z[k - 1] * (b.z - c.z);
    }
    double ph = 0.0, gx = 0.0, gy = 0.0, gz = 0.0;
    static_for<N>([&](auto I) {
      constexpr int ii = decltype(I)::value;
      constexpr int a = T::ea(ii), e = T::eb(ii), f = T::ec(ii);
      const double l = sL[w][ii];
      ph = fma(l, X[a] * Y[e] * Z[f], ph);
      if constexpr (a > 0) gx = fma(l * double(a), X[a - 1] * Y[e] * Z[f], gx);
      if constexpr (e > 0) gy = fma(l * double(e), X[a] * Y[e - 1] * Z[f], gy);
      if constexpr (f > 0) gz = fma(l * double(f), X[a] * Y[e] * Z[f - 1], gz);
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
      k_m2m<P><<<e - b, 256, 0, s>>>(b, e, c->c_child_begin.p, c->c_child_count.p, c->c_cr.p, M, owner, want);
      CK_LAUNCH("k_m2m");
      ++launches;
    }
    c->kernel_launches += launches;
  }
};

template <int P>
struct Downward {
  static void run(fmm_ctx* c, cudaStream_t s) {
    const int N = MI<P>::N;
    int launches = 0;
    for (int l = 1; l <= c->depth; ++l) {
      const int32_t b = c->level_start[l], e = c->level_start[l + 1];
      if (e <= b) continue;
      k_l2l<P><<<ceil_div(e - b, 4), 128, 0, s>>>(b, e, c->c_parent.p, c->c_cr.p, c->L.p);
      CK_LAUNCH("k_l2l");
      ++launches;
    }
    (void)N;
    if (c->nwl > 0)
    k_l2p<P><<<ceil_div(c->nwl, 4), 128, 0, s>>>(c->wl, c->nwl, c->c_body_begin.p, c->c_body_end.p,
                                                     c->c_cr.p, c->bodies.p, c->L.p, c->phi_p2p.p, c->acc_p2p.p,
                                                     c->phi.ensure(c->N), c->acc.ensure(3 * c->N),
                                                     c->cfg.with_acc ? 1 : 0);
    CK_LAUNCH("k_l2p");
    c->kernel_launches += launches + 1;
  }
};

}  // namespace

void run_upward(fmm_ctx* c, cudaStream_t s, int mode) {
  if (!c->have_tree) fail(FMM_ERR_STATE, "upward: no tree");
  if (mode != 0 && !c->shard_planned) fail(FMM_ERR_STATE, "sharded upward before the partition (run traverse)");
  dispatch_order<Upward>(c->cfg.order, c, s, mode);
  c->have_M = true;
}

void run_downward(fmm_ctx* c, cudaStream_t s) {
  if (!c->have_tree) fail(FMM_ERR_STATE, "downward: no tree");
  dispatch_order<Downward>(c->cfg.order, c, s);
  c->have_out = true;
}

}  // namespace fmmb
