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
#include "context.cuh"

namespace fmmb {
namespace {

constexpr int odd_stride(int n) { return (n % 2 == 0) ? n + 1 : n; }

// ---------------------------------------------------------------- derivative table ----
// Reference recurrence (multi_index.cpp:64-83) into row[0..N), then scaled by g! when
// `scaled` (Dt). row has unit stride (a lane-private shared-memory row).
template <int P, bool kScaled>
__device__ __forceinline__ void derivs_row(double rx, double ry, double rz, double* row) {
  using T = MI<P>;
  const double r2 = (rx * rx + ry * ry) + rz * rz;
  const double inv_r2 = 1.0 / r2;
  row[0] = 1.0 / sqrt(r2);
  static_for<T::N>([&](auto I) {
    constexpr int i = decltype(I)::value;
    if constexpr (i > 0) {
      constexpr int a = T::ea(i), b = T::eb(i), c = T::ec(i), n = T::deg(i);
      double s1 = 0.0, s2 = 0.0;
      if constexpr (a >= 1) s1 += rx * row[index_of(a - 1, b, c)];
      if constexpr (a >= 2) s2 += row[index_of(a - 2, b, c)];
      if constexpr (b >= 1) s1 += ry * row[index_of(a, b - 1, c)];
      if constexpr (b >= 2) s2 += row[index_of(a, b - 2, c)];
      if constexpr (c >= 1) s1 += rz * row[index_of(a, b, c - 1)];
      if constexpr (c >= 2) s2 += row[index_of(a, b, c - 2)];
      row[i] = -(double(2 * n - 1) * s1 + double(n - 1) * s2) * inv_r2 / double(n);
    }
  });
  if constexpr (kScaled) {
    static_for<T::N>([&](auto I) {
      constexpr int i = decltype(I)::value;
      if constexpr (T::fact(i) != 1.0) row[i] *= T::fact(i);
    });
  }
}

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
// Warp per non-leaf cell of one level; children accumulated in order k = 0..count-1, each
// child's multipole staged in shared memory with the power lines d^k/k! of its shift.
template <int P>
__global__ void __launch_bounds__(128)
k_m2m(int32_t cbeg, int32_t cend, const int32_t* __restrict__ cb, const int32_t* __restrict__ cc,
      const double4* __restrict__ cr, double* __restrict__ M) {
  using T = MI<P>;
  constexpr int N = T::N;
  __shared__ double sD[4][3 * P];
  __shared__ double sM[4][N];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int32_t ci = cbeg + blockIdx.x * 4 + w;
  if (ci >= cend) return;
  const int32_t nch = cc[ci];
  if (nch == 0) return;
  const double4 pc = cr[ci];
  constexpr int KPL = (N + 31) / 32;
  double acc[KPL];
  int ea[KPL], eb[KPL], ec[KPL];
#pragma unroll
  for (int k = 0; k < KPL; ++k) {
    acc[k] = 0.0;
    const int i = lane + 32 * k;
    int n = 0;
    if (i < N) {
      while (n_coef(n + 1) <= i) ++n;
      int r = i - n_coef(n), a = 0;
      while (r >= n - a + 1) { r -= n - a + 1; ++a; }
      ea[k] = a;
      eb[k] = r;
      ec[k] = n - a - r;
    }
  }
  const int32_t c0 = cb[ci];
  for (int32_t ch = 0; ch < nch; ++ch) {
    const int32_t child = c0 + ch;
    const double4 cc4 = cr[child];
    if (lane < 3) {
      const double d = lane == 0 ? cc4.x - pc.x : (lane == 1 ? cc4.y - pc.y : cc4.z - pc.z);
      double* L = sD[w] + lane * P;
      L[0] = 1.0;
      for (int k = 1; k < P; ++k) L[k] = L[k - 1] * d / k;
    }
    for (int i = lane; i < N; i += 32) sM[w][i] = M[(int64_t)child * N + i];
    __syncwarp();
#pragma unroll
    for (int k = 0; k < KPL; ++k) {
      const int i = lane + 32 * k;
      if (i < N) {
        const int a = ea[k], bb_ = eb[k], cc_ = ec[k];
        double s = 0.0;
        for (int ax = 0; ax <= a; ++ax)
          for (int ay = 0; ay <= bb_; ++ay) {
            const double xy = sD[w][a - ax] * sD[w][P + bb_ - ay];
            for (int az = 0; az <= cc_; ++az) s += sM[w][index_of(ax, ay, az)] * (xy * sD[w][2 * P + cc_ - az]);
          }
        acc[k] += s;
      }
    }
    __syncwarp();
  }
#pragma unroll
  for (int k = 0; k < KPL; ++k) {
    const int i = lane + 32 * k;
    if (i < N) M[(int64_t)ci * N + i] = acc[k];
  }
}

// ------------------------------------------------------------------------------ M2L ----
template <int P>
struct M2LCfg {
  static constexpr int N = MI<P>::N;
  static constexpr int S = odd_stride(N);
  static constexpr int kWarps = (P <= 6) ? 4 : 2;
  // Lambda in registers when it fits; otherwise blocks of kBlk coefficients in shared memory
  static constexpr bool kRegs = N <= 56;
  static constexpr int kBlk = kRegs ? N : 40;
};

template <int P>
__global__ void __launch_bounds__(32 * M2LCfg<P>::kWarps)
k_m2l(const int32_t* __restrict__ targets, int64_t ntargets, const int64_t* __restrict__ off,
      const int32_t* __restrict__ src, const double4* __restrict__ cr, const double* __restrict__ M,
      double* __restrict__ L) {
  using T = MI<P>;
  using C = M2LCfg<P>;
  constexpr int N = C::N, S = C::S;
  extern __shared__ double smem[];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* sD = smem + (size_t)w * 32 * S * (C::kRegs ? 1 : 2);  // Dt rows (+ Lambda rows)
  double* myD = sD + lane * S;
  double* myLam = sD + 32 * S + lane * S;  // only when !kRegs
  const int64_t wid = blockIdx.x * (int64_t)C::kWarps + w;
  if (wid >= ntargets) return;
  const int32_t t = targets[wid];
  const double4 ct = cr[t];
  const int64_t l0 = off[t], l1 = off[t + 1];

  double lam[C::kBlk];
  if constexpr (C::kRegs) {
#pragma unroll
    for (int i = 0; i < N; ++i) lam[i] = 0.0;
  } else {
    for (int i = 0; i < N; ++i) myLam[i] = 0.0;
  }
  for (int64_t base = l0; base < l1; base += 32) {
    const int64_t k = base + lane;
    const bool valid = k < l1;
    const int32_t s = valid ? src[k] : t;
    double rx = 1.0, ry = 0.0, rz = 0.0;
    if (valid) {
      const double4 cs = cr[s];
      rx = cs.x - ct.x;  // R = source centre - target centre (traversal.hpp:146)
      ry = cs.y - ct.y;
      rz = cs.z - ct.z;
    }
    derivs_row<P, true>(rx, ry, rz, myD);
    const double* Ms = M + (int64_t)s * N;
    const double mscale = valid ? 1.0 : 0.0;
    if constexpr (C::kRegs) {
      static_for<N>([&](auto IA) {
        constexpr int ia = decltype(IA)::value;
        constexpr int aa = T::ea(ia), ab = T::eb(ia), ac = T::ec(ia), da = T::deg(ia);
        const double m = __ldg(Ms + ia) * mscale;
        static_for<N>([&](auto IB) {
          constexpr int ib = decltype(IB)::value;
          if constexpr (da + T::deg(ib) <= P - 1) {
            constexpr int ig = index_of(aa + T::ea(ib), ab + T::eb(ib), ac + T::ec(ib));
            lam[ib] = fma(m, myD[ig], lam[ib]);
          }
        });
      });
    } else {
      // beta blocks of kBlk coefficients; Lambda block round-trips through shared memory
      static_for<(N + C::kBlk - 1) / C::kBlk>([&](auto BI) {
        constexpr int b0 = decltype(BI)::value * C::kBlk;
        constexpr int b1 = (b0 + C::kBlk < N) ? b0 + C::kBlk : N;
        static_for<b1 - b0>([&](auto J) { lam[decltype(J)::value] = myLam[b0 + decltype(J)::value]; });
        static_for<N>([&](auto IA) {
          constexpr int ia = decltype(IA)::value;
          constexpr int aa = T::ea(ia), ab = T::eb(ia), ac = T::ec(ia), da = T::deg(ia);
          if constexpr (da + T::deg(b0) <= P - 1) {
            const double m = __ldg(Ms + ia) * mscale;
            static_for<b1 - b0>([&](auto J) {
              constexpr int ib = b0 + decltype(J)::value;
              if constexpr (da + T::deg(ib) <= P - 1) {
                constexpr int ig = index_of(aa + T::ea(ib), ab + T::eb(ib), ac + T::ec(ib));
                lam[ib - b0] = fma(m, myD[ig], lam[ib - b0]);
              }
            });
          }
        });
        static_for<b1 - b0>([&](auto J) { myLam[b0 + decltype(J)::value] = lam[decltype(J)::value]; });
      });
    }
  }
  // warp reduction of the per-lane partials, then L_b += (-1)^{|b|}/b! * Lambda_b
  __syncwarp();
  if constexpr (C::kRegs) {
#pragma unroll
    for (int i = 0; i < N; ++i) myD[i] = lam[i];
  } else {
    for (int i = 0; i < N; ++i) myD[i] = myLam[i];
  }
  __syncwarp();
  double* Lt = L + (int64_t)t * N;
  for (int i = lane; i < N; i += 32) {
    double s = 0.0;
    for (int j = 0; j < 32; ++j) s += sD[j * S + i];
    int n = 0;
    while (n_coef(n + 1) <= i) ++n;
    // 1/b! for coefficient i
    int r = i - n_coef(n), a = 0;
    while (r >= n - a + 1) { r -= n - a + 1; ++a; }
    const int bexp = r, cexp = n - a - r;
    double f = 1.0;
    for (int q = 2; q <= a; ++q) f *= q;
    for (int q = 2; q <= bexp; ++q) f *= q;
    for (int q = 2; q <= cexp; ++q) f *= q;
    const double sgn = (n & 1) ? -1.0 : 1.0;
    Lt[i] += sgn * s / f;
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
  double fact[P];  // k! for k < P
  fact[0] = 1.0;
#pragma unroll
  for (int k = 1; k < P; ++k) fact[k] = fact[k - 1] * k;
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
        const double wxy = (fact[a + dx] / fact[a]) * (fact[b + dy] / fact[b]);
        const double pxy = sD[w][dx] * sD[w][P + dy];
        for (int dz = 0; dx + dy + dz + n < P; ++dz) {
          const double w_ = wxy * (fact[cz + dz] / fact[cz]);
          s += sL[w][index_of(a + dx, b + dy, cz + dz)] * w_ * (pxy * sD[w][2 * P + dz]);
        }
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


// ------------------------------------------------------------ single-operator kernels ----
// Thread per instance; the same formulas as the tree kernels above (fmm_op_* entry points,
// used by the operator-level parity tests mirroring proj/tests/test_kernels.cpp).
__device__ __forceinline__ void exps_of(int i, int& a, int& b, int& c) {
  int n = 0;
  while (n_coef(n + 1) <= i) ++n;
  int r = i - n_coef(n);
  a = 0;
  while (r >= n - a + 1) { r -= n - a + 1; ++a; }
  b = r;
  c = n - a - r;
}
__device__ __forceinline__ double dfact(int k) {
  double f = 1.0;
  for (int q = 2; q <= k; ++q) f *= q;
  return f;
}

template <int P>
__global__ void k_op(int kind, int64_t count, const int32_t* __restrict__ off, const double* __restrict__ in,
                     const double* __restrict__ v3, const double* __restrict__ xyzq, double* __restrict__ out,
                     double* __restrict__ out2) {
  using T = MI<P>;
  constexpr int N = T::N;
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= count) return;
  double row[N];
  if (kind == OP_DERIV) {
    derivs_row<P, false>(v3[3 * k], v3[3 * k + 1], v3[3 * k + 2], row);
    for (int i = 0; i < N; ++i) out[k * N + i] = row[i];
  } else if (kind == OP_M2L) {
    derivs_row<P, true>(v3[3 * k], v3[3 * k + 1], v3[3 * k + 2], row);
    const double* Ms = in + k * N;
    double lam[N];
    for (int i = 0; i < N; ++i) lam[i] = 0.0;
    static_for<N>([&](auto IA) {
      constexpr int ia = decltype(IA)::value;
      constexpr int aa = T::ea(ia), ab = T::eb(ia), ac = T::ec(ia), da = T::deg(ia);
      const double m = Ms[ia];
      static_for<N>([&](auto IB) {
        constexpr int ib = decltype(IB)::value;
        if constexpr (da + T::deg(ib) <= P - 1) {
          constexpr int ig = index_of(aa + T::ea(ib), ab + T::eb(ib), ac + T::ec(ib));
          lam[ib] = fma(m, row[ig], lam[ib]);
        }
      });
    });
    for (int i = 0; i < N; ++i) {
      int a, b, c;
      exps_of(i, a, b, c);
      const double sgn = ((a + b + c) & 1) ? -1.0 : 1.0;
      out[k * N + i] += sgn * lam[i] / (dfact(a) * dfact(b) * dfact(c));
    }
  } else if (kind == OP_EVAL) {
    // evaluate_multipole (kernels.cpp:197-208): sum_a (-1)^{|a|} a! M_a D_a(x - c)
    const double rx = v3[6 * k] - v3[6 * k + 3], ry = v3[6 * k + 1] - v3[6 * k + 4], rz = v3[6 * k + 2] - v3[6 * k + 5];
    derivs_row<P, true>(rx, ry, rz, row);
    double phi = 0.0;
    for (int i = 0; i < N; ++i) {
      int a, b, c;
      exps_of(i, a, b, c);
      phi += (((a + b + c) & 1) ? -1.0 : 1.0) * in[k * N + i] * row[i];
    }
    out[k] = phi;
  } else if (kind == OP_M2M || kind == OP_L2L) {
    const double d[3] = {v3[3 * k], v3[3 * k + 1], v3[3 * k + 2]};
    double X[3][P];
    for (int ax = 0; ax < 3; ++ax) {
      X[ax][0] = 1.0;
      for (int q = 1; q < P; ++q) X[ax][q] = X[ax][q - 1] * d[ax] / q;
    }
    const double* src = in + k * N;
    for (int i = 0; i < N; ++i) {
      int a, b, c;
      exps_of(i, a, b, c);
      double s = 0.0;
      if (kind == OP_M2M) {
        for (int ax = 0; ax <= a; ++ax)
          for (int ay = 0; ay <= b; ++ay)
            for (int az = 0; az <= c; ++az) s += src[index_of(ax, ay, az)] * (X[0][a - ax] * X[1][b - ay] * X[2][c - az]);
      } else {
        for (int dx = 0; dx + a + b + c < P; ++dx)
          for (int dy = 0; dx + dy + a + b + c < P; ++dy)
            for (int dz = 0; dx + dy + dz + a + b + c < P; ++dz) {
              const double w_ = (dfact(a + dx) / dfact(a)) * (dfact(b + dy) / dfact(b)) * (dfact(c + dz) / dfact(c));
              s += src[index_of(a + dx, b + dy, c + dz)] * w_ * (X[0][dx] * X[1][dy] * X[2][dz]);
            }
      }
      out[k * N + i] += s;
    }
  } else if (kind == OP_P2M) {
    double acc[N];
    for (int i = 0; i < N; ++i) acc[i] = 0.0;
    for (int32_t j = off[k]; j < off[k + 1]; ++j) {
      const double v[3] = {xyzq[4 * j] - v3[3 * k], xyzq[4 * j + 1] - v3[3 * k + 1], xyzq[4 * j + 2] - v3[3 * k + 2]};
      double X[3][P];
      for (int ax = 0; ax < 3; ++ax) {
        X[ax][0] = 1.0;
        for (int q = 1; q < P; ++q) X[ax][q] = X[ax][q - 1] * v[ax] / q;
      }
      for (int i = 0; i < N; ++i) {
        int a, b, c;
        exps_of(i, a, b, c);
        acc[i] += xyzq[4 * j + 3] * (X[0][a] * X[1][b] * X[2][c]);
      }
    }
    for (int i = 0; i < N; ++i) out[k * N + i] += acc[i];
  } else if (kind == OP_L2P) {
    const double* Lk = in + k * N;
    for (int32_t j = off[k]; j < off[k + 1]; ++j) {
      double X[P], Y[P], Z[P];
      X[0] = Y[0] = Z[0] = 1.0;
      for (int q = 1; q < P; ++q) {
        X[q] = X[q - 1] * (xyzq[4 * j] - v3[3 * k]);
        Y[q] = Y[q - 1] * (xyzq[4 * j + 1] - v3[3 * k + 1]);
        Z[q] = Z[q - 1] * (xyzq[4 * j + 2] - v3[3 * k + 2]);
      }
      double ph = 0.0, gx = 0.0, gy = 0.0, gz = 0.0;
      static_for<N>([&](auto I) {
        constexpr int ii = decltype(I)::value;
        constexpr int a = T::ea(ii), e = T::eb(ii), f = T::ec(ii);
        const double l = Lk[ii];
        ph = fma(l, X[a] * Y[e] * Z[f], ph);
        if constexpr (a > 0) gx = fma(l * double(a), X[a - 1] * Y[e] * Z[f], gx);
        if constexpr (e > 0) gy = fma(l * double(e), X[a] * Y[e - 1] * Z[f], gy);
        if constexpr (f > 0) gz = fma(l * double(f), X[a] * Y[e] * Z[f - 1], gz);
      });
      out[j] += ph;
      if (out2) {
        out2[3 * j] -= gx;
        out2[3 * j + 1] -= gy;
        out2[3 * j + 2] -= gz;
      }
    }
  }
}

template <int P>
struct OpRun {
  static void run(int kind, int64_t count, const int32_t* off, const double* in, const double* v3,
                  const double* xyzq, double* out, double* out2) {
    k_op<P><<<ceil_div(count, 64), 64>>>(kind, count, off, in, v3, xyzq, out, out2);
    CK_LAUNCH("k_op");
  }
};

// --------------------------------------------------------------------- launchers ------
template <int P>
struct Upward {
  static void run(fmm_ctx* c, cudaStream_t s) {
    const int N = MI<P>::N;
    double* M = c->M.ensure((size_t)c->ncells * N);
    k_p2m<P><<<ceil_div(c->nleaves, 4), 128, 0, s>>>(c->leaves.p, c->nleaves, c->c_body_begin.p, c->c_body_end.p,
                                                     c->c_cr.p, c->bodies.p, M);
    CK_LAUNCH("k_p2m");
    int launches = 1;
    for (int l = c->depth - 1; l >= 0; --l) {
      const int32_t b = c->level_start[l], e = c->level_start[l + 1];
      if (e <= b) continue;
      k_m2m<P><<<ceil_div(e - b, 4), 128, 0, s>>>(b, e, c->c_child_begin.p, c->c_child_count.p, c->c_cr.p, M);
      CK_LAUNCH("k_m2m");
      ++launches;
    }
    c->kernel_launches += launches;
  }
};

template <int P>
struct M2L {
  static void run(fmm_ctx* c, cudaStream_t s) {
    using C = M2LCfg<P>;
    const size_t smem = sizeof(double) * C::kWarps * 32 * C::S * (C::kRegs ? 1 : 2);
    static bool attr_set = false;
    if (!attr_set) {
      CK(cudaFuncSetAttribute(k_m2l<P>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      attr_set = true;
    }
    if (c->n_m2l_targets == 0) return;
    k_m2l<P><<<ceil_div(c->n_m2l_targets, C::kWarps), 32 * C::kWarps, smem, s>>>(
        c->m2l_targets.p, c->n_m2l_targets, c->m2l_off.p, c->m2l_src.p, c->c_cr.p, c->M.p, c->L.p);
    CK_LAUNCH("k_m2l");
    c->kernel_launches += 1;
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
    k_l2p<P><<<ceil_div(c->nleaves, 4), 128, 0, s>>>(c->leaves.p, c->nleaves, c->c_body_begin.p, c->c_body_end.p,
                                                     c->c_cr.p, c->bodies.p, c->L.p, c->phi_p2p.p, c->acc_p2p.p,
                                                     c->phi.ensure(c->N), c->acc.ensure(3 * c->N),
                                                     c->cfg.with_acc ? 1 : 0);
    CK_LAUNCH("k_l2p");
    c->kernel_launches += launches + 1;
  }
};

}  // namespace

namespace {
template <class T>
struct DevCopy {
  T* p = nullptr;
  DevCopy(const T* h, size_t n, bool copy = true) {
    CK(cudaMalloc(&p, (n ? n : 1) * sizeof(T)));
    if (h && n && copy) CK(cudaMemcpy(p, h, n * sizeof(T), cudaMemcpyHostToDevice));
    else if (n) CK(cudaMemset(p, 0, n * sizeof(T)));
  }
  ~DevCopy() { cudaFree(p); }
  void back(T* h, size_t n) const { if (h && n) CK(cudaMemcpy(h, p, n * sizeof(T), cudaMemcpyDeviceToHost)); }
};
}  // namespace

void op_expansion(int kind, int order, int64_t count, const int32_t* offsets, const double* in,
                  const double* vec3, const double* xyzq, int64_t nbodies, double* out, double* out2) {
  if (count <= 0) return;
  const int N = n_coef(order);
  const int64_t nin = (kind == OP_P2M || kind == OP_DERIV) ? 0 : count * N;
  const int64_t nv = (kind == OP_EVAL) ? 6 * count : 3 * count;
  int64_t nout = count * N, nout2 = 0;
  if (kind == OP_L2P) { nout = nbodies; nout2 = out2 ? 3 * nbodies : 0; }
  if (kind == OP_EVAL) nout = count;
  const bool has_bodies = (kind == OP_P2M || kind == OP_L2P);
  DevCopy<int32_t> d_off(offsets, has_bodies ? count + 1 : 0);
  DevCopy<double> d_in(in, nin), d_v(vec3, nv), d_x(xyzq, has_bodies ? 4 * nbodies : 0);
  DevCopy<double> d_out(out, nout, kind != OP_DERIV && kind != OP_EVAL), d_out2(out2, nout2);
  dispatch_order<OpRun>(order, kind, count, d_off.p, d_in.p, d_v.p, d_x.p, d_out.p, nout2 ? d_out2.p : nullptr);
  CK(cudaDeviceSynchronize());
  d_out.back(out, nout);
  if (nout2) d_out2.back(out2, nout2);
}

void run_upward(fmm_ctx* c, cudaStream_t s) {
  if (!c->have_tree) fail(FMM_ERR_STATE, "upward: no tree");
  dispatch_order<Upward>(c->cfg.order, c, s);
  c->have_M = true;
}

void run_m2l(fmm_ctx* c, cudaStream_t s) {
  if (!c->have_lists) fail(FMM_ERR_STATE, "m2l: no interaction lists");
  if (!c->have_M) fail(FMM_ERR_STATE, "m2l: no multipoles (run upward first)");
  dispatch_order<M2L>(c->cfg.order, c, s);
  c->have_L = true;
}

void run_downward(fmm_ctx* c, cudaStream_t s) {
  if (!c->have_tree) fail(FMM_ERR_STATE, "downward: no tree");
  dispatch_order<Downward>(c->cfg.order, c, s);
  c->have_out = true;
}

}  // namespace fmmb
