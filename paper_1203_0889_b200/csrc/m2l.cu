// m2l.cu — the FP64 M2L kernel (reference: m2l, kernels.cpp:98-111, applied over the M2L list
// by KernelVisitor::m2l_pair, traversal.hpp:143-152). See expansions.cu for the conventions.
#include "expansions.cuh"

namespace fmmb {
namespace {

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

// ---------------------------------------------------------------- register M2L (p <= 6) ----
// Dt_g = g! D_g = d^g(1/|R|) computed in registers by the reference's degree recurrence
// rescaled by g! (multi_index.cpp:64-83 times g!):
//   n r^2 Dt_g = -(2n-1) sum_d g_d r_d Dt_{g-e_d} - (n-1) sum_d g_d (g_d - 1) Dt_{g-2e_d},
// every index and coefficient a compile-time constant; then the fully unrolled folded
// contraction Lambda_b += M_a Dt_{a+b} with Lambda in registers (one FMA per term). Lane =
// source, warp = target; the lane partials are reduced through shared memory per target.
// Row stride (doubles) of the staged multipoles: even (16-B aligned rows for cp.async) with an
// odd half, so a quarter-warp's LDS.128 of 8 distinct rows hits 8 distinct bank groups.
constexpr int m2l_row_stride(int n) {
  int s = n + (n & 1);
  return (s / 2) % 2 == 1 ? s : s + 2;
}

template <int P>
__device__ __forceinline__ void derivs_reg(double rx, double ry, double rz, double (&D)[MI<P>::N]) {
  using T = MI<P>;
  const double r2 = (rx * rx + ry * ry) + rz * rz;
  D[0] = rsqrt(r2);
  const double inv_r2 = D[0] * D[0];
  double rk[3][P];  // k * r_d
#pragma unroll
  for (int k = 0; k < P; ++k) {
    rk[0][k] = double(k) * rx;
    rk[1][k] = double(k) * ry;
    rk[2][k] = double(k) * rz;
  }
  double an[P];  // -(2n-1)/(n r^2); the s2 weight -(n-1)/(n r^2) = an * (n-1)/(2n-1) is folded
#pragma unroll
  for (int n = 1; n < P; ++n) an[n] = (-double(2 * n - 1) / double(n)) * inv_r2;
  static_for<T::N>([&](auto I) {
    constexpr int i = decltype(I)::value;
    if constexpr (i > 0) {
      constexpr int a = T::ea(i), b = T::eb(i), c = T::ec(i), n = T::deg(i);
      constexpr double cn = double(n - 1) / double(2 * n - 1);
      double acc = 0.0;
      if constexpr (a >= 1) acc = fma(rk[0][a], D[index_of(a - 1, b, c)], acc);
      if constexpr (b >= 1) acc = fma(rk[1][b], D[index_of(a, b - 1, c)], acc);
      if constexpr (c >= 1) acc = fma(rk[2][c], D[index_of(a, b, c - 1)], acc);
      if constexpr (a >= 2) acc = fma(double(a * (a - 1)) * cn, D[index_of(a - 2, b, c)], acc);
      if constexpr (b >= 2) acc = fma(double(b * (b - 1)) * cn, D[index_of(a, b - 2, c)], acc);
      if constexpr (c >= 2) acc = fma(double(c * (c - 1)) * cn, D[index_of(a, b, c - 2)], acc);
      D[i] = an[n] * acc;
    }
  });
}

template <int P>
__global__ void __launch_bounds__(128, 2)
k_m2l_reg(const int32_t* __restrict__ targets, int64_t ntargets, const int64_t* __restrict__ off,
          const int32_t* __restrict__ src, const double4* __restrict__ cr, const double* __restrict__ M,
          double* __restrict__ L) {
  using T = MI<P>;
  constexpr int N = T::N, S = m2l_row_stride(N);
  extern __shared__ double smem[];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* sR = smem + (size_t)w * 32 * S;  // per-warp source rows, then reduction rows
  const int64_t wid = blockIdx.x * 4ll + w;
  if (wid >= ntargets) return;
  const int32_t t = targets[wid];
  const double4 ct = cr[t];
  const int64_t l0 = off[t], l1 = off[t + 1];
  double lam[N];
#pragma unroll
  for (int i = 0; i < N; ++i) lam[i] = 0.0;
  static_assert((N * 8) % 16 == 0 || N % 2 == 1, "row copy granularity");
  int32_t s_next = (l0 + lane < l1) ? src[l0 + lane] : t;
  for (int64_t base = l0; base < l1; base += 32) {
    const int64_t k = base + lane;
    const bool valid = k < l1;
    const int32_t s = s_next;
    // stage this lane's source multipole (async; hidden behind the Dt recurrence)
    if (!valid) {
      for (int e = 0; e < N; ++e) sR[lane * S + e] = 0.0;  // tail lanes contribute nothing
    } else {
      const char* row = reinterpret_cast<const char*>(M + (int64_t)s * N);
      const unsigned dst = static_cast<unsigned>(__cvta_generic_to_shared(sR + lane * S));
      if constexpr ((N * 8) % 16 == 0) {
#pragma unroll
        for (int e = 0; e < N * 8; e += 16)
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(dst + e), "l"(row + e));
      } else {
#pragma unroll
        for (int e = 0; e < N * 8; e += 8)
          asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(dst + e), "l"(row + e));
      }
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
    if (base + 32 + lane < l1) s_next = src[base + 32 + lane];
    double rx = 1.0, ry = 0.0, rz = 0.0;
    if (valid) {
      const double4 cs = cr[s];
      rx = cs.x - ct.x;  // R = source centre - target centre (traversal.hpp:146)
      ry = cs.y - ct.y;
      rz = cs.z - ct.z;
    }
    double D[N];
    derivs_reg<P>(rx, ry, rz, D);
    asm volatile("cp.async.wait_all;\n" ::: "memory");
    __syncwarp();
    const double* Ms = sR + lane * S;
    auto contract = [&](auto IA, const double m) {
      constexpr int ia = decltype(IA)::value;
      constexpr int aa = T::ea(ia), ab = T::eb(ia), ac = T::ec(ia), da = T::deg(ia);
      static_for<N>([&](auto IB) {
        constexpr int ib = decltype(IB)::value;
        if constexpr (da + T::deg(ib) <= P - 1) {
          constexpr int ig = index_of(aa + T::ea(ib), ab + T::eb(ib), ac + T::ec(ib));
          lam[ib] = fma(m, D[ig], lam[ib]);
        }
      });
    };
    // 16-B loads of the staged row (conflict-free: S/2 is odd), two coefficients at a time
    static_for<N / 2>([&](auto IP) {
      constexpr int i0 = 2 * decltype(IP)::value;
      const double2 mm = *reinterpret_cast<const double2*>(Ms + i0);
      contract(std::integral_constant<int, i0>{}, mm.x);
      contract(std::integral_constant<int, i0 + 1>{}, mm.y);
    });
    if constexpr (N & 1) contract(std::integral_constant<int, N - 1>{}, Ms[N - 1]);
    __syncwarp();  // every lane done reading sR before the next chunk's copies land
  }
  // reduce the 32 lane partials (shared-memory transpose), then L_b += (-1)^{|b|}/b! Lambda_b
#pragma unroll
  for (int i = 0; i < N; ++i) sR[lane * S + i] = lam[i];
  __syncwarp();
  double* Lt = L + (int64_t)t * N;
  for (int i = lane; i < N; i += 32) {
    double acc = 0.0;
#pragma unroll 8
    for (int j = 0; j < 32; ++j) acc += sR[j * S + i];
    int n = 0;
    while (n_coef(n + 1) <= i) ++n;
    int r = i - n_coef(n), a = 0;
    while (r >= n - a + 1) { r -= n - a + 1; ++a; }
    const int bexp = r, cexp = n - a - r;
    double f = 1.0;
    for (int q = 2; q <= a; ++q) f *= q;
    for (int q = 2; q <= bexp; ++q) f *= q;
    for (int q = 2; q <= cexp; ++q) f *= q;
    Lt[i] += ((n & 1) ? -acc : acc) / f;
  }
}

template <int P>
struct M2L {
  static void run(fmm_ctx* c, cudaStream_t s) {
    if constexpr (P <= 6) {
      constexpr int S = m2l_row_stride(MI<P>::N);
      const size_t smem = sizeof(double) * 4 * 32 * S;
      static bool attr = false;
      if (!attr) {
        CK(cudaFuncSetAttribute(k_m2l_reg<P>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        attr = true;
      }
      if (c->n_m2l_targets == 0) return;
      k_m2l_reg<P><<<ceil_div(c->n_m2l_targets, 4), 128, smem, s>>>(c->m2l_targets.p, c->n_m2l_targets, c->m2l_off.p,
                                                                    c->m2l_src.p, c->c_cr.p, c->M.p, c->L.p);
      CK_LAUNCH("k_m2l_reg");
      c->kernel_launches += 1;
      return;
    }
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

}  // namespace

void run_m2l(fmm_ctx* c, cudaStream_t s) {
  if (!c->have_lists) fail(FMM_ERR_STATE, "m2l: no interaction lists");
  if (!c->have_M) fail(FMM_ERR_STATE, "m2l: no multipoles (run upward first)");
  dispatch_order<M2L>(c->cfg.order, c, s);
  c->have_L = true;
}

}  // namespace fmmb
