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

}  // namespace

void run_m2l(fmm_ctx* c, cudaStream_t s) {
  if (!c->have_lists) fail(FMM_ERR_STATE, "m2l: no interaction lists");
  if (!c->have_M) fail(FMM_ERR_STATE, "m2l: no multipoles (run upward first)");
  dispatch_order<M2L>(c->cfg.order, c, s);
  c->have_L = true;
}

}  // namespace fmmb
