// common.cuh — shared device/host helpers for the B200 FMM: status/error plumbing,
// grow-only device buffers, the compile-time multi-index tables and static_for.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <mutex>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <utility>

#include "fmm_b200.h"

namespace fmmb {

// ------------------------------------------------------------ checked build -----------
// FMM_CHECKS=1 (tools/checked_build.sh): device-side bounds checks on the index streams the
// kernels dereference (bodies, cells, list entries, tile offsets). A failed check prints the
// site and traps, which the host sees as a CUDA error on the next synchronisation. The limits
// live in this TU's constant bank (each .cu file has its own copy; set_check_limits fills it
// before the TU's launches). compute-sanitizer is not available on the GPU pool, so this build,
// run over the whole GPU test suite, is the memory-safety evidence (profiles/r2_checked_build.log).
#ifndef FMM_CHECKS
#define FMM_CHECKS 0
#endif
struct CheckLimits {
  int64_t nbodies, ncells, n_m2l, n_p2p;
};
#if FMM_CHECKS
static __constant__ CheckLimits g_lim;
#define FMM_CHECK(cond, what)                                                                            \
  do {                                                                                                 \
    if (!(cond)) {                                                                                     \
      printf("FMM_CHECK failed: %s (%s:%d) block %d thread %d\n", what, __FILE__, __LINE__, blockIdx.x, \
             threadIdx.x);                                                                             \
      __trap();                                                                                        \
    }                                                                                                  \
  } while (0)
#define FMM_LIM(field) (::fmmb::g_lim.field)
// the constant bank is per process (shared by every context of this TU): it holds the maximum
// over the contexts seen so far, so concurrent contexts (sharded ranks on host threads) never see
// each other's smaller limits; the checks still catch any index past every live array
// static (internal linkage): each TU's copy updates that TU's own g_lim (an inline function would
// be merged across TUs by the linker and update only one of them)
template <class Ctx>
static void set_check_limits(const Ctx* c, cudaStream_t s) {
  static std::mutex mu;
  static CheckLimits cur{0, 0, 0, 0};
  std::lock_guard<std::mutex> lock(mu);
  const CheckLimits l{c->N > cur.nbodies ? c->N : cur.nbodies, c->ncells > cur.ncells ? c->ncells : cur.ncells,
                      c->n_m2l > cur.n_m2l ? c->n_m2l : cur.n_m2l, c->n_p2p > cur.n_p2p ? c->n_p2p : cur.n_p2p};
  if (l.nbodies == cur.nbodies && l.ncells == cur.ncells && l.n_m2l == cur.n_m2l && l.n_p2p == cur.n_p2p) return;
  cur = l;
  cudaMemcpyToSymbolAsync(g_lim, &cur, sizeof(cur), 0, cudaMemcpyHostToDevice, s);
  cudaStreamSynchronize(s);
}
#else
#define FMM_CHECK(cond, what) \
  do {                        \
  } while (0)
template <class Ctx>
static inline void set_check_limits(const Ctx*, cudaStream_t) {}
#endif

// ---------------------------------------------------------------- errors --------------
struct Error : std::runtime_error {
  int status;
  Error(int s, const std::string& m) : std::runtime_error(m), status(s) {}
};

[[noreturn]] inline void fail(int status, const std::string& msg) { throw Error(status, msg); }

inline void cuda_check(cudaError_t e, const char* what, const char* file, int line) {
  if (e != cudaSuccess) {
    const int st = (e == cudaErrorMemoryAllocation) ? FMM_ERR_OOM
                   : (e == cudaErrorNoDevice || e == cudaErrorInsufficientDriver) ? FMM_ERR_NO_DEVICE
                                                                                 : FMM_ERR_CUDA;
    fail(st, std::string("CUDA error in ") + what + " (" + file + ":" + std::to_string(line) +
                 "): " + cudaGetErrorString(e));
  }
}
#define CK(x) ::fmmb::cuda_check((x), #x, __FILE__, __LINE__)
#define CK_LAUNCH(name) ::fmmb::cuda_check(cudaGetLastError(), name, __FILE__, __LINE__)

inline const char* reference_message(int status) {
  switch (status) {
    case FMM_ERR_EMPTY_INPUT: return "empty input";
    case FMM_ERR_NCRIT: return "n_crit must be >= 1";
    case FMM_ERR_ORDER: return "expansion order must be >= 1";
    case FMM_ERR_LEVEL_OVERFLOW: return "level overflow";
    case FMM_ERR_SINGULAR_M2L: return "singular M2L displacement";
    case FMM_ERR_SINGULAR_EVAL: return "singular evaluation point";
    case FMM_ERR_CANNOT_SPLIT: return "cannot split leaf pair";
    case FMM_ERR_THETA: return "theta must be in (0,1)";
    default: return "error";
  }
}

// ------------------------------------------------------------- device buffers ---------
template <class T>
struct DBuf {
  T* p = nullptr;
  size_t cap = 0;
  DBuf() = default;
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  ~DBuf() {
    if (p) cudaFree(p);
  }
  // Grow-only; contents are NOT preserved when growing.
  T* ensure(size_t n) {
    if (n > cap) {
      if (p) CK(cudaFree(p));
      p = nullptr;
      cap = 0;
      size_t want = n + n / 8 + 16;
      CK(cudaMalloc(&p, want * sizeof(T)));
      cap = want;
    }
    return p;
  }
  T* get() const { return p; }
};

// ------------------------------------------------------------------ launch math --------
inline int ceil_div(long long a, long long b) { return static_cast<int>((a + b - 1) / b); }

// --------------------------------------------------------------- compile-time loops ----
template <int... Is, class F>
__host__ __device__ __forceinline__ void static_for_impl(std::integer_sequence<int, Is...>, F&& f) {
  (f(std::integral_constant<int, Is>{}), ...);
}
template <int N, class F>
__host__ __device__ __forceinline__ void static_for(F&& f) {
  static_for_impl(std::make_integer_sequence<int, N>{}, static_cast<F&&>(f));
}

// --------------------------------------------------------------- multi-index ---------
// Coefficient order of the reference (multi_index.cpp:16-20): degree ascending, then
// lexicographic on (a,b,c); index_of closed form (multi_index.hpp:32-35).
__host__ __device__ constexpr int n_coef(int p) { return p * (p + 1) * (p + 2) / 6; }
__host__ __device__ constexpr int index_of(int a, int b, int c) {
  const int n = a + b + c;
  return n_coef(n) + a * (n + 1) - a * (a - 1) / 2 + b;
}

template <int P>  // order P: degrees 0..P-1
struct MI {
  static constexpr int N = n_coef(P);
  struct Tab {
    int e[N][3];
    int deg[N];
    double fact[N];  // alpha!
  };
  static constexpr Tab make() {
    Tab t{};
    int i = 0;
    for (int n = 0; n < P; ++n)
      for (int a = 0; a <= n; ++a)
        for (int b = 0; b <= n - a; ++b) {
          const int c = n - a - b;
          t.e[i][0] = a;
          t.e[i][1] = b;
          t.e[i][2] = c;
          t.deg[i] = n;
          double f = 1.0;
          for (int k = 2; k <= a; ++k) f *= k;
          for (int k = 2; k <= b; ++k) f *= k;
          for (int k = 2; k <= c; ++k) f *= k;
          t.fact[i] = f;
          ++i;
        }
    return t;
  }
  static constexpr Tab tab = make();
  static constexpr int ea(int i) { return tab.e[i][0]; }
  static constexpr int eb(int i) { return tab.e[i][1]; }
  static constexpr int ec(int i) { return tab.e[i][2]; }
  static constexpr int deg(int i) { return tab.deg[i]; }
  static constexpr double fact(int i) { return tab.fact[i]; }
};

// Host-side runtime multi-index table (for ops and host bookkeeping).
struct MIHost {
  int N = 0;
  int e[n_coef(FMM_MAX_ORDER + 1)][3];
  int deg[n_coef(FMM_MAX_ORDER + 1)];
  explicit MIHost(int max_degree) {
    int i = 0;
    for (int n = 0; n <= max_degree; ++n)
      for (int a = 0; a <= n; ++a)
        for (int b = 0; b <= n - a; ++b) {
          e[i][0] = a;
          e[i][1] = b;
          e[i][2] = n - a - b;
          deg[i] = n;
          ++i;
        }
    N = i;
  }
};

// Dispatch a runtime order 1..FMM_MAX_ORDER to a template functor F::template run<P>(args).
template <template <int> class F, class... Args>
inline void dispatch_order(int p, Args&&... args) {
  switch (p) {
    case 1: F<1>::run(std::forward<Args>(args)...); break;
    case 2: F<2>::run(std::forward<Args>(args)...); break;
    case 3: F<3>::run(std::forward<Args>(args)...); break;
    case 4: F<4>::run(std::forward<Args>(args)...); break;
    case 5: F<5>::run(std::forward<Args>(args)...); break;
    case 6: F<6>::run(std::forward<Args>(args)...); break;
    case 7: F<7>::run(std::forward<Args>(args)...); break;
    case 8: F<8>::run(std::forward<Args>(args)...); break;
    case 9: F<9>::run(std::forward<Args>(args)...); break;
    case 10: F<10>::run(std::forward<Args>(args)...); break;
    default: fail(FMM_ERR_UNSUPPORTED, "expansion order " + std::to_string(p) + " > FMM_MAX_ORDER");
  }
}

}  // namespace fmmb
