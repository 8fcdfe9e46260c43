// expansions.cuh — device helpers shared by the expansion kernels (expansions.cu, m2l.cu,
// ops.cu): the reference's derivative recurrence and multi-index helpers.
#pragma once

#include "context.cuh"


namespace fmmb {

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

}  // namespace fmmb
