// ops.cu — single-operator kernels behind fmm_op_* (operator-level parity tests mirroring
// proj/tests/test_kernels.cpp); thread per instance, the same formulas as the tree kernels.
#include "expansions.cuh"

namespace fmmb {
namespace {

// ------------------------------------------------------------ single-operator kernels ----
// Thread per instance; the same formulas as the tree kernels above (fmm_op_* entry points,
// used by the operator-level parity tests mirroring proj/tests/test_kernels.cpp).
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

}  // namespace fmmb
