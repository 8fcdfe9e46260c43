// Pipe-throughput microbenchmark for the P2P / M2L design decisions on sm_100a:
// FFMA (scalar) vs FFMA2 (packed f32x2), MUFU.RSQ, DFMA. Prints lane-ops/clk/SM.
#include <cstdio>
#include <cuda_runtime.h>

#define ITERS 4096
#define CHAINS 8

__global__ void k_ffma(float* out, float a, float b) {
  float x[CHAINS];
  for (int i = 0; i < CHAINS; ++i) x[i] = threadIdx.x * 1e-3f + i;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < CHAINS; ++i) x[i] = fmaf(x[i], a, b);
  }
  float s = 0;
  for (int i = 0; i < CHAINS; ++i) s += x[i];
  if (s == 12345.f) out[0] = s;
}

__global__ void k_ffma_reg(float* out, const float* ab) {
  float a = ab[threadIdx.x & 1], b = ab[2 + (threadIdx.x & 1)];
  float x[CHAINS];
  float c[CHAINS];
  for (int i = 0; i < CHAINS; ++i) { x[i] = threadIdx.x * 1e-3f + i; c[i] = ab[4 + i]; }
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < CHAINS; ++i) x[i] = fmaf(x[i], c[i], b * a);
  }
  float s = 0;
  for (int i = 0; i < CHAINS; ++i) s += x[i];
  if (s == 12345.f) out[0] = s;
}

__global__ void k_ffma2(float* out, float a, float b) {
  float2 x[CHAINS];
  const float2 a2 = make_float2(a, a), b2 = make_float2(b, b);
  for (int i = 0; i < CHAINS; ++i) x[i] = make_float2(threadIdx.x * 1e-3f + i, i);
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < CHAINS; ++i) x[i] = __ffma2_rn(x[i], a2, b2);
  }
  float s = 0;
  for (int i = 0; i < CHAINS; ++i) s += x[i].x + x[i].y;
  if (s == 12345.f) out[0] = s;
}

__global__ void k_ffma2_reg(float* out, const float* ab) {
  float2 x[CHAINS], c[CHAINS];
  const float2 b2 = make_float2(ab[0], ab[1]);
  for (int i = 0; i < CHAINS; ++i) {
    x[i] = make_float2(threadIdx.x * 1e-3f + i, i);
    c[i] = make_float2(ab[4 + i], ab[5 + i]);
  }
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < CHAINS; ++i) x[i] = __ffma2_rn(x[i], c[i], b2);
  }
  float s = 0;
  for (int i = 0; i < CHAINS; ++i) s += x[i].x + x[i].y;
  if (s == 12345.f) out[0] = s;
}

__global__ void k_rsq(float* out, float a) {
  float x[CHAINS];
  for (int i = 0; i < CHAINS; ++i) x[i] = threadIdx.x * 1e-3f + i + 1.f;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < CHAINS; ++i) x[i] = rsqrtf(x[i]);
  }
  float s = 0;
  for (int i = 0; i < CHAINS; ++i) s += x[i];
  if (s == 12345.f) out[0] = s;
}

__global__ void k_dfma(double* out, double a, double b) {
  double x[CHAINS];
  for (int i = 0; i < CHAINS; ++i) x[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < ITERS / 4; ++it) {
#pragma unroll
    for (int i = 0; i < CHAINS; ++i) x[i] = fma(x[i], a, b);
  }
  double s = 0;
  for (int i = 0; i < CHAINS; ++i) s += x[i];
  if (s == 12345.) out[0] = s;
}

// mixed: FFMA2 chains interleaved with scalar FFMA chains (heavy + lite pipes?)
__global__ void k_mixed(float* out, const float* ab) {
  float2 x[CHAINS], c2[CHAINS];
  float y[CHAINS], c1[CHAINS];
  const float2 b2 = make_float2(ab[0], ab[1]);
  const float b1 = ab[2];
  for (int i = 0; i < CHAINS; ++i) {
    x[i] = make_float2(threadIdx.x * 1e-3f + i, i);
    c2[i] = make_float2(ab[4 + i], ab[5 + i]);
    y[i] = threadIdx.x * 2e-3f + i;
    c1[i] = ab[4 + i];
  }
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < CHAINS; ++i) {
      x[i] = __ffma2_rn(x[i], c2[i], b2);
      y[i] = __fmaf_rn(y[i], c1[i], b1);
    }
  }
  float s = 0;
  for (int i = 0; i < CHAINS; ++i) s += x[i].x + x[i].y + y[i];
  if (s == 12345.f) out[0] = s;
}

// operand-form variants of the packed ops used by the P2P pair (register-read pressure)
__global__ void k_fadd2_bc(float* out, const float* ab) {  // pair + broadcast scalar
  float2 x[CHAINS];
  float c[CHAINS];
  for (int i = 0; i < CHAINS; ++i) { x[i] = make_float2(threadIdx.x * 1e-3f + i, i); c[i] = ab[4 + i] * 1e-6f; }
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < CHAINS; ++i) x[i] = __fadd2_rn(x[i], make_float2(c[i], c[i]));
  }
  float s = 0;
  for (int i = 0; i < CHAINS; ++i) s += x[i].x + x[i].y;
  if (s == 12345.f) out[0] = s;
}

__global__ void k_fmul2_pp(float* out, const float* ab) {  // pair x pair
  float2 x[CHAINS], c[CHAINS];
  for (int i = 0; i < CHAINS; ++i) { x[i] = make_float2(threadIdx.x * 1e-3f + i, i); c[i] = make_float2(ab[4 + i], ab[5 + i]); }
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < CHAINS; ++i) x[i] = __fmul2_rn(x[i], c[i]);
  }
  float s = 0;
  for (int i = 0; i < CHAINS; ++i) s += x[i].x + x[i].y;
  if (s == 12345.f) out[0] = s;
}

__global__ void k_ffma2_3p(float* out, const float* ab) {  // three distinct pairs (acc update)
  float2 x[CHAINS], y[CHAINS], c[CHAINS];
  for (int i = 0; i < CHAINS; ++i) {
    x[i] = make_float2(threadIdx.x * 1e-3f + i, i);
    y[i] = make_float2(ab[6 + i] * 1e-3f, ab[7 + i] * 1e-3f);
    c[i] = make_float2(ab[4 + i], ab[5 + i]);
  }
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < CHAINS; ++i) x[i] = __ffma2_rn(y[i], c[i], x[i]);
  }
  float s = 0;
  for (int i = 0; i < CHAINS; ++i) s += x[i].x + x[i].y;
  if (s == 12345.f) out[0] = s;
}

template <class F>
float time_it(F f, int reps = 5) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  f();
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < reps; ++r) {
    cudaEventRecord(e0);
    f();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  return best;
}

int main() {
  cudaDeviceProp prop;
  cudaGetDeviceProperties(&prop, 0);
  int clk_khz = 0;
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  const int sms = prop.multiProcessorCount;
  printf("device %s sms=%d clock_attr=%d kHz\n", prop.name, sms, clk_khz);
  float* d;
  cudaMalloc(&d, 1024);
  float h[16];
  for (int i = 0; i < 16; ++i) h[i] = 0.999f + i * 1e-6f;
  cudaMemcpy(d, h, sizeof(h), cudaMemcpyHostToDevice);
  const int blocks = sms * 8, threads = 256;
  const double lanes = double(blocks) * threads;
  auto report = [&](const char* name, float ms, double ops_per_lane) {
    const double ops = lanes * ops_per_lane;
    printf("%-12s %8.3f ms  %8.2f Gop/s  => %.1f ops/clk/SM at 1.965GHz, %.1f at 1.35GHz\n", name,
           ms, ops / ms * 1e-6, ops / (ms * 1e-3) / sms / 1.965e9, ops / (ms * 1e-3) / sms / 1.35e9);
  };
  float ms;
  ms = time_it([&] { k_ffma<<<blocks, threads>>>(d, 0.999f, 1e-4f); });
  report("ffma_imm", ms, double(ITERS) * CHAINS);
  ms = time_it([&] { k_ffma_reg<<<blocks, threads>>>(d, d); });
  report("ffma_reg", ms, double(ITERS) * CHAINS);
  ms = time_it([&] { k_ffma2<<<blocks, threads>>>(d, 0.999f, 1e-4f); });
  report("ffma2", ms, double(ITERS) * CHAINS * 2);
  ms = time_it([&] { k_ffma2_reg<<<blocks, threads>>>(d, d); });
  report("ffma2_reg", ms, double(ITERS) * CHAINS * 2);
  ms = time_it([&] { k_fadd2_bc<<<blocks, threads>>>(d, d); });
  report("fadd2_bcast", ms, double(ITERS) * CHAINS * 2);
  ms = time_it([&] { k_fmul2_pp<<<blocks, threads>>>(d, d); });
  report("fmul2_pair", ms, double(ITERS) * CHAINS * 2);
  ms = time_it([&] { k_ffma2_3p<<<blocks, threads>>>(d, d); });
  report("ffma2_3pair", ms, double(ITERS) * CHAINS * 2);
  ms = time_it([&] { k_mixed<<<blocks, threads>>>(d, d); });
  report("ffma2+ffma", ms, double(ITERS) * CHAINS * 3);
  ms = time_it([&] { k_rsq<<<blocks, threads>>>(d, 1.f); });
  report("mufu_rsq", ms, double(ITERS) * CHAINS);
  ms = time_it([&] { k_dfma<<<blocks, threads>>>((double*)d, 0.999, 1e-4); });
  report("dfma", ms, double(ITERS / 4) * CHAINS);
  cudaError_t err = cudaGetLastError();
  printf("status: %s\n", cudaGetErrorString(err));
  return err == cudaSuccess ? 0 : 1;
}
