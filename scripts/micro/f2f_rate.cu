// Microbenchmark: throughput of F2F.F64.F32 (float -> double), F2F.F32.F64, DFMA and an
// integer-only float->double widening, per SM per clock, on the local GPU.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void k_f2f(const float *in, double *out, int iters) {
  float a = in[threadIdx.x] , b = a * 1.5f, c = a * 0.5f, d = a * 0.25f;
  double s0 = 0, s1 = 0, s2 = 0, s3 = 0;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      s0 += (double)a; s1 += (double)b; s2 += (double)c; s3 += (double)d;
      a += 1.0f; b += 1.0f; c += 1.0f; d += 1.0f;
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s0 + s1 + s2 + s3;
}
__global__ void k_dfma(const float *in, double *out, int iters) {
  double a = in[threadIdx.x], b = a * 1.5, c = a * 0.5, d = a * 0.25, e = 1.0000001;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      a = fma(a, e, 1.0); b = fma(b, e, 1.0); c = fma(c, e, 1.0); d = fma(d, e, 1.0);
      a = fma(a, e, 1.0); b = fma(b, e, 1.0); c = fma(c, e, 1.0); d = fma(d, e, 1.0);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a + b + c + d;
}
__global__ void k_f2f_d2f(const float *in, double *out, int iters) {
  double a = in[threadIdx.x], b = a * 1.5, c = a * 0.5, d = a * 0.25;
  float s0 = 0, s1 = 0, s2 = 0, s3 = 0;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      s0 += (float)a; s1 += (float)b; s2 += (float)c; s3 += (float)d;
      a += 1.0; b += 1.0; c += 1.0; d += 1.0;
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s0 + s1 + s2 + s3;
}
int main() {
  float *in; double *out;
  cudaMalloc(&in, 1024 * 4); cudaMemset(in, 0, 4096);
  cudaMalloc(&out, 148 * 8 * 1024 * 8);
  int clk = 0; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const int iters = 2000, blocks = 148 * 8, thr = 256;
  auto run = [&](const char *name, void (*k)(const float *, double *, int), double ops_per_iter) {
    k<<<blocks, thr>>>(in, out, 10);
    cudaEventRecord(a);
    k<<<blocks, thr>>>(in, out, iters);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    const double ops = (double)blocks * thr * iters * ops_per_iter;
    printf("%-10s %.3f ms  %.2f Gop/s  %.1f op/clk/SM (at %d MHz)\n", name, ms, ops / ms / 1e6,
           ops / (ms * 1e-3) / 148 / (clk * 1e3), clk / 1000);
  };
  run("f2f64", k_f2f, 64);     // 64 conversions (+64 FADD +64 DADD) per iter
  run("dfma", k_dfma, 128);
  run("f2f32", k_f2f_d2f, 64);
  return 0;
}
