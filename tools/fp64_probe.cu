// Microbenchmark: fp64 DFMA latency (one dependent chain) and throughput (many warps, 8 chains).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void lat(double* out, double a, double b, int iters, long long* cyc) {
  double x = out[threadIdx.x];
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) x = fma(x, a, b);
  }
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}
__global__ void latf(float* out, float a, float b, int iters, long long* cyc) {
  float x = out[threadIdx.x];
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) x = fmaf(x, a, b);
  }
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}
__global__ void thr(double* out, double a, double b, int iters, long long* cyc) {
  double x0 = out[threadIdx.x], x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
      x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
    }
  }
  long long t1 = clock64();
  out[threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}
__global__ void rcp(double* out, int iters, long long* cyc) {
  double x = out[threadIdx.x] + 2.0;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) x = rsqrt(x) + 1.5;
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}
int main() {
  double* d; float* f; long long* c; long long h;
  cudaMalloc(&d, 1 << 20); cudaMalloc(&f, 1 << 20); cudaMalloc(&c, 8);
  cudaMemset(d, 0, 1 << 20); cudaMemset(f, 0, 1 << 20);
  const int it = 1000;
  lat<<<1, 32>>>(d, 0.999, 1e-3, it, c); cudaDeviceSynchronize();
  lat<<<1, 32>>>(d, 0.999, 1e-3, it, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("{\"dfma_latency_cyc\": %.2f, ", (double)h / (16.0 * it));
  latf<<<1, 32>>>(f, 0.999f, 1e-3f, it, c); cudaDeviceSynchronize();
  latf<<<1, 32>>>(f, 0.999f, 1e-3f, it, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("\"ffma_latency_cyc\": %.2f, ", (double)h / (16.0 * it));
  for (int warps : {1, 4, 8, 16, 32}) {
    thr<<<1, 32 * warps>>>(d, 0.999, 1e-3, it, c); cudaDeviceSynchronize();
    thr<<<1, 32 * warps>>>(d, 0.999, 1e-3, it, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("\"dfma_per_clk_sm_w%d\": %.2f, ", warps, 32.0 * warps * 32.0 * it / (double)h);
  }
  rcp<<<1, 32>>>(d, it, c); cudaDeviceSynchronize();
  rcp<<<1, 32>>>(d, it, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("\"rsqrt64_plus_add_latency_cyc\": %.2f}\n", (double)h / it);
  return 0;
}
