// Per-step cycles of the split-block cholinv64 elimination (linalg.cu) and stripped variants:
// 0 full step, 1 no trailing update, 2 no rsqrt, 3 barrier + row publish only, 4 update without
// the shared-memory row reads, 5 full step with 128 threads (two rows per thread pair).
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
__device__ __forceinline__ double fast_rsqrt(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double h = 0.5 * x;
  double e = fma(-h * y, y, 0.5);
  y = fma(y, e, y);
  e = fma(-h * y, y, 0.5);
  return fma(y, e, y);
}
// VAR 5: var1 with the fast rsqrt; 6: var0 with the fast rsqrt; 7: var1 without any rsqrt;
// 8: var1 without the row scaling
template <int VAR>
__global__ void __launch_bounds__(256) probe(const double* Gin, int l, double* out, long long* tsteps) {
  __shared__ __align__(16) double rowL[2][64];
  __shared__ __align__(16) double rowR[2][64];
  const int t = threadIdx.x, r = t & 63, c0 = (t >> 6) * 16;
  double wl[16], wr[16];
#pragma unroll
  for (int u = 0; u < 16; ++u) {
    const int c = c0 + u;
    wl[u] = (c >= r) ? Gin[r * l + c] : 0.0;
    wr[u] = c == r ? 1.0 : 0.0;
  }
  __syncthreads();
  long long t0 = clock64();
#pragma unroll 1
  for (int j = 0; j < l; ++j) {
    double* bl = rowL[j & 1];
    double* br = rowR[j & 1];
    if (r == j) {
#pragma unroll
      for (int u = 0; u < 16; u += 2) {
        *reinterpret_cast<double2*>(&bl[c0 + u]) = make_double2(wl[u], wl[u + 1]);
        *reinterpret_cast<double2*>(&br[c0 + u]) = make_double2(wr[u], wr[u + 1]);
      }
    }
    __syncthreads();
    if (VAR == 3) { if (t == 0) tsteps[j] = clock64() - t0; continue; }
    double p = VAR == 10 ? 100.0 + j : bl[j];
    if (!(p > 0.0)) p = 1.0;
    const double rsq = (VAR == 2 || VAR == 7 || VAR == 9 || VAR == 10) ? p : (VAR == 5 || VAR == 6) ? fast_rsqrt(p) : rsqrt(p);
    if (VAR == 9) {
      const double sc = (r == j) ? rsq : 1.0;
#pragma unroll
      for (int u = 0; u < 16; ++u) { wl[u] *= sc; wr[u] *= sc; }
    } else if (r > j && VAR != 1 && VAR != 5 && VAR != 7 && VAR != 8 && VAR != 10) {
      const double f = bl[r] * (rsq * rsq);
      if (c0 + 15 > j) {
#pragma unroll
        for (int u = 0; u < 16; u += 2) {
          const double2 bv = VAR == 4 ? make_double2(1e-3, 2e-3) : *reinterpret_cast<const double2*>(&bl[c0 + u]);
          wl[u] = fma(-f, bv.x, wl[u]);
          wl[u + 1] = fma(-f, bv.y, wl[u + 1]);
        }
      }
      if (c0 <= j) {
#pragma unroll
        for (int u = 0; u < 16; u += 2) {
          const double2 bv = VAR == 4 ? make_double2(1e-3, 2e-3) : *reinterpret_cast<const double2*>(&br[c0 + u]);
          wr[u] = fma(-f, bv.x, wr[u]);
          wr[u + 1] = fma(-f, bv.y, wr[u + 1]);
        }
      }
    } else if (r == j && VAR != 8) {
#pragma unroll
      for (int u = 0; u < 16; ++u) { wl[u] *= rsq; wr[u] *= rsq; }
    }
    if (t == 0) tsteps[j] = clock64() - t0;
  }
  double s = 0;
#pragma unroll
  for (int u = 0; u < 16; ++u) s += wl[u] + wr[u];
  out[t] = s;
}
int main() {
  const int l = 64;
  double* h = (double*)malloc(l * l * 8);
  for (int i = 0; i < l; ++i)
    for (int j = 0; j < l; ++j) h[i * l + j] = (i == j ? 100.0 : 0.0) + 1.0 / (1 + i + j);
  double *G, *o;
  long long *ts, hts[64];
  cudaMalloc(&G, l * l * 8); cudaMalloc(&o, 256 * 8); cudaMalloc(&ts, 64 * 8);
  cudaMemcpy(G, h, l * l * 8, cudaMemcpyHostToDevice);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  printf("{");
#define RUN(V)                                                                              \
  {                                                                                         \
    probe<V><<<1, 256>>>(G, l, o, ts); cudaDeviceSynchronize();                             \
    cudaEventRecord(e0); for (int it = 0; it < 20; ++it) probe<V><<<1, 256>>>(G, l, o, ts); \
    cudaEventRecord(e1); cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1); \
    cudaMemcpy(hts, ts, 64 * 8, cudaMemcpyDeviceToHost);                                    \
    printf("\"var%d\": {\"us_per_launch\": %.2f, \"cyc_first8\": %lld, \"cyc_total\": %lld}, ", V, ms * 1000 / 20, hts[7], hts[63]); \
  }
  RUN(0) RUN(1) RUN(2) RUN(3) RUN(4) RUN(5) RUN(6) RUN(7) RUN(8) RUN(9) RUN(10)
  printf("\"done\": 1}\n");
  return 0;
}
