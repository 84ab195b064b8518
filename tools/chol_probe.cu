// Per-step timing of the one-CTA elimination kernel (cholinv64) pattern, to find where the
// ~1300 cycles per pivot step go. Variants: 0 full step, 1 no trailing update, 2 no rsqrt,
// 3 barrier only.
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
template <int VAR>
__global__ void __launch_bounds__(256) probe(const double* Gin, int l, double* out, long long* tsteps) {
  __shared__ __align__(16) double rowbuf[2][64];
  // thread t: row t % 64, columns [16 (t / 64), +16): the lanes of a warp share their columns,
  // so the row-j reads are shared-memory broadcasts
  const int t = threadIdx.x, r = t & 63, c0 = (t >> 6) * 16;
  double w[16];
#pragma unroll
  for (int u = 0; u < 16; ++u) {
    const int c = c0 + u;
    w[u] = (c >= r) ? Gin[r * l + c] : 0.0;
  }
  __syncthreads();
  long long t0 = clock64();
#pragma unroll 1
  for (int j = 0; j < 64; ++j) {
    double* b = rowbuf[j & 1];
    if (r == j) {
#pragma unroll
      for (int u = 0; u < 16; u += 2) *reinterpret_cast<double2*>(&b[c0 + u]) = make_double2(w[u], w[u + 1]);
    }
    __syncthreads();
    if (VAR == 3) continue;
    double p = b[j];
    if (!(p > 0.0)) p = 1.0;
    const double rsq = VAR == 2 ? p : rsqrt(p);
    if (r > j && VAR != 1) {
      const double f = b[r] * (rsq * rsq);
      const unsigned lo = (unsigned)min(max(r - c0, 0), 16);
      const unsigned hi = (unsigned)min(max(j - c0 + 1, 0), 16);
      const unsigned act = (0xffffu << lo) | ((1u << hi) - 1u);
#pragma unroll
      for (int u = 0; u < 16; u += 2) {
        const double2 bv = VAR == 6 ? make_double2(1.0, 2.0) : *reinterpret_cast<const double2*>(&b[c0 + u]);
        const double b0 = (VAR != 4 && c0 + u == j) ? 1.0 : bv.x, b1 = (VAR != 4 && c0 + u + 1 == j) ? 1.0 : bv.y;
        // branch-free: inactive entries fold in a zero multiple (divergent per-entry branches
        // cost ~4x the whole step)
        const double f0 = (VAR == 5 || (act & (1u << u))) ? f : 0.0, f1 = (VAR == 5 || (act & (2u << u))) ? f : 0.0;
        w[u] = fma(-f0, b0, w[u]);
        w[u + 1] = fma(-f1, b1, w[u + 1]);
      }
    } else if (r == j) {
#pragma unroll
      for (int u = 0; u < 16; ++u) w[u] *= rsq;
    }
    if (t == 0) tsteps[j] = clock64() - t0;
  }
  double s = 0;
#pragma unroll
  for (int u = 0; u < 16; ++u) s += w[u];
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
    printf("\"var%d\": {\"us_per_launch\": %.2f, \"cyc_step1\": %lld, \"cyc_total\": %lld}, ", V, ms * 1000 / 20, hts[0], hts[63]); \
  }
  RUN(0) RUN(1) RUN(2) RUN(3) RUN(4) RUN(5) RUN(6)
  printf("\"done\": 1}\n");
  return 0;
}
