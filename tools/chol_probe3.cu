// Phase timing inside one pivot step of the per-row-mbarrier Cholesky-inverse (linalg.cu
// cholinv64f_kernel): the thread that will publish row j+1 (r = j+1, first column chunk) stamps
// clock64 at: row j visible (after the wait), pivot read, f computed, update done, row j+1
// published. Prints mean cycles per phase over the 64 steps.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ double fast_rcp(double x) {
  double y; asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  double e = fma(-x, y, 1.0); y = fma(y, e, y); e = fma(-x, y, 1.0); return fma(y, e, y);
}
__global__ void __launch_bounds__(256) k(const double* Gin, int l, double* out, long long* st) {
  extern __shared__ __align__(16) double rows[];
  __shared__ __align__(8) unsigned long long rbar[64];
  __shared__ long long ph_s[3];
  if (threadIdx.x < 3) ph_s[threadIdx.x] = 0;
  const int t = threadIdx.x, r = t & 63, c0 = (t >> 6) * 16;
  if (t < 64) asm volatile("mbarrier.init.shared::cta.b64 [%0], 4;" ::"r"((unsigned)__cvta_generic_to_shared(&rbar[t])));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  double wl[16], wr[16];
  for (int u = 0; u < 16; ++u) { const int c = c0 + u; wl[u] = c >= r ? Gin[r * l + c] : 0.0; wr[u] = c == r ? 1.0 : 0.0; }
  __syncthreads();
  
  long long tprev = clock64();
  for (int j = 0; j < l; ++j) {
    double* bl = rows + (size_t)j * 128; double* br = bl + 64;
    const unsigned bar = (unsigned)__cvta_generic_to_shared(&rbar[j]);
    const bool me = (r == j + 1) && c0 == 0;
    if (r == j) {
      for (int u = 0; u < 16; u += 2) {
        *reinterpret_cast<double2*>(&bl[c0 + u]) = make_double2(wl[u], wl[u + 1]);
        *reinterpret_cast<double2*>(&br[c0 + u]) = make_double2(wr[u], wr[u + 1]);
      }
      asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
    }
    asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%0], 0;\n@!p bra W_%=;\n}\n" ::"r"(bar) : "memory");
    long long t0 = clock64(); if (me) ph_s[0] += t0 - tprev;
    double p = bl[j];
    if (!(p > 1e-300)) p = 1.0;
    if (r > j) {
      const double f = bl[r] * fast_rcp(p);
      long long t1 = clock64(); if (me) ph_s[1] += t1 - t0;
      if (c0 + 15 > j) for (int u = 0; u < 16; u += 2) { const double2 bv = *reinterpret_cast<const double2*>(&bl[c0 + u]); wl[u] = fma(-f, bv.x, wl[u]); wl[u + 1] = fma(-f, bv.y, wl[u + 1]); }
      if (c0 <= j) for (int u = 0; u < 16; u += 2) { const double2 bv = *reinterpret_cast<const double2*>(&br[c0 + u]); wr[u] = fma(-f, bv.x, wr[u]); wr[u + 1] = fma(-f, bv.y, wr[u + 1]); }
      if (me) { double s = 0; for (int u = 0; u < 16; ++u) s += wl[u]; if (s == 12345.0) out[0] = s; }  // force completion
      long long t2 = clock64(); if (me) ph_s[2] += t2 - t1;
      tprev = t2;
    } else tprev = clock64();
  }
  __syncthreads();
  if (t == 0) for (int i = 0; i < 3; ++i) st[i] = ph_s[i] / (l - 1);
  double s = 0; for (int u = 0; u < 16; ++u) s += wl[u] + wr[u]; out[t] = s;
}
int main() {
  const int l = 64; double h[64 * 64];
  for (int i = 0; i < l; ++i) for (int j = 0; j < l; ++j) h[i * l + j] = (i == j ? 100.0 : 0.0) + 1.0 / (1 + i + j);
  double *G, *o; long long *s, hs[6];
  cudaMalloc(&G, sizeof(h)); cudaMalloc(&o, 256 * 8); cudaMalloc(&s, 48);
  cudaMemcpy(G, h, sizeof(h), cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 128 * 8);
  k<<<1, 256, 64 * 128 * 8>>>(G, l, o, s); cudaDeviceSynchronize();
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a); for (int i = 0; i < 20; ++i) k<<<1, 256, 64 * 128 * 8>>>(G, l, o, s); cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  cudaMemcpy(hs, s, 48, cudaMemcpyDeviceToHost);
  printf("{\"us_per_launch\": %.2f, \"cyc_wait_for_row\": %lld, \"cyc_pivot_to_f\": %lld, \"cyc_update\": %lld, \"err\": \"%s\"}\n",
         ms * 50, hs[0], hs[1], hs[2], cudaGetErrorString(cudaGetLastError()));
  return 0;
}
