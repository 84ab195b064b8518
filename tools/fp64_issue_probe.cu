// fp64 issue rate per warp: one CTA of W warps, each thread runs ITER x 32 independent DMULs
// (or DFMAs); cycles per warp-instruction from clock64. Prints JSON.
#include <cstdio>
#include <cuda_runtime.h>
template <int OP>
__global__ void k(double* out, long long* cyc, int iters, double s) {
  double a[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) a[i] = threadIdx.x + i;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 32; ++i) a[i] = OP == 0 ? a[i] * s : fma(a[i], s, 0.25);
  }
  long long t1 = clock64();
  double r = 0;
#pragma unroll
  for (int i = 0; i < 32; ++i) r += a[i];
  out[threadIdx.x] = r;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 1024 * 8); cudaMalloc(&c, 8);
  printf("{");
  for (int op = 0; op < 2; ++op)
    for (int w : {1, 2, 4, 8, 16, 32}) {
      long long h;
      if (op == 0) k<0><<<1, 32 * w>>>(o, c, 64, 0.999); else k<1><<<1, 32 * w>>>(o, c, 64, 0.999);
      cudaDeviceSynchronize();
      if (op == 0) k<0><<<1, 32 * w>>>(o, c, 64, 0.999); else k<1><<<1, 32 * w>>>(o, c, 64, 0.999);
      cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
      printf("\"%s_w%d_cyc_per_warp_instr\": %.2f, ", op ? "dfma" : "dmul", w, (double)h / (64.0 * 32));
    }
  printf("\"done\": 1}\n");
  return 0;
}
