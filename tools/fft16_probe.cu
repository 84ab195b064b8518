// Validation and timing of fft4096_r16 (csrc/fft16.cuh) against a direct fp64 DFT and against
// fft_block (csrc/fft.cuh): batches of length-4096 transforms, two per 512-thread CTA.
#include <cstdio>
#include <cmath>
#include <vector>
#include <cuda_runtime.h>
#include "../paper_2504_19308_b200/csrc/common.cuh"
#include "../paper_2504_19308_b200/csrc/fft16.cuh"
using namespace apx;
namespace apx { void set_error(const char*, ...) {} void count_launch() {} void stage_mark(int, cudaStream_t) {} }

template <bool INV>
__global__ void __launch_bounds__(512) k16(const double2* in, double2* out, const double2* roots) {
  extern __shared__ __align__(16) double2 sm[];
  const int half = threadIdx.x >> 8, t = threadIdx.x & 255;
  const size_t base = ((size_t)blockIdx.x * 2 + half) * 4096;
  double2 v[16];
#pragma unroll
  for (int m = 0; m < 16; ++m) v[m] = in[base + t + 256 * m];
  fft4096_r16<INV>(v, sm + half * kFFT16Buf, roots, t, 1 + half);
#pragma unroll
  for (int m = 0; m < 16; ++m) out[base + t + 256 * m] = v[m];
}
__global__ void __launch_bounds__(512) kblk(const double2* in, double2* out, const double2* roots) {
  extern __shared__ __align__(16) double2 sm[];
  for (int h = 0; h < 2; ++h) {
    const size_t base = ((size_t)blockIdx.x * 2 + h) * 4096;
    for (int i = threadIdx.x; i < 4096; i += 512) sm[fsw(i, 4096)] = in[base + i];
    __syncthreads();
    fft_block(sm, nullptr, 4096, roots, false);
    for (int i = threadIdx.x; i < 4096; i += 512) out[base + i] = sm[fsw(i, 4096)];
    __syncthreads();
  }
}
int main() {
  const int n = 4096, batch = 4096;
  std::vector<double2> h((size_t)n * batch), r(n);
  for (size_t i = 0; i < h.size(); ++i) h[i] = make_double2(sin(0.37 * i) + 0.1 * (i % 7), cos(0.11 * i * i));
  for (int k = 0; k < n; ++k) r[k] = make_double2(cos(-2 * M_PI * k / n), sin(-2 * M_PI * k / n));
  double2 *din, *dout, *droots;
  cudaMalloc(&din, h.size() * 16); cudaMalloc(&dout, h.size() * 16); cudaMalloc(&droots, n * 16);
  cudaMemcpy(din, h.data(), h.size() * 16, cudaMemcpyHostToDevice);
  cudaMemcpy(droots, r.data(), n * 16, cudaMemcpyHostToDevice);
  const size_t sm16 = 2 * kFFT16Buf * 16;
  cudaFuncSetAttribute(k16<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm16);
  cudaFuncSetAttribute(k16<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm16);
  cudaFuncSetAttribute(kblk, cudaFuncAttributeMaxDynamicSharedMemorySize, 4096 * 16);
  k16<false><<<batch / 2, 512, sm16>>>(din, dout, droots);
  cudaDeviceSynchronize();
  std::vector<double2> o((size_t)n * batch);
  cudaMemcpy(o.data(), dout, o.size() * 16, cudaMemcpyDeviceToHost);
  double maxerr = 0, maxref = 0;
  for (int s : {0, 1, 2, 4095}) {
    for (int k = 0; k < n; k += 7) {
      long double re = 0, im = 0;
      for (int j = 0; j < n; ++j) {
        const long double a = -2.0L * M_PI * (((long long)j * k) % n) / n;
        const double2 x = h[(size_t)s * n + j];
        re += x.x * cosl(a) - x.y * sinl(a);
        im += x.x * sinl(a) + x.y * cosl(a);
      }
      const double2 g = o[(size_t)s * n + k];
      maxerr = fmax(maxerr, hypot(g.x - (double)re, g.y - (double)im));
      maxref = fmax(maxref, hypot((double)re, (double)im));
    }
  }
  // inverse round trip
  k16<true><<<batch / 2, 512, sm16>>>(dout, dout, droots);
  cudaDeviceSynchronize();
  cudaMemcpy(o.data(), dout, o.size() * 16, cudaMemcpyDeviceToHost);
  double rt = 0;
  for (size_t i = 0; i < o.size(); i += 13) rt = fmax(rt, hypot(o[i].x / n - h[i].x, o[i].y / n - h[i].y));
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  float t16, tb;
  cudaEventRecord(a); for (int i = 0; i < 10; ++i) k16<false><<<batch / 2, 512, sm16>>>(din, dout, droots); cudaEventRecord(b);
  cudaEventSynchronize(b); cudaEventElapsedTime(&t16, a, b);
  cudaEventRecord(a); for (int i = 0; i < 10; ++i) kblk<<<batch / 2, 512, 4096 * 16>>>(din, dout, droots); cudaEventRecord(b);
  cudaEventSynchronize(b); cudaEventElapsedTime(&tb, a, b);
  printf("{\"max_abs_err_vs_dft\": %.3e, \"max_abs_ref\": %.3e, \"roundtrip_err\": %.3e, \"r16_us\": %.1f, \"fft_block_us\": %.1f, \"err\": \"%s\"}\n",
         maxerr, maxref, rt, t16 * 100, tb * 100, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
