// Pipe-peak microbenchmarks for the roofline denominators that MEASURED_PEAKS.json lacks:
// FP32 FFMA, FP32x2 FFMA2, FP64 DFMA, FP64 DMMA (mma.sync m8n8k4), TF32 mma.sync m16n8k8.
// Timed with CUDA events; prints one JSON line.
#include <cstdio>
#include <cuda_runtime.h>
#include <cuda_fp16.h>

#define ITERS 4096
__global__ void k_ffma(float* out, float s) {
  float a[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) a[i] = threadIdx.x * 1e-3f + i;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) a[i] = fmaf(a[i], s, 0.5f);
  }
  float r = 0; for (int i = 0; i < 16; ++i) r += a[i];
  if (r == 1234.5f) out[0] = r;
}
__global__ void k_ffma2(float* out, float s) {
  unsigned long long a[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) { float2 v = make_float2(threadIdx.x * 1e-3f + i, i); a[i] = *reinterpret_cast<unsigned long long*>(&v); }
  float2 sv = make_float2(s, s); unsigned long long ss = *reinterpret_cast<unsigned long long*>(&sv);
  float2 hv = make_float2(0.5f, 0.5f); unsigned long long hh = *reinterpret_cast<unsigned long long*>(&hv);
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(a[i]) : "l"(ss), "l"(hh));
  }
  float r = 0; for (int i = 0; i < 16; ++i) { float2 v = *reinterpret_cast<float2*>(&a[i]); r += v.x + v.y; }
  if (r == 1234.5f) out[0] = r;
}
// mixed-precision FMA (sm_100: FHFMA): f16 x f16 products accumulated in fp32, the half operands
// taken from the .H0 / .H1 halves of packed registers (the f16 residual gather's inner op)
__global__ void k_fhfma(float* out, float s) {
  float a[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) a[i] = threadIdx.x * 1e-3f + i;
  const unsigned x = 0x3c003bffu ^ (unsigned)threadIdx.x;  // two halves
  unsigned short lo = (unsigned short)(x & 0xffff), hi = (unsigned short)(x >> 16);
  unsigned short l = __half_as_ushort(__float2half_rn(s));  // scalar half operand
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      if (i & 1) asm volatile("fma.rn.f32.f16 %0, %1, %2, %0;" : "+f"(a[i]) : "h"(hi), "h"(l));
      else asm volatile("fma.rn.f32.f16 %0, %1, %2, %0;" : "+f"(a[i]) : "h"(lo), "h"(l));
    }
  }
  float r = 0; for (int i = 0; i < 16; ++i) r += a[i];
  if (r == 1234.5f) out[0] = r;
}
__global__ void k_dfma(double* out, double s) {
  double a[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) a[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < ITERS / 4; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) a[i] = fma(a[i], s, 0.5);
  }
  double r = 0; for (int i = 0; i < 16; ++i) r += a[i];
  if (r == 1234.5) out[0] = r;
}
__global__ void k_dmma(double* out) {
  double acc[8][2];
  for (int i = 0; i < 8; ++i) { acc[i][0] = 0; acc[i][1] = 0; }
  double a = threadIdx.x * 1e-3, b = 1.0001;
  for (int it = 0; it < ITERS / 8; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(acc[i][0]), "+d"(acc[i][1]) : "d"(a), "d"(b));
  }
  double r = 0; for (int i = 0; i < 8; ++i) r += acc[i][0] + acc[i][1];
  if (r == 1234.5) out[0] = r;
}
__global__ void k_tf32(float* out) {
  float acc[8][4];
  for (int i = 0; i < 8; ++i) for (int j = 0; j < 4; ++j) acc[i][j] = 0;
  unsigned a0 = __float_as_uint(threadIdx.x * 1e-3f), b0 = __float_as_uint(1.0001f);
  for (int it = 0; it < ITERS / 4; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                   : "+f"(acc[i][0]), "+f"(acc[i][1]), "+f"(acc[i][2]), "+f"(acc[i][3])
                   : "r"(a0), "r"(a0), "r"(a0), "r"(a0), "r"(b0), "r"(b0));
  }
  float r = 0; for (int i = 0; i < 8; ++i) for (int j = 0; j < 4; ++j) r += acc[i][j];
  if (r == 1234.5f) out[0] = r;
}

// Shared-memory load bandwidth: every thread reads conflict-free V-wide words (LDS.32 / .64 /
// .128) from a 32 KB buffer, 16 independent loads per iteration, XOR-folded so nothing is dead.
template <typename V>
__device__ __forceinline__ unsigned fold(const V& v);
template <> __device__ __forceinline__ unsigned fold<unsigned>(const unsigned& v) { return v; }
template <> __device__ __forceinline__ unsigned fold<uint2>(const uint2& v) { return v.x ^ v.y; }
template <> __device__ __forceinline__ unsigned fold<uint4>(const uint4& v) { return v.x ^ v.y ^ v.z ^ v.w; }
template <typename V>
__global__ void k_lds(unsigned* out, int iters) {
  constexpr int W = sizeof(V) / 4;
  __shared__ __align__(16) unsigned buf[8192];
  for (int i = threadIdx.x; i < 8192; i += blockDim.x) buf[i] = i * 2654435761u;
  __syncthreads();
  const V* b = reinterpret_cast<const V*>(buf);
  const int nv = 8192 / W;
  unsigned acc = 0;
  int base = threadIdx.x;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 16; ++u) acc += fold<V>(b[(base + u * (nv / 16)) & (nv - 1)]);
    base += 7 * 32;  // warp-uniform stride keeps the 32 lanes on consecutive words
  }
  if (acc == 0x12345678u) out[0] = acc;
}

template <typename F>
float time_it(F f) {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  f(); cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(a); f(); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms;
  }
  return best;
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int blocks = sms * 8, threads = 256;
  float* f; double* d; cudaMalloc(&f, 64); cudaMalloc(&d, 64);
  double nthr = (double)blocks * threads;
  float t1 = time_it([&] { k_ffma<<<blocks, threads>>>(f, 0.999f); });
  double ffma = nthr * ITERS * 16 * 2 / (t1 * 1e-3) / 1e12;
  float t2 = time_it([&] { k_ffma2<<<blocks, threads>>>(f, 0.999f); });
  double ffma2 = nthr * ITERS * 16 * 4 / (t2 * 1e-3) / 1e12;
  float t2h = time_it([&] { k_fhfma<<<blocks, threads>>>(f, 0.999f); });
  double fhfma = nthr * ITERS * 16 * 2 / (t2h * 1e-3) / 1e12;
  float t3 = time_it([&] { k_dfma<<<blocks, threads>>>(d, 0.999); });
  double dfma = nthr * (ITERS / 4) * 16 * 2 / (t3 * 1e-3) / 1e12;
  float t4 = time_it([&] { k_dmma<<<blocks, threads>>>(d); });
  double dmma = (nthr / 32) * (ITERS / 8) * 8 * (8.0 * 8 * 4 * 2) / (t4 * 1e-3) / 1e12;
  float t5 = time_it([&] { k_tf32<<<blocks, threads>>>(f); });
  double tf32 = (nthr / 32) * (ITERS / 4) * 8 * (16.0 * 8 * 8 * 2) / (t5 * 1e-3) / 1e12;
  unsigned* u; cudaMalloc(&u, 64);
  const int li = 2048;
  int clk_khz = 0;
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  float t6 = time_it([&] { k_lds<unsigned><<<blocks, threads>>>(u, li); });
  float t7 = time_it([&] { k_lds<uint2><<<blocks, threads>>>(u, li); });
  float t8 = time_it([&] { k_lds<uint4><<<blocks, threads>>>(u, li); });
  auto lds_tbs = [&](float t, int bytes) { return nthr * li * 16.0 * bytes / (t * 1e-3) / 1e12; };
  const double l32 = lds_tbs(t6, 4), l64 = lds_tbs(t7, 8), l128 = lds_tbs(t8, 16);
  const double hz = clk_khz * 1e3;
  printf("{\"sms\": %d, \"fp32_ffma_tflops\": %.2f, \"fp32_ffma2_tflops\": %.2f, \"f16f32_fhfma_tflops\": %.2f, \"fp64_dfma_tflops\": %.2f, "
         "\"fp64_dmma_mma_sync_tflops\": %.2f, \"tf32_mma_sync_tflops\": %.2f, "
         "\"lds32_tbs\": %.2f, \"lds64_tbs\": %.2f, \"lds128_tbs\": %.2f, "
         "\"lds128_bytes_per_clk_per_sm_at_attr_clock\": %.1f, \"attr_clock_mhz\": %.0f, \"err\": \"%s\"}\n",
         sms, ffma, ffma2, fhfma, dfma, dmma, tf32, l32, l64, l128, l128 * 1e12 / hz / sms, hz / 1e6,
         cudaGetErrorString(cudaGetLastError()));
  return 0;
}
