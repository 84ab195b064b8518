// Frobenius reductions of the core.py helpers (frobenius core.py:64-79, relative_error :157-166):
// deterministic two-level sums (fixed per-thread order, fixed block tree, fixed final order).
#include "../../include/apx.h"
#include "common.cuh"
#include "kernels.cuh"

namespace apx {

template <typename T>
__device__ __forceinline__ double2 ldz(const T* p, size_t i);
template <>
__device__ __forceinline__ double2 ldz<double>(const double* p, size_t i) { return make_double2(p[i], 0.0); }
template <>
__device__ __forceinline__ double2 ldz<double2>(const double2* p, size_t i) { return p[i]; }

// mode 0: out += (sum conj(a) b); mode 1: (sum |b - a|^2, sum |b|^2)
template <typename TA, typename TB>
__global__ void __launch_bounds__(256) pair_reduce_kernel(const TA* __restrict__ a, const TB* __restrict__ b,
                                                          size_t cnt, int mode, double* __restrict__ part) {
  __shared__ double red[32];
  double s0 = 0.0, s1 = 0.0;
  for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < cnt; e += (size_t)gridDim.x * blockDim.x) {
    const double2 x = ldz<TA>(a, e), y = ldz<TB>(b, e);
    if (mode == 0) {
      s0 = fma(x.x, y.x, fma(x.y, y.y, s0));   // Re conj(x) y
      s1 = fma(x.x, y.y, fma(-x.y, y.x, s1));  // Im conj(x) y
    } else {
      const double dx = y.x - x.x, dy = y.y - x.y;
      s0 = fma(dx, dx, fma(dy, dy, s0));
      s1 = fma(y.x, y.x, fma(y.y, y.y, s1));
    }
  }
  s0 = block_sum(s0, red);
  __syncthreads();
  s1 = block_sum(s1, red);
  if (threadIdx.x == 0) {
    part[2 * blockIdx.x] = s0;
    part[2 * blockIdx.x + 1] = s1;
  }
}

__global__ void pair_finalize_kernel(const double* __restrict__ part, int parts, double* __restrict__ out) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    double s0 = 0.0, s1 = 0.0;
    for (int p = 0; p < parts; ++p) {
      s0 += part[2 * p];
      s1 += part[2 * p + 1];
    }
    out[0] = s0;
    out[1] = s1;
  }
}

template <typename TA, typename TB>
static int pair_run(const void* a, const void* b, size_t cnt, int mode, double* part, double* out, cudaStream_t st) {
  const int blocks = kNumSMs * 4;
  pair_reduce_kernel<TA, TB><<<blocks, 256, 0, st>>>((const TA*)a, (const TB*)b, cnt, mode, part);
  APX_LAUNCH_CHECK();
  pair_finalize_kernel<<<1, 32, 0, st>>>(part, blocks, out);
  APX_LAUNCH_CHECK();
  return OK;
}

}  // namespace apx

using namespace apx;

extern "C" {

size_t apx_pair_reduce_workspace(void) { return (size_t)2 * kNumSMs * 4 * sizeof(double) + 256; }

// mode 0: out[0..1] = <A, B>_F = sum conj(A) B (re, im); mode 1: out = (||B - A||^2, ||B||^2).
// dtypes APX_F64 / APX_C128 per operand; count elements each.
int apx_pair_reduce(int dtype_a, const void* A, int dtype_b, const void* B, int64_t count, int mode, double* out,
                    void* wsp, size_t ws_bytes, void* stream) {
  APX_REQUIRE((dtype_a == F64 || dtype_a == C128) && (dtype_b == F64 || dtype_b == C128), "fp64/complex128 only");
  APX_REQUIRE(count >= 1 && (mode == 0 || mode == 1), "bad reduction arguments");
  Workspace ws(wsp, ws_bytes);
  double* part = ws.take<double>(2 * kNumSMs * 4);
  APX_WS_CHECK(ws);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (dtype_a == F64 && dtype_b == F64) return pair_run<double, double>(A, B, count, mode, part, out, st);
  if (dtype_a == F64) return pair_run<double, double2>(A, B, count, mode, part, out, st);
  if (dtype_b == F64) return pair_run<double2, double>(A, B, count, mode, part, out, st);
  return pair_run<double2, double2>(A, B, count, mode, part, out, st);
}

}  // extern "C"
