// Shared-memory DFT building blocks (fp64 complex) for the circulant and Fourier-sparsified paths.
//
// fft_block(): one length-n transform held in shared memory by a whole CTA. Power-of-two n uses
// an in-place radix-2 Cooley-Tukey (bit reversal + log2 n butterfly stages) with an accurate
// twiddle table tw[k] = exp(-2 pi i k / n) (k < n/2) read through L1; other n (the reference's
// conformance sizes 3, 5, 31, 97, 700, ...) use a direct O(n^2) DFT against the full root table
// (k < n), which keeps fp64 accuracy for any length. Unnormalised; `inverse` uses conj twiddles.
#pragma once
#include "common.cuh"

namespace apx {

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ double2 cmulc(double2 a, double2 b) {  // a * conj(b)
  return make_double2(fma(a.x, b.x, a.y * b.y), fma(a.y, b.x, -a.x * b.y));
}
__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 cconj(double2 a) { return make_double2(a.x, -a.y); }
__device__ __forceinline__ double2 cscale(double2 a, double s) { return make_double2(a.x * s, a.y * s); }

__host__ __device__ inline bool is_pow2(int n) { return n > 0 && (n & (n - 1)) == 0; }
__host__ __device__ inline int ilog2(int n) {
  int l = 0;
  while ((1 << l) < n) ++l;
  return l;
}

// roots[k] = exp(-2 pi i k / n) for k < n (full table; pow2 transforms use the first n/2)
void launch_roots(double2* roots, int n, cudaStream_t st);

// In-place transform of x[0..n) in shared memory; `scratch` (n entries) is used by the direct
// DFT only. All threads of the CTA must call it (contains __syncthreads).
__device__ inline void fft_block(double2* x, double2* scratch, int n, const double2* __restrict__ roots,
                                 bool inverse) {
  const int tid = threadIdx.x, nt = blockDim.x;
  if (n == 1) return;
  if (is_pow2(n)) {
    const int logn = ilog2(n);
    for (int i = tid; i < n; i += nt) {
      const int j = (int)(__brev((unsigned)i) >> (32 - logn));
      if (i < j) {
        const double2 t = x[i];
        x[i] = x[j];
        x[j] = t;
      }
    }
    __syncthreads();
    for (int s = 1; s <= logn; ++s) {
      const int half = 1 << (s - 1);
      for (int b = tid; b < (n >> 1); b += nt) {
        const int pos = b & (half - 1);
        const int i = ((b >> (s - 1)) << s) + pos;
        const int j = i + half;
        double2 w = __ldg(roots + (pos << (logn - s)));
        if (inverse) w.y = -w.y;
        const double2 t = cmul(w, x[j]);
        const double2 u = x[i];
        x[i] = cadd(u, t);
        x[j] = csub(u, t);
      }
      __syncthreads();
    }
  } else {
    for (int i = tid; i < n; i += nt) scratch[i] = x[i];
    __syncthreads();
    for (int q = tid; q < n; q += nt) {
      double2 acc = make_double2(0.0, 0.0);
      int idx = 0;  // (p * q) mod n
      for (int p = 0; p < n; ++p) {
        double2 w = __ldg(roots + idx);
        if (inverse) w.y = -w.y;
        acc = cadd(acc, cmul(scratch[p], w));
        idx += q;
        if (idx >= n) idx -= n;
      }
      x[q] = acc;
    }
    __syncthreads();
  }
}

}  // namespace apx
