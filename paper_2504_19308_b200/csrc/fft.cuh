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
// acc + a * b as four fused multiply-adds (cadd(acc, cmul(a, b)) takes six double ops)
__device__ __forceinline__ double2 cmac(double2 acc, double2 a, double2 b) {
  return make_double2(fma(-a.y, b.y, fma(a.x, b.x, acc.x)), fma(a.y, b.x, fma(a.x, b.y, acc.y)));
}
// acc + a * conj(b) as four fused multiply-adds
__device__ __forceinline__ double2 cmacc(double2 acc, double2 a, double2 b) {
  return make_double2(fma(a.y, b.y, fma(a.x, b.x, acc.x)), fma(-a.x, b.y, fma(a.y, b.x, acc.y)));
}
__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 cconj(double2 a) { return make_double2(a.x, -a.y); }
__device__ __forceinline__ double2 cscale(double2 a, double s) { return make_double2(a.x * s, a.y * s); }

__host__ __device__ inline bool is_pow2(int n) { return n > 0 && (n & (n - 1)) == 0; }

// The eight twiddles of one radix-8 group (three radix-2 DIT stages s, s+1, s+2 at offset pos):
// stage s+2 uses u2 * e^{-+i pi m/4} (m = 0..3), stage s+1 uses u1 = u2^2 and u1 * (-+i), stage s
// uses w0 = u2^4, with u2 = roots[pos << (logn - s - 2)]. One table load per group instead of
// twelve (the table reads were most of the transform's L1 traffic); the squarings cost a few
// ulp, far inside the 1e-10 parity bar.
struct Radix8Tw {
  double2 w0, u1, u1r, u2[4];
};
__device__ __forceinline__ Radix8Tw radix8_twiddles(const double2* __restrict__ roots, int idx, bool inverse) {
  constexpr double r = 0.70710678118654752440;
  double2 u = __ldg(roots + idx);
  if (inverse) u.y = -u.y;
  Radix8Tw t;
  t.u1 = cmul(u, u);
  t.w0 = cmul(t.u1, t.u1);
  // times -i (forward) / +i (inverse)
  t.u1r = inverse ? make_double2(-t.u1.y, t.u1.x) : make_double2(t.u1.y, -t.u1.x);
  const double sg = inverse ? 1.0 : -1.0;
  t.u2[0] = u;
  t.u2[1] = cmul(u, make_double2(r, sg * r));
  t.u2[2] = inverse ? make_double2(-u.y, u.x) : make_double2(u.y, -u.x);
  t.u2[3] = cmul(u, make_double2(-r, sg * r));
  return t;
}

// radix-8 butterflies on v[0..8) (same order as three radix-2 DIT stages)
__device__ __forceinline__ void radix8_apply(double2 (&v)[8], const Radix8Tw& t) {
#pragma unroll
  for (int m = 0; m < 8; m += 2) {
    const double2 tt = cmul(t.w0, v[m + 1]);
    const double2 u = v[m];
    v[m] = cadd(u, tt);
    v[m + 1] = csub(u, tt);
  }
#pragma unroll
  for (int m = 0; m < 8; ++m) {
    if (m & 2) continue;
    const double2 tt = cmul((m & 1) ? t.u1r : t.u1, v[m + 2]);
    const double2 u = v[m];
    v[m] = cadd(u, tt);
    v[m + 2] = csub(u, tt);
  }
#pragma unroll
  for (int m = 0; m < 4; ++m) {
    const double2 tt = cmul(t.u2[m], v[m + 4]);
    const double2 u = v[m];
    v[m] = cadd(u, tt);
    v[m + 4] = csub(u, tt);
  }
}
__host__ __device__ inline int ilog2(int n) {
  int l = 0;
  while ((1 << l) < n) ++l;
  return l;
}

// Shared-memory slot of element i of a transform buffer of length n. Power-of-two buffers are
// XOR-swizzled inside each group of 8 complex values (slot = i ^ ((i >> 3) & 7)), which makes
// every radix-8 pass below -- stride-8 groups in the first pass, stride-1 in the later ones --
// hit all eight 16-byte bank groups evenly. Every access to a buffer passed to fft_block must go
// through fsw().
__device__ __forceinline__ int fsw(int i, int n) { return (n & (n - 1)) == 0 ? (i ^ ((i >> 3) & 7)) : i; }

// Visiting order of the bit-reversal swap: the e-th index swapped (a bijection of [0, 2^logn)).
// An 8-lane phase gets indices with distinct low three bits (distinct bank groups on the i side)
// and distinct top three bits (the partners j = brev(i) then differ in their low three bits),
// all other bits shared, so both sides of the swap are conflict-free under fsw(). In plain
// order the j side was an 8-way conflict: half of the transforms' excess shared wavefronts.
__device__ __forceinline__ int bitrev_order(int e, int logn) {
  if (logn < 6) return e;
  const int lam = e & 7, rho = (e >> 3) & 7, mid = e >> 6;
  return (((lam + rho) & 7) << (logn - 3)) | (mid << 3) | lam;
}

// roots[k] = exp(-2 pi i k / n) for k < n (full table; pow2 transforms use the first n/2)
void launch_roots(double2* roots, int n, cudaStream_t st);

// True when fft_block(..., linear_out = true) can leave its result in plain order x[i] instead of
// x[fsw(i)]: the last pass must be a radix-8 pass (log2 n a multiple of 3) with one group per
// thread, so that all its reads can finish (barrier) before the unswizzled writes.
__device__ __forceinline__ bool fft_linear_ok(int n) {
  return is_pow2(n) && n >= 8 && ilog2(n) % 3 == 0 && (n >> 3) <= (int)blockDim.x;
}

// In-place transform of x[0..n) in shared memory; `scratch` (n entries) is used by the direct
// DFT only. All threads of the CTA must call it (contains __syncthreads). With linear_out (and
// fft_linear_ok(n)) the output is in plain order: unaligned runs of consecutive elements -- the
// frequency-domain gathers -- then read conflict-free, where the swizzle split them over bank
// groups.
__device__ inline void fft_block(double2* x, double2* scratch, int n, const double2* __restrict__ roots,
                                 bool inverse, bool linear_out = false) {
  const int tid = threadIdx.x, nt = blockDim.x;
  if (n == 1) return;
  if (is_pow2(n)) {
    const int logn = ilog2(n);
    for (int e = tid; e < n; e += nt) {
      const int i = bitrev_order(e, logn);
      const int j = (int)(__brev((unsigned)i) >> (32 - logn));
      if (i < j) {
        APX_DCHECK(i < n && j < n);
        const double2 t = x[fsw(i, n)];
        x[fsw(i, n)] = x[fsw(j, n)];
        x[fsw(j, n)] = t;
      }
    }
    __syncthreads();
    // radix-8 passes: three consecutive radix-2 DIT stages s, s+1, s+2 on the 8 elements
    // base + pos + m*h (h = 2^(s-1)) held in registers -- one shared-memory round trip and one
    // barrier per three stages; the same twiddles and butterfly order as the radix-2 stages below
    int s = 1;
    const bool lin = linear_out && fft_linear_ok(n);
    for (; s + 2 <= logn; s += 3) {
      const int h = 1 << (s - 1);
      if (lin && s + 3 > logn) {  // last pass: all reads, barrier, plain-order writes
        const int g = tid;
        double2 v[8];
        const int pos = g & (h - 1);
        const int base = (g >> (s - 1)) << (s + 2);
        if (g < (n >> 3)) {
#pragma unroll
          for (int m = 0; m < 8; ++m) v[m] = x[fsw(base + pos + m * h, n)];
          radix8_apply(v, radix8_twiddles(roots, pos << (logn - s - 2), inverse));
        }
        __syncthreads();
        if (g < (n >> 3)) {
#pragma unroll
          for (int m = 0; m < 8; ++m) x[base + pos + m * h] = v[m];
        }
        __syncthreads();
        continue;
      }
      for (int g = tid; g < (n >> 3); g += nt) {
        const int pos = g & (h - 1);
        const int base = (g >> (s - 1)) << (s + 2);
        double2 v[8];
        APX_DCHECK(base + pos + 7 * h < n);
#pragma unroll
        for (int m = 0; m < 8; ++m) v[m] = x[fsw(base + pos + m * h, n)];
        radix8_apply(v, radix8_twiddles(roots, pos << (logn - s - 2), inverse));
#pragma unroll
        for (int m = 0; m < 8; ++m) x[fsw(base + pos + m * h, n)] = v[m];
      }
      __syncthreads();
    }
    for (; s <= logn; ++s) {
      const int half = 1 << (s - 1);
      for (int b = tid; b < (n >> 1); b += nt) {
        const int pos = b & (half - 1);
        const int i = ((b >> (s - 1)) << s) + pos;
        const int j = i + half;
        double2 w = __ldg(roots + (pos << (logn - s)));
        if (inverse) w.y = -w.y;
        const double2 t = cmul(w, x[fsw(j, n)]);
        const double2 u = x[fsw(i, n)];
        x[fsw(i, n)] = cadd(u, t);
        x[fsw(j, n)] = csub(u, t);
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
