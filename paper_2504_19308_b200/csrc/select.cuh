// Block-level top-k selection with the reference tie rule (circulant.py:63-70):
// the k largest weights, ties broken toward the LOWER index, emitted in ascending index order.
//
// One CTA of 1024 threads. Weights are non-negative doubles, so their IEEE bit patterns order
// like the values; an MSB-first 8-bit radix select finds the exact k-th largest key T, then a
// block scan over index order keeps every key > T plus the lowest-index keys == T.
#pragma once
#include "common.cuh"

namespace apx {

constexpr int kSelThreads = 1024;

// Exclusive block scan of one int per thread (1024 threads). Returns the exclusive prefix;
// *total receives the block total.
__device__ __forceinline__ int block_exclusive_scan_1024(int v, int* sh /*>=32*/, int* total) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  __syncthreads();
  if (lane == 31) sh[w] = x;
  __syncthreads();
  if (w == 0) {
    int s = sh[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int y = __shfl_up_sync(0xffffffffu, s, o);
      if (lane >= o) s += y;
    }
    sh[lane] = s;  // inclusive over warps
  }
  __syncthreads();
  int warp_excl = w == 0 ? 0 : sh[w - 1];
  *total = sh[31];
  return warp_excl + x - v;
}

// Order-preserving map of a double to an unsigned key (any sign); -0.0 is folded onto +0.0 so
// that zeros tie like numpy's comparison of -w does.
__device__ __forceinline__ unsigned long long dkey(double v) {
  if (v == 0.0) v = 0.0;
  const unsigned long long u = (unsigned long long)__double_as_longlong(v);
  return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}

// Selects into sel[0..k) (ascending). w: n doubles (global). Must be launched with 1024 threads.
__device__ inline void topk_select_block(const double* __restrict__ w, int n, int k, int* __restrict__ sel) {
  __shared__ unsigned int hist[256];
  __shared__ unsigned long long s_prefix, s_mask;
  __shared__ int s_krem;
  __shared__ int scan_sh[32];
  const int tid = threadIdx.x;
  if (k <= 0) return;
  if (tid == 0) { s_prefix = 0ull; s_mask = 0ull; s_krem = k; }
  __syncthreads();
  for (int pass = 0; pass < 8; ++pass) {
    const int shift = 56 - 8 * pass;
    for (int d = tid; d < 256; d += blockDim.x) hist[d] = 0u;
    __syncthreads();
    const unsigned long long prefix = s_prefix, mask = s_mask;
    for (int i = tid; i < n; i += blockDim.x) {
      unsigned long long key = dkey(w[i]);
      if ((key & mask) == prefix) atomicAdd(&hist[(key >> shift) & 255u], 1u);
    }
    __syncthreads();
    if (tid < 32) {
      // warp-parallel scan from the top digit down: lane l owns digits [248-8l .. 255-8l]
      int krem = s_krem;
      unsigned int local[8];
      unsigned int lsum = 0;
#pragma unroll
      for (int q = 0; q < 8; ++q) { local[q] = hist[255 - (tid * 8 + q)]; lsum += local[q]; }
      // inclusive prefix over lanes (lane 0 = highest digits)
      unsigned int incl = lsum;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        unsigned int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (tid >= o) incl += y;
      }
      unsigned int excl = incl - lsum;
      bool mine = (excl < (unsigned)krem) && (incl >= (unsigned)krem);
      if (mine) {
        unsigned int cum = excl;
        for (int q = 0; q < 8; ++q) {
          if (cum + local[q] >= (unsigned)krem) {
            int digit = 255 - (tid * 8 + q);
            s_krem = krem - (int)cum;
            s_prefix = prefix | ((unsigned long long)digit << shift);
            s_mask = mask | (255ull << shift);
            break;
          }
          cum += local[q];
        }
      }
    }
    __syncthreads();
  }
  const unsigned long long T = s_prefix;
  const int krem = s_krem;  // how many keys == T to take (lowest indices first)
  // contiguous chunk per thread, in index order
  const int chunk = (n + blockDim.x - 1) / blockDim.x;
  const int lo = min(n, tid * chunk), hi = min(n, lo + chunk);
  int eq = 0, gt = 0;
  for (int i = lo; i < hi; ++i) {
    unsigned long long key = dkey(w[i]);
    eq += key == T;
    gt += key > T;
  }
  int tot;
  int eq_before = block_exclusive_scan_1024(eq, scan_sh, &tot);
  int take_eq = max(0, min(eq, krem - eq_before));
  int pos = block_exclusive_scan_1024(gt + take_eq, scan_sh, &tot);
  int e = eq_before;
  for (int i = lo; i < hi; ++i) {
    unsigned long long key = dkey(w[i]);
    bool take = key > T;
    if (key == T) { take = e < krem; ++e; }
    if (take) sel[pos++] = i;
  }
}

}  // namespace apx
