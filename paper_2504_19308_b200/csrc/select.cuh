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
// n <= 8 * 1024: every thread keeps its contiguous chunk of keys in registers (one global read);
// larger n re-reads w per pass. The radix passes stop early once the bucket holding the k-th
// largest key is taken whole. Optional fused reductions (the callers' next launches):
//   kept  = kept_scale * sum_t kept_w[sel[t]]^2 over ascending t   (circulant.py:132 order)
//   total = sum_i tot_w[i]
__device__ inline void topk_select_block(const double* __restrict__ w, int n, int k, int* __restrict__ sel,
                                         const double* __restrict__ kept_w = nullptr, double kept_scale = 1.0,
                                         double* __restrict__ kept = nullptr, const double* __restrict__ tot_w = nullptr,
                                         double* __restrict__ total = nullptr) {
  constexpr int kReg = 8;
  __shared__ unsigned int hist[256];
  __shared__ unsigned long long s_prefix, s_mask;
  __shared__ int s_krem, s_done;
  __shared__ int scan_sh[32];
  __shared__ double s_red[32];
  const int tid = threadIdx.x;
  if (total && tot_w) {
    double t = 0.0;
    for (int i = tid; i < n; i += blockDim.x) t += tot_w[i];
    t = block_sum(t, s_red);
    if (tid == 0) *total = t;
  }
  if (k <= 0) {
    if (kept && tid == 0) *kept = 0.0;
    return;
  }
  const int chunk = (n + blockDim.x - 1) / blockDim.x;
  const int lo = min(n, tid * chunk), hi = min(n, lo + chunk);
  const bool in_regs = chunk <= kReg;
  unsigned long long kr[kReg];
#pragma unroll
  for (int q = 0; q < kReg; ++q) kr[q] = (in_regs && lo + q < hi) ? dkey(w[lo + q]) : 0ull;
  if (tid == 0) { s_prefix = 0ull; s_mask = 0ull; s_krem = k; s_done = 0; }
  __syncthreads();
  for (int pass = 0; pass < 8; ++pass) {
    const int shift = 56 - 8 * pass;
    for (int d = tid; d < 256; d += blockDim.x) hist[d] = 0u;
    __syncthreads();
    const unsigned long long prefix = s_prefix, mask = s_mask;
    if (in_regs) {
#pragma unroll
      for (int q = 0; q < kReg; ++q)
        if (lo + q < hi && (kr[q] & mask) == prefix) atomicAdd(&hist[(kr[q] >> shift) & 255u], 1u);
    } else {
      for (int i = tid; i < n; i += blockDim.x) {
        unsigned long long key = dkey(w[i]);
        if ((key & mask) == prefix) atomicAdd(&hist[(key >> shift) & 255u], 1u);
      }
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
            if (local[q] == (unsigned)(krem - (int)cum)) s_done = 1;  // the whole bucket is taken
            break;
          }
          cum += local[q];
        }
      }
    }
    __syncthreads();
    if (s_done) break;
  }
  const unsigned long long T = s_prefix, M = s_mask;
  const int krem = s_krem;  // how many keys with (key & M) == T to take (lowest indices first)
  int eq = 0, gt = 0;
  if (in_regs) {
#pragma unroll
    for (int q = 0; q < kReg; ++q)
      if (lo + q < hi) {
        eq += (kr[q] & M) == T;
        gt += (kr[q] & M) > T;
      }
  } else {
    for (int i = lo; i < hi; ++i) {
      unsigned long long key = dkey(w[i]) & M;
      eq += key == T;
      gt += key > T;
    }
  }
  int tot;
  int eq_before = block_exclusive_scan_1024(eq, scan_sh, &tot);
  int take_eq = max(0, min(eq, krem - eq_before));
  int pos = block_exclusive_scan_1024(gt + take_eq, scan_sh, &tot);
  int e = eq_before;
  if (in_regs) {
#pragma unroll
    for (int q = 0; q < kReg; ++q)
      if (lo + q < hi) {
        const unsigned long long key = kr[q] & M;
        bool take = key > T;
        if (key == T) { take = e < krem; ++e; }
        APX_DCHECK(!take || pos < k);
        if (take) sel[pos++] = lo + q;
      }
  } else {
    for (int i = lo; i < hi; ++i) {
      unsigned long long key = dkey(w[i]) & M;
      bool take = key > T;
      if (key == T) { take = e < krem; ++e; }
      APX_DCHECK(!take || pos < k);
      if (take) sel[pos++] = i;
    }
  }
  if (kept) {
    __syncthreads();  // sel[] complete (global writes by this CTA are visible after the barrier)
    double* sv = reinterpret_cast<double*>(hist);  // 256 x 4 B = room for 128 doubles per round
    double acc = 0.0;
    for (int t0 = 0; t0 < k; t0 += 128) {
      const int m = min(128, k - t0);
      if (tid < m) {
        const double v = kept_w[sel[t0 + tid]];
        sv[tid] = v * v;
      }
      __syncthreads();
      if (tid == 0)
        for (int t = 0; t < m; ++t) acc += sv[t];
      __syncthreads();
    }
    if (tid == 0) *kept = kept_scale * acc;
  }
}

}  // namespace apx
