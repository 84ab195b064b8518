// Cycle-decomposition kernels: A = sum_j Lambda_j C^j (left layout, reference core.py:113,123-124,
// lambda_j[i] = A[i, (i-j) mod n]) and the gather passes of the cycle-truncated product.
//
//  K3  cycle_energy_partial / cycle_energy_finalize : ||lambda_j||^2 for all j in one HBM pass
//  K4  topk_select_kernel (select.cuh)              : top_indices semantics (circulant.py:63-70)
//      cycle_extract                                : lambda_t for the selected shifts (k x n)
//  K10 cycle_left_gather  : M[r,c] (+)= sum_t lamA_t[r] * X[(r - JA_t) mod n, c]   (Ahat . X)
//  K11 cycle_right_gather : M[r,c] (+)= sum_t X[r, m] * lamB'_t[c],  m = (c + JB_t) mod n,
//                           lamB'_t[c] = B[m, c] (column-aligned table, read coalesced)
//                           (X . Bhat), X optionally masked to dA (kept cycles of A zeroed)
#include "common.cuh"
#include "select.cuh"
#include "kernels.cuh"

namespace apx {

// ------------------------------------------------------------------------------------------
// K3: energies. Thread j walks the wrapped diagonal of cycle j over a chunk of rows; a warp
// reads 32 consecutive columns of one row per step (coalesced). fp32 inputs accumulate in fp32
// per chunk (<= 256 terms) and combine chunks in fp64; fp64 inputs accumulate in fp64.
// ------------------------------------------------------------------------------------------
// With `counters` (one per 256-column block, zero on entry, left zero on exit) the last CTA of
// each column block to finish also reduces that block's partials in fixed group order
// (energies, norms) -- the finalize pass without its own launch.
template <typename T>
__global__ void __launch_bounds__(256, 8) cycle_energy_partial(const T* __restrict__ A, int n, int rows_per_chunk,
                                                            double* __restrict__ partial,
                                                            unsigned* __restrict__ counters,
                                                            double* __restrict__ energies,
                                                            double* __restrict__ norms, int m_rows, int row_off) {
  using Acc = T;
  pdl_trigger();
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  const int g = blockIdx.y;
  const int r0 = g * rows_per_chunk;
  const int r1 = min(m_rows, r0 + rows_per_chunk);
  const bool valid = j < n;  // ragged last column block: idle threads still join the barriers
  if (valid) {
    Acc acc0 = 0, acc1 = 0, acc2 = 0, acc3 = 0;
    // local rows [0, m_rows) are global rows row_off + r (a row block of a sharded operand)
    int col = (r0 + row_off - j) % n;
    if (col < 0) col += n;
    const T* rowp = A + (size_t)r0 * n;
    int r = r0;
    // 8 rows per step: 8 independent loads in flight per thread (row r, column (r - j) mod n)
    for (; r + 8 <= r1; r += 8) {
      T v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        int cu = col + u;
        if (cu >= n) cu -= n;
        v[u] = __ldg(rowp + (size_t)u * n + cu);
      }
      acc0 += v[0] * v[0]; acc1 += v[1] * v[1]; acc2 += v[2] * v[2]; acc3 += v[3] * v[3];
      acc0 += v[4] * v[4]; acc1 += v[5] * v[5]; acc2 += v[6] * v[6]; acc3 += v[7] * v[7];
      col += 8;
      if (col >= n) col -= n;
      rowp += 8 * (size_t)n;
    }
    for (; r < r1; ++r) {
      T v = __ldg(rowp + col);
      acc0 += v * v;
      col = col + 1 == n ? 0 : col + 1;
      rowp += n;
    }
    partial[(size_t)g * n + j] = (double)((acc0 + acc1) + (acc2 + acc3));
  }
  if (counters == nullptr) return;
  __shared__ unsigned s_last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_last = atomicAdd(&counters[blockIdx.x], 1u) == gridDim.y - 1;
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  if (valid) {
    // fixed group order; 8 loads in flight at a time (the sum itself stays sequential)
    const int groups = (int)gridDim.y;
    double e = 0.0;
    for (int g0 = 0; g0 < groups; g0 += 8) {
      double v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = g0 + u < groups ? __ldcg(&partial[(size_t)(g0 + u) * n + j]) : 0.0;
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (g0 + u < groups) e += v[u];
    }
    energies[j] = e;
    norms[j] = sqrt(e);
  }
  if (threadIdx.x == 0) counters[blockIdx.x] = 0u;
}

// K3 (fp32, n % 4 == 0): the same energies from a row-major stream. A CTA (one per SM) walks its
// rows, each row staged whole into shared memory by one bulk async copy into a ring of kEnRing row
// buffers (three rows in flight behind the one being folded in: ~100 KB per SM), and accumulates
// each element's square into a per-cycle fp32 array in shared memory (cycle of (r, c) =
// (r - c) mod n). All threads fold one row at a time (a barrier per row), so no two threads touch a
// cycle at once and the sums are deterministic; the array is stored permuted, q -> (q mod 4) n/4 +
// q/4, so a warp's updates for one vector component hit consecutive words (conflict-free). Per CTA
// <= rows_per_chunk terms per cycle in fp32; the partials go out as fp64 for
// cycle_energy_finalize (fixed group order). (The diagonal walk of cycle_energy_partial reads one
// 4-byte element per thread and row: 3.9 TB/s at n = 8192; a register-prefetched row stream
// measured the same -- too few bytes in flight.)
constexpr int kEnRing = 4;
constexpr int kEnThreads = 512;
__global__ void __launch_bounds__(kEnThreads, 1) cycle_energy_rows4_kernel(const float* __restrict__ A, int n,
                                                                    int rows_per_chunk, double* __restrict__ partial) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int tid = threadIdx.x, nq = n >> 2;
  float4* ring = reinterpret_cast<float4*>(smem_raw);                  // kEnRing rows of nq float4
  float* s_en = reinterpret_cast<float*>(ring + (size_t)kEnRing * nq);  // n accumulators
  __shared__ __align__(8) uint64_t bars[kEnRing];
  for (int i = tid; i < n; i += kEnThreads) s_en[i] = 0.f;
  const int r0 = blockIdx.x * rows_per_chunk, r1 = min(n, r0 + rows_per_chunk);
  const uint32_t bytes = (uint32_t)nq * 16u;
  auto issue = [&](int r) {  // thread 0: row r into slot (r - r0) % kEnRing
    const int slot = (r - r0) % kEnRing;
    const uint32_t b = (uint32_t)__cvta_generic_to_shared(&bars[slot]);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(bytes) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(ring + (size_t)slot * nq)),
                 "l"(A + (size_t)r * n), "r"(bytes), "r"(b)
                 : "memory");
  };
  if (tid == 0) {
    for (int i = 0; i < kEnRing; ++i)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&bars[i])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int r = r0; r < min(r1, r0 + kEnRing); ++r) issue(r);
  }
  __syncthreads();
  for (int r = r0; r < r1; ++r) {
    const int it = r - r0, slot = it % kEnRing;
    const uint32_t b = (uint32_t)__cvta_generic_to_shared(&bars[slot]);
    asm volatile(
        "{\n.reg .pred p;\nEW_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra EW_%=;\n}\n" ::"r"(b),
        "r"((uint32_t)((it / kEnRing) & 1))
        : "memory");
    const float4* row = ring + (size_t)slot * nq;
    for (int c4 = tid; c4 < nq; c4 += kEnThreads) {
      const float4 v4 = row[c4];
      int q = r - 4 * c4;  // cycle of column 4 c4 (r, 4 c4 < n), minus x for component x
      if (q < 0) q += n;
      const float v[4] = {v4.x, v4.y, v4.z, v4.w};
#pragma unroll
      for (int x = 0; x < 4; ++x) {
        int qx = q - x;
        if (qx < 0) qx += n;
        float* e = s_en + (qx & 3) * nq + (qx >> 2);
        *e = fmaf(v[x], v[x], *e);
      }
    }
    __syncthreads();  // the slot's reads and this row's updates done
    if (tid == 0 && r + kEnRing < r1) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic reads before the async refill
      issue(r + kEnRing);
    }
  }
  for (int j = tid; j < n; j += kEnThreads) partial[(size_t)blockIdx.x * n + j] = (double)s_en[(j & 3) * nq + (j >> 2)];
}

static size_t rows4_smem(int n) { return (size_t)(kEnRing + 1) * n * sizeof(float); }
static int rows4_groups(int n, int* rpc, int ctas = 0) {
  static const int env = getenv("APX_EN_CTAS") ? atoi(getenv("APX_EN_CTAS")) : 0;  // tuning knob
  if (env > 0) ctas = env;
  const int want = ctas > 0 ? std::min(ctas, kNumSMs) : kNumSMs;  // one CTA per SM
  *rpc = (int)ceil_div(n, std::min(want, n));
  return (int)ceil_div(n, *rpc);
}
static bool rows4_ok(int n) {
  static const bool off = getenv("APX_EN_ROWS") != nullptr && atoi(getenv("APX_EN_ROWS")) == 0;
  return !off && n % 4 == 0 && n >= 1024 && rows4_smem(n) <= 200 * 1024;
}

// energies[j] = sum_g partial[g][j] (fixed order, 8 loads in flight); norms[j] = sqrt(energies[j]).
// energies[j] = sum_g partial[g][j]; norms[j] = sqrt(energies[j]). A CTA covers 32 columns with
// 8 slices of the groups (slice s: groups s, s+8, ...), combined in slice order -- a fixed order,
// and 8x the threads of a column-per-thread pass (which ran on only n/256 SMs, latency-bound).
__global__ void __launch_bounds__(256) cycle_energy_finalize(const double* __restrict__ partial, int n, int groups,
                                                             double* __restrict__ energies,
                                                             double* __restrict__ norms) {
  __shared__ double part[8][33];
  pdl_trigger();
  pdl_wait();
  const int jx = threadIdx.x & 31, sl = threadIdx.x >> 5;
  const int j = blockIdx.x * 32 + jx;
  double acc = 0.0;
  if (j < n)
    for (int g = sl; g < groups; g += 8) acc += partial[(size_t)g * n + j];
  part[sl][jx] = acc;
  __syncthreads();
  if (sl == 0 && j < n) {
    double e = 0.0;
#pragma unroll
    for (int q = 0; q < 8; ++q) e += part[q][jx];
    energies[j] = e;
    if (norms) norms[j] = sqrt(e);
  }
}

// Single-block deterministic sum of v[0..n) into *out (fixed order per thread, fixed tree).
__global__ void sum_vector_kernel(const double* __restrict__ v, int n, double* __restrict__ out) {
  __shared__ double sh[32];
  double s = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) s += v[i];
  s = block_sum(s, sh);
  if (threadIdx.x == 0) *out = s;
}

__global__ void __launch_bounds__(kSelThreads) topk_select_kernel(const double* __restrict__ w, int n, int k,
                                                                  int* __restrict__ sel, const double* kept_w,
                                                                  double kept_scale, double* kept,
                                                                  const double* tot_w, double* total) {
  pdl_trigger();
  pdl_wait();
  topk_select_block(w, n, k, sel, kept_w, kept_scale, kept, tot_w, total);
}

// kept = sum over selected t of norms[sel[t]]^2, ascending t (mirrors circulant.py:132 order).
__global__ void kept_energy_kernel(const double* __restrict__ norms, const int* __restrict__ sel, int k,
                                   double scale, double* __restrict__ out) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    double s = 0.0;
    for (int t = 0; t < k; ++t) {
      double m = norms[sel[t]];
      s += m * m;
    }
    *out = scale * s;
  }
}

// left layout (row-indexed):       lam[t][i] = A[i, (i - J_t) mod n]
// column-aligned layout (aligned): lam[t][c] = A[(c + J_t) mod n, c]  -- the coefficient that
// output column c of X . Ahat takes from shift t, so the right gather reads it coalesced.
// Each thread gathers kExtractT shifts of one index (all loads in flight before the stores).
constexpr int kExtractT = 8;
template <typename T, bool ALIGNED>
__global__ void cycle_extract(const T* __restrict__ A, int n, const int* __restrict__ J, int k,
                              T* __restrict__ lam, int m_rows, int row_off) {
  pdl_trigger();
  pdl_wait();
  // left layout over local rows i < m_rows (global row row_off + i), table row stride m_rows;
  // the aligned layout is always over all n columns (m_rows == n, row_off == 0)
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int t0 = blockIdx.y * kExtractT;
  if (i >= m_rows) return;
  T v[kExtractT];
#pragma unroll
  for (int u = 0; u < kExtractT; ++u) {
    const int t = t0 + u;
    if (t >= k) break;
    if (ALIGNED) {
      int r = i + __ldg(J + t);
      if (r >= n) r -= n;
      v[u] = A[(size_t)r * n + i];
    } else {
      int c = (i + row_off - __ldg(J + t)) % n;
      if (c < 0) c += n;
      v[u] = A[(size_t)i * n + c];
    }
  }
#pragma unroll
  for (int u = 0; u < kExtractT; ++u)
    if (t0 + u < k) lam[(size_t)(t0 + u) * m_rows + i] = v[u];
}

// Dense materialization of sum_t Lambda_t C^{J_t} (zero elsewhere).
template <typename T>
__global__ void cycle_materialize_kernel(const T* __restrict__ lam, const int* __restrict__ J, int k, int n,
                                         T* __restrict__ out) {
  const size_t total = (size_t)n * n;
  for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < total; e += (size_t)gridDim.x * blockDim.x)
    out[e] = T(0);
}
template <typename T>
__global__ void cycle_scatter_kernel(const T* __restrict__ lam, const int* __restrict__ J, int k, int n,
                                     T* __restrict__ out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int t = blockIdx.y;
  if (i >= n || t >= k) return;
  int c = i - J[t];
  if (c < 0) c += n;
  out[(size_t)i * n + c] = lam[(size_t)t * n + i];
}

// ------------------------------------------------------------------------------------------
// K10: left gather on a column strip. The CTA keeps X[:, c0:c0+W] in shared memory (row stride
// padded to avoid bank conflicts); thread = output row, W accumulators.
// ------------------------------------------------------------------------------------------
// 1024 threads: the strip's shared memory (up to (W + 1) n elements) leaves one CTA per SM at
// the largest strips, so the CTA itself must carry enough warps to hide the lambda loads
constexpr int kLeftThreads = 1024;
template <typename T, int W>
__global__ void __launch_bounds__(kLeftThreads) cycle_left_gather(const T* __restrict__ X, const T* __restrict__ lam,
                                                         const int* __restrict__ J, int k, int n, int accumulate,
                                                         T* __restrict__ M, int r_lo, int r_hi, int lam_ld) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* Xs = reinterpret_cast<T*>(smem_raw);
  constexpr int S = (W == 1) ? 1 : W + 1;  // padded row stride
  int* sJ = reinterpret_cast<int*>(Xs + (size_t)n * S);
  const int c0 = blockIdx.x * W;
  const int wcols = min(W, n - c0);
  // load strip (8 loads per thread in flight) and the shifts
  for (int e0 = threadIdx.x; e0 < n * W; e0 += 8 * blockDim.x) {
    T v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int e = e0 + u * blockDim.x, r = e / W, q = e - r * W;
      v[u] = (e < n * W && q < wcols) ? __ldg(X + (size_t)r * n + c0 + q) : T(0);
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int e = e0 + u * blockDim.x, r = e / W, q = e - r * W;
      if (e < n * W) Xs[r * S + q] = v[u];
    }
  }
  for (int t = threadIdx.x; t < k; t += blockDim.x) sJ[t] = J[t];
  __syncthreads();
  // output rows [r_lo, r_hi) (a sharded row block: lam holds those rows, stride lam_ld, and M
  // row r - r_lo); the whole matrix is r_lo = 0, r_hi = n, lam_ld = n
  const int rows_per_group = (r_hi - r_lo + gridDim.y - 1) / gridDim.y;
  const int rlo = r_lo + blockIdx.y * rows_per_group, rhi = min(r_hi, rlo + rows_per_group);
  for (int r = rlo + threadIdx.x; r < rhi; r += blockDim.x) {
    T acc[W];
#pragma unroll
    for (int q = 0; q < W; ++q) acc[q] = T(0);
    const T* lp = lam + (r - r_lo);
    // 8 shifts' lambda loads in flight before their FMAs
    for (int t0 = 0; t0 < k; t0 += 8) {
      T l[8];
      int src[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int t = t0 + u;
        l[u] = t < k ? __ldg(lp + (size_t)t * lam_ld) : T(0);
        int sr = r - (t < k ? sJ[t] : 0);
        src[u] = sr < 0 ? sr + n : sr;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const T* xs = Xs + src[u] * S;
#pragma unroll
        for (int q = 0; q < W; ++q) acc[q] = fma(l[u], xs[q], acc[q]);
      }
    }
    T* mp = M + (size_t)(r - r_lo) * n + c0;
    for (int q = 0; q < wcols; ++q) mp[q] = accumulate ? mp[q] + acc[q] : acc[q];
  }
}

// ------------------------------------------------------------------------------------------
// K11: right gather on a row block. The CTA keeps X[r0:r0+R, :] in shared memory, stored
// row-INTERLEAVED (Xs[m*RP + rr]) so that the R values one output column needs at source column
// m are contiguous: one address per (shift, column), then LDS.64 pairs feeding packed
// fma.rn.f32x2 (fp32) or scalar DFMA (fp64). X is optionally masked to dA (kept cycles of A
// zeroed on load). Thread = output column(s); each lambda value (an L2 load) feeds R FMAs.
// Also emits the block's partial sums of |M|^2 (report's ||M||_F) and |X|^2 (||A||_F).
// ------------------------------------------------------------------------------------------
__device__ __forceinline__ unsigned long long ffma2(unsigned long long a, unsigned long long b,
                                                    unsigned long long c) {
  unsigned long long d;
  asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ unsigned long long pack2(float x, float y) {
  return ((unsigned long long)__float_as_uint(y) << 32) | __float_as_uint(x);
}

// Non-coherent load as volatile asm: volatile statements keep their relative order, so all U*CPT
// lambda loads of a batch are issued before the first FMA consumes one (the scheduler otherwise
// sinks each load next to its use and exposes the L2 latency every time).
__device__ __forceinline__ float ldg_nc_ordered(const float* p) {
  float v;
  asm volatile("ld.global.nc.f32 %0, [%1];" : "=f"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ double ldg_nc_ordered(const double* p) {
  double v;
  asm volatile("ld.global.nc.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}

// Row-interleave pitch of the right gather's shared-memory block: even (8-byte aligned fp32 pairs)
// except for a single row, which the largest n (32768 fp32, 16384 fp64) can only afford unpadded.
// fp32: even (LDS.64 pairs, pitch 24 B for R = 6 spreads a warp over all banks); fp64: odd, so a
// warp's 32 consecutive m (8-byte loads at stride 8 * pitch) cover all 16 bank pairs (an even
// fp64 pitch of 8 put 16 lanes on each bank pair).
__host__ __device__ constexpr int gather_pitch(int r, size_t elem = 4) {
  return r == 1 ? 1 : (elem == 8 ? (r | 1) : r + (r & 1));
}

// shifts per lambda batch (U) and columns per thread (CPT) of the right gather (tuning knobs)
#ifndef APX_GATHER_U
#define APX_GATHER_U 4
#endif
#ifndef APX_GATHER_CPT
#define APX_GATHER_CPT 4
#endif
#ifndef APX_GATHER_THREADS
#define APX_GATHER_THREADS 512
#endif
constexpr int kGatherThreads = APX_GATHER_THREADS;

// TRUNC (fp32 only): operands truncated to TF32 (low 13 mantissa bits cleared) exactly as the
// tcgen05 kind::tf32 datapath reads them, so subtracting this gather from a TF32 GEMM over the
// same operands cancels the kept part exactly (up to fp32 summation order). TM = 2 (DELTA): lambda
// replaced by lambda - tf32(lambda), X as is -- for a TF32-exact X (the residual plan's Bm) this is
// the difference of the plain and the TRUNC gathers in one pass.
__device__ __forceinline__ float tf32_trunc(float x) { return __uint_as_float(__float_as_uint(x) & 0xffffe000u); }
__device__ __forceinline__ double tf32_trunc(double x) { return x; }

template <typename T, int R, bool FAST, int TM = 0>
__global__ void __launch_bounds__(kGatherThreads, 1) cycle_right_gather(const T* __restrict__ X, const int* __restrict__ JA, int ka,
                                                          const T* __restrict__ lam, const int* __restrict__ J, int k,
                                                          int n, int m_rows, int accumulate, T* __restrict__ M,
                                                          double* __restrict__ msq_partial,
                                                          double* __restrict__ xsq_partial, int* __restrict__ ticket,
                                                          int* __restrict__ ready, int x_early, int row_off,
                                                          const int* __restrict__ skip_if) {
  constexpr bool TRUNC = TM == 1, DELTA = TM == 2 && sizeof(T) == 4;
  if (skip_if != nullptr && *skip_if != 0) return;  // a gated-off launch (the C4 residual plan's fallback)
  constexpr int RP = gather_pitch(R, sizeof(T));
  // x_early: X (and the ticket / ready flags) predate the previous kernel of the stream, so under
  // a programmatic dependent launch the first row block is staged before waiting for that
  // kernel (the cycle selection / lambda extraction this gather consumes)
  if (!x_early) pdl_wait();  // interleave pitch (see gather_pitch)
  constexpr int CPT = APX_GATHER_CPT, U = APX_GATHER_U;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* Xs = reinterpret_cast<T*>(smem_raw);
  int* sJ = reinterpret_cast<int*>(Xs + (size_t)RP * n);
  __shared__ double red[32];
  __shared__ int s_blk, s_nxt;
  const int nblk = (int)ceil_div(m_rows, R);
  // ticket == nullptr: one row block per CTA (blockIdx.x). Otherwise a persistent grid smaller
  // than the SM count pulls row blocks from an atomic ticket, leaving the remaining SMs to a
  // concurrent stream (the mixed product's range finder).
  for (int it = 0;; ++it) {
    int blk;
    if (ticket) {
      // the next block is claimed (and its rows prefetched into L2) during the last column pass
      // of the current one; the first block, or a block that ended without claiming, takes a
      // ticket here
      if (threadIdx.x == 0) {
        s_blk = (it == 0 || s_nxt < 0) ? atomicAdd(ticket, 1) : s_nxt;
        s_nxt = -1;
      }
      __syncthreads();
      blk = s_blk;
    } else {
      if (it > 0) break;
      blk = blockIdx.x;
    }
    if (blk >= nblk) break;
    const int r0 = blk * R;
    const int rows = min(R, m_rows - r0);
    APX_DCHECK(rows > 0 && rows <= R);
    // coalesced row reads, interleaved shared-memory writes; rows past the end are zero.
    // The row block is read in batches of 16-byte vectors with all RP rows' loads issued before
    // any is stored, so a CTA pays ~one DRAM latency per batch instead of one per element.
    double xs = 0.0;
    constexpr int V = 16 / sizeof(T);
    using Vec = typename std::conditional<sizeof(T) == 4, float4, double2>::type;
    if (FAST && (n % V) == 0) {
      const int nv = n / V;
      for (int base = threadIdx.x; base < nv; base += blockDim.x * 2) {
        Vec buf[RP][2];
#pragma unroll
        for (int rr = 0; rr < RP; ++rr)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int iv = base + h * blockDim.x;
            if (rr < rows && iv < nv)
              buf[rr][h] = __ldg(reinterpret_cast<const Vec*>(X + (size_t)(r0 + rr) * n) + iv);
            else
              buf[rr][h] = Vec{};
          }
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int iv = base + h * blockDim.x;
          if (iv >= nv) continue;
          // the V columns of this vector times RP rows are one contiguous V*RP run of the
          // interleaved layout: transpose in registers, then RP 16-byte stores
          alignas(16) T tr[V * RP];
#pragma unroll
          for (int rr = 0; rr < RP; ++rr) {
            const T* e = reinterpret_cast<const T*>(&buf[rr][h]);
            T s = T(0);
#pragma unroll
            for (int q = 0; q < V; ++q) {
              s = fma(e[q], e[q], s);
              tr[q * RP + rr] = TRUNC ? tf32_trunc(e[q]) : e[q];
            }
            xs += (double)s;
          }
          Vec* dst = reinterpret_cast<Vec*>(Xs + (size_t)iv * V * RP);
#pragma unroll
          for (int w = 0; w < RP; ++w) dst[w] = reinterpret_cast<const Vec*>(tr)[w];
        }
      }
    } else {
      for (int rr = 0; rr < RP; ++rr) {
        const T* src = X + (size_t)(r0 + rr) * n;
        for (int m = threadIdx.x; m < n; m += blockDim.x) {
          T v = T(0);
          if (rr < rows) v = __ldg(src + m);
          xs = fma((double)v, (double)v, xs);
          Xs[(size_t)m * RP + rr] = TRUNC ? tf32_trunc(v) : v;
        }
      }
    }
    if (x_early && it == 0) pdl_wait();
    // shifts, padded with zeros to a multiple of U (FAST: the lambda rows are zero-padded too)
    const int kp = FAST ? (int)ceil_div(k, U) * U : k;
    for (int t = threadIdx.x; t < kp; t += blockDim.x) sJ[t] = t < k ? J[t] : 0;
    __syncthreads();
    if (xsq_partial != nullptr) {  // ||X||^2 of the (unmasked) rows
      xs = block_sum(xs, red);
      if (threadIdx.x == 0) xsq_partial[blk] = xs;
    }
    if (JA != nullptr) {
      for (int e = threadIdx.x; e < rows * ka; e += blockDim.x) {
        const int rr = e / ka, t = e - rr * ka;
        int m = (r0 + rr + row_off - JA[t]) % n;  // global row of local row r0 + rr
        if (m < 0) m += n;
        Xs[(size_t)m * RP + rr] = T(0);
      }
      __syncthreads();
    }
    double msq = 0.0;
    // Each thread owns CPT columns (blockDim apart, so warps stay coalesced). U shifts' worth of
    // lambda loads are issued before any is consumed (U*CPT L2 loads in flight per thread).
    constexpr int NP = (sizeof(T) == 4) ? R / 2 : 0;    // packed float pairs
    constexpr int NS = (sizeof(T) == 4) ? (R & 1) : R;  // scalar rows
    const int stride = FAST ? kGatherThreads : (int)blockDim.x;  // FAST launches exactly kGatherThreads
    // column chunk of this CTA (grid.y > 1 only in FAST mode: chunk widths are multiples of stride*CPT)
    const int cw = (int)ceil_div(ceil_div(n, stride * CPT), gridDim.y) * stride * CPT;
    const int c_lo = blockIdx.y * cw, c_hi = min(n, c_lo + cw);
    for (int cb = c_lo + threadIdx.x; cb < c_hi; cb += stride * CPT) {
      if (FAST && ticket && threadIdx.x == 0 && cb + stride * CPT >= c_hi) {
        const int nx = atomicAdd(ticket, 1);
        s_nxt = nx;
        if (nx < nblk && ((uintptr_t)X & 15) == 0) {  // bulk prefetch: 16-byte granules
          const int nrows = min(R, m_rows - nx * R);
          for (int rr = 0; rr < nrows; ++rr)
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(X + (size_t)(nx * R + rr) * n),
                         "r"((unsigned)(n * sizeof(T)))
                         : "memory");
        }
      }
      unsigned long long acc2[CPT][NP > 0 ? NP : 1];
      T accs[CPT][NS > 0 ? NS : 1];
#pragma unroll
      for (int q = 0; q < CPT; ++q) {
#pragma unroll
        for (int p = 0; p < (NP > 0 ? NP : 1); ++p) acc2[q][p] = 0ull;
#pragma unroll
        for (int s = 0; s < (NS > 0 ? NS : 1); ++s) accs[q][s] = T(0);
      }
      // software pipeline across shift batches: batch i+1's lambda loads are in flight while
      // batch i is consumed (ping-pong register buffers A/B)
      auto load_batch = [&](int t0, int (&mm)[U][CPT], T (&lv)[U][CPT]) {
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int t = t0 + u;
          const int jt = sJ[t];  // broadcast
          const T* lrow = lam + (size_t)t * n;
#pragma unroll
          for (int q = 0; q < CPT; ++q) {
            const int c = cb + q * stride;
            if constexpr (FAST) {
              // (c + jt) mod n as an unsigned min: c + jt - n wraps above c + jt unless c + jt >= n
              unsigned m = (unsigned)(c + jt);
              m = min(m, m - (unsigned)n);
              APX_DCHECK(m < (unsigned)n && jt >= 0 && jt < n);
              mm[u][q] = (int)m;
              lv[u][q] = ldg_nc_ordered(lrow + c);
              if constexpr (TRUNC) lv[u][q] = tf32_trunc(lv[u][q]);
              if constexpr (DELTA) lv[u][q] = lv[u][q] - tf32_trunc(lv[u][q]);
            } else {
              int m = c + jt;
              m = m >= n ? m - n : m;
              const bool ok = t < k && c < n;
              mm[u][q] = ok ? m * RP : 0;
              lv[u][q] = ok ? __ldg(lrow + c) : T(0);
              if constexpr (TRUNC) lv[u][q] = tf32_trunc(lv[u][q]);
              if constexpr (DELTA) lv[u][q] = lv[u][q] - tf32_trunc(lv[u][q]);
            }
          }
        }
      };
      auto compute_batch = [&](const int (&mm)[U][CPT], const T (&lv)[U][CPT]) {
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
          for (int q = 0; q < CPT; ++q) {
            const T* xp = Xs + (FAST ? (unsigned)mm[u][q] * RP : mm[u][q]);
            if constexpr (NP > 0) {
              const unsigned long long l2 = pack2((float)lv[u][q], (float)lv[u][q]);
              const unsigned long long* xp2 = reinterpret_cast<const unsigned long long*>(xp);
#pragma unroll
              for (int p = 0; p < NP; ++p) acc2[q][p] = ffma2(xp2[p], l2, acc2[q][p]);
            }
            if constexpr (NS > 0) {
#pragma unroll
              for (int s2 = 0; s2 < NS; ++s2) accs[q][s2] = fma(xp[2 * NP + s2], lv[u][q], accs[q][s2]);
            }
          }
      };
      // the epilogue reads back M (written by the preceding low-rank GEMM, usually DRAM-resident):
      // pull those lines toward L2 now so the read-modify-write does not stall on DRAM latency
      if (accumulate) {
#pragma unroll
        for (int q = 0; q < CPT; ++q) {
          const int c = cb + q * stride;
#pragma unroll
          for (int rr = 0; rr < R; ++rr)
            if ((FAST || c < n) && rr < rows)
              asm volatile("prefetch.global.L2 [%0];" ::"l"(M + (size_t)(r0 + rr) * n + c));
        }
      }
      int mmA[U][CPT], mmB[U][CPT];
      T lvA[U][CPT], lvB[U][CPT];
      load_batch(0, mmA, lvA);
      for (int t0 = 0; t0 < kp; t0 += 2 * U) {
        if (t0 + U < kp) load_batch(t0 + U, mmB, lvB);
        compute_batch(mmA, lvA);
        if (t0 + U >= kp) break;
        if (t0 + 2 * U < kp) load_batch(t0 + 2 * U, mmA, lvA);
        compute_batch(mmB, lvB);
      }
      // read-modify-write of M: all CPT*R old values are loaded before the first store, so the
      // thread waits one L2 latency per column block rather than one per element (the compiler
      // cannot hoist a load of M above a store to M on its own)
      T mold[CPT][R];
#pragma unroll
      for (int q = 0; q < CPT; ++q) {
        const int c = cb + q * stride;
#pragma unroll
        for (int rr = 0; rr < R; ++rr)
          mold[q][rr] = (accumulate && (FAST || c < n) && rr < rows) ? M[(size_t)(r0 + rr) * n + c] : T(0);
      }
#pragma unroll
      for (int q = 0; q < CPT; ++q) {
        const int c = cb + q * stride;
        if (!FAST && c >= n) continue;
#pragma unroll
        for (int rr = 0; rr < R; ++rr) {
          T a;
          if constexpr (NP > 0) {
            if (rr < 2 * NP) {
              const unsigned long long v = acc2[q][rr >> 1];
              a = (T)__uint_as_float((unsigned)(rr & 1 ? (v >> 32) : (v & 0xffffffffull)));
            } else {
              a = accs[q][rr - 2 * NP];
            }
          } else {
            a = accs[q][rr];
          }
          if (rr < rows) {
            T* mp = M + (size_t)(r0 + rr) * n + c;
            T v = accumulate < 0 ? mold[q][rr] - a : mold[q][rr] + a;
            *mp = v;
            msq += (double)v * (double)v;
          }
        }
      }
    }
    double s = block_sum(msq, red);  // (its barriers also order every thread's M stores before the flag)
    if (threadIdx.x == 0 && msq_partial) msq_partial[blk] = s;
    if (threadIdx.x == 0 && ready) {
      // publish the finished row block to a concurrent consumer (the mixed product's M += Q.W)
      __threadfence();
      atomicExch(ready + blk, 1);
    }
    __syncthreads();  // Xs / sJ / red are refilled by the next row block
  }
}

// ------------------------------------------------------------------------------------------
// K11s: segmented right gather for large n, where a whole row no longer fits shared memory R>2
// times (fp32 n = 32768: one 128 KB row per CTA, so each lambda' value -- an L2 load -- fed a
// single FMA and the kernel was L2-bound). The CTA keeps R rows but only a column SEGMENT of
// them, [s0, s0 + sw), in shared memory, and sweeps the segments: for output column c only the
// shifts whose source column m = (c + J_t) mod n falls in the segment contribute. With J sorted
// once per CTA, those shifts are one cyclic run of the sorted list, found by binary search per
// (warp, segment) -- so every (c, t) pair is visited exactly once over the sweep, each lambda'
// load again feeds R FMAs, and M is read-modified-written once per segment (from L2).
// ------------------------------------------------------------------------------------------
constexpr int kSegThreads = 512;
constexpr int kSegU = 4;    // shifts per batch (kSegU * kSegCPT lambda loads in flight per thread)
// columns per thread (lane + 32 q of the warp's column chunk): 4 fp32, 2 fp64 (register budget)
template <typename T>
__host__ __device__ constexpr int seg_cpt() { return sizeof(T) == 4 ? 4 : 2; }

// L2 eviction policies: lambda' (re-read for every row block) is kept, the streamed operand rows
// and the M read-modify-write traffic go first
__device__ __forceinline__ unsigned long long l2_policy_evict_last() {
  unsigned long long p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ unsigned long long l2_policy_evict_first() {
  unsigned long long p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ float ldg_nc_hint(const float* a, unsigned long long pol) {
  float v;
  asm volatile("ld.global.nc.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(v) : "l"(a), "l"(pol));
  return v;
}
__device__ __forceinline__ double ldg_nc_hint(const double* a, unsigned long long pol) {
  double v;
  asm volatile("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(a), "l"(pol));
  return v;
}
__device__ __forceinline__ float ldg_hint(const float* a, unsigned long long pol) {
  float v;
  asm volatile("ld.global.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(v) : "l"(a), "l"(pol));
  return v;
}
__device__ __forceinline__ double ldg_hint(const double* a, unsigned long long pol) {
  double v;
  asm volatile("ld.global.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(a), "l"(pol));
  return v;
}
__device__ __forceinline__ void stg_hint(float* a, float v, unsigned long long pol) {
  asm volatile("st.global.L2::cache_hint.f32 [%0], %1, %2;" ::"l"(a), "f"(v), "l"(pol) : "memory");
}
__device__ __forceinline__ void stg_hint(double* a, double v, unsigned long long pol) {
  asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(a), "d"(v), "l"(pol) : "memory");
}

// first index i >= from with tab[i].x >= v (tab ascending in .x)
__device__ __forceinline__ int lower_index(const int2* tab, int k, int v, int from) {
  int a = from, b = k;
  while (a < b) {
    const int h = (a + b) >> 1;
    if (tab[h].x < v) a = h + 1; else b = h;
  }
  return a;
}

// residual-energy rule of the f16 plans (mixed_f16.cu kResidF16MaxEnergy): the masked operand
// X - Xhat carries at most 1% of ||X||^2, so f16 rounding of it (2^-11 relative) stays below
// ~4e-5 of the product
__device__ __forceinline__ bool resid_small(const double* fro2, const double* kept) {
  const double f = *fro2, kp = *kept;
  return f > 0.0 && f < 1e300 && (f - kp) <= 0.01 * f;
}

// lower_index for a converged warp and a short table: every lane counts its entries below v
// (independent loads) and one warp reduction adds them -- ~60 cycles instead of log2(k)
// dependent shared-memory round trips (16% of the f16 segmented gather's stall samples)
__device__ __forceinline__ int count_below(const int2* tab, int k, int v) {
  int c = 0;
  for (int i = threadIdx.x & 31; i < k; i += 32) c += tab[i].x < v ? 1 : 0;
  return __reduce_add_sync(0xffffffffu, c);
}
__device__ __forceinline__ void red_add(float* a, float v) {
  asm volatile("red.relaxed.gpu.global.add.f32 [%0], %1;" ::"l"(a), "f"(v) : "memory");
}
__device__ __forceinline__ void red_add(double* a, double v) {
  asm volatile("red.relaxed.gpu.global.add.f64 [%0], %1;" ::"l"(a), "d"(v) : "memory");
}
__device__ __forceinline__ float ld_relaxed_f32(const float* a) {
  float v;
  asm volatile("ld.relaxed.gpu.global.f32 %0, [%1];" : "=f"(v) : "l"(a) : "memory");
  return v;
}
__device__ __forceinline__ float ld_relaxed(const float* a) { return ld_relaxed_f32(a); }
__device__ __forceinline__ double ld_relaxed(const double* a) {
  double v;
  asm volatile("ld.relaxed.gpu.global.f64 %0, [%1];" : "=d"(v) : "l"(a) : "memory");
  return v;
}

template <typename T, int R, int TUNE>
__global__ void __launch_bounds__(kSegThreads, 1)
    cycle_right_gather_seg(const T* __restrict__ X, const int* __restrict__ JA, int ka, const T* __restrict__ lam,
                           const int* __restrict__ J, int k, int n, int m_rows, int accumulate, T* __restrict__ M,
                           double* __restrict__ msq_partial, double* __restrict__ xsq_partial, int SW, int row_off,
                           int c_lo, int c_hi, int lam_ld, int out_ld, const double* __restrict__ g_fro2,
                           const double* __restrict__ g_kept) {
  // the f16-staged variant (cycle_right_gather_seg_h) takes the product when the masked operand is
  // a small residual; this kernel is then its no-op twin (same device-side decision, no host sync)
  if (g_fro2 != nullptr && resid_small(g_fro2, g_kept)) return;
  constexpr int RP = gather_pitch(R, sizeof(T));
  constexpr int CPT = seg_cpt<T>();
  constexpr int NP = (sizeof(T) == 4) ? R / 2 : 0;
  constexpr int NS = (sizeof(T) == 4) ? (R & 1) : R;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* Xs = reinterpret_cast<T*>(smem_raw);
  int2* sJT = reinterpret_cast<int2*>(Xs + (size_t)RP * SW);  // (shift, lambda row), ascending shift
  __shared__ double red[32];
  const unsigned long long pol_keep = l2_policy_evict_last(), pol_stream = l2_policy_evict_first();
  // rank sort of the (distinct) shifts
  for (int t = threadIdx.x; t < k; t += blockDim.x) {
    const int j = J[t];
    int rank = 0;
    for (int u = 0; u < k; ++u) rank += J[u] < j;
    sJT[rank] = make_int2(j, t);
  }
  const int r0 = blockIdx.x * R;
  const int rows = min(R, m_rows - r0);
  const int nseg = (int)ceil_div(n, SW);
  double xs = 0.0, msq = 0.0;
  for (int s = 0; s < nseg; ++s) {
    const int s0 = s * SW, sw = min(SW, n - s0);
    __syncthreads();  // the previous segment's readers are done (and the sort is visible)
    // fill: coalesced 16-byte row reads, transposed in registers to the interleaved layout
    {
      constexpr int V = 16 / sizeof(T);
      using Vec = typename std::conditional<sizeof(T) == 4, float4, double2>::type;
      const int nv = sw / V;
      for (int iv = threadIdx.x; iv < nv; iv += blockDim.x) {
        Vec buf[RP];
#pragma unroll
        for (int rr = 0; rr < RP; ++rr)
          buf[rr] = rr < rows ? __ldg(reinterpret_cast<const Vec*>(X + (size_t)(r0 + rr) * n + s0) + iv) : Vec{};
        alignas(16) T tr[V * RP];
#pragma unroll
        for (int rr = 0; rr < RP; ++rr) {
          const T* e = reinterpret_cast<const T*>(&buf[rr]);
#pragma unroll
          for (int q = 0; q < V; ++q) {
            xs = fma((double)e[q], (double)e[q], xs);
            tr[q * RP + rr] = e[q];
          }
        }
        Vec* dst = reinterpret_cast<Vec*>(Xs + (size_t)iv * V * RP);
#pragma unroll
        for (int w = 0; w < RP; ++w) dst[w] = reinterpret_cast<const Vec*>(tr)[w];
      }
    }
    if (JA != nullptr) {
      __syncthreads();
      for (int e = threadIdx.x; e < rows * ka; e += blockDim.x) {
        const int rr = e / ka, t = e - rr * ka;
        int m = (r0 + rr + row_off - JA[t]) % n;
        if (m < 0) m += n;
        if (m >= s0 && m < s0 + sw) Xs[(size_t)(m - s0) * RP + rr] = T(0);
      }
    }
    __syncthreads();
    const bool last = s == nseg - 1;
    if (threadIdx.x == 0 && s + 1 < nseg) {  // next segment's rows toward L2 while this one runs
      const int n1 = min(SW, n - (s0 + SW));
      for (int rr = 0; rr < rows; ++rr)
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(X + (size_t)(r0 + rr) * n + s0 + SW),
                     "r"((unsigned)(n1 * sizeof(T)))
                     : "memory");
    }
    const int lane = threadIdx.x & 31;
    constexpr int CW = 32 * CPT;  // a warp's column chunk: lane + 32 q, q < CPT
    const T* xlane = Xs + (size_t)lane * RP;
    // output columns [c_lo, c_hi) (all n, or a sharded block); lambda' column c at lam_c[c - c_lo]
    // in rows of stride lam_ld; M column c at M_c[c - c_lo] in rows of stride out_ld
    for (int cw = c_lo + (threadIdx.x >> 5) * CW; cw < c_hi; cw += (blockDim.x >> 5) * CW) {
      // The chunk's source window under shift J is [m0, m0 + CW), m0 = (cw + J) mod n.
      //  interior: the window lies inside the segment (m0 in [s0, s0 + sw - CW]): one warp-uniform
      //            offset, no per-lane checks;
      //  boundary: the window straddles a segment end (m0 in [s0 - CW + 1, s0) or
      //            (s0 + sw - CW, s0 + sw)): per-lane checks, ~2 such shifts per chunk over the sweep.
      // Each is a cyclic interval of J values, i.e. a cyclic run of the sorted table.
      auto lower = [&](int v) -> int { return (k <= 256 && (TUNE & 2)) ? count_below(sJT, k, v) : lower_index(sJT, k, v, 0); };
      auto run = [&](int v, int len, int& first) -> int {  // J in [v, v + len) mod n, len < n
        v %= n;
        if (v < 0) v += n;
        first = lower(v);
        int cnt;
        if (v + len <= n) {
          cnt = lower(v + len) - first;
        } else {
          cnt = (k - first) + min(lower(v + len - n), first);
        }
        if (first >= k) first -= k;  // every shift is below v: the run starts at index 0
        return cnt;
      };
      int f_int, f_lo, f_hi;
      const int c_int = run(s0 - cw, sw - CW + 1, f_int);
      const int n_blo = run(s0 - CW + 1 - cw, CW - 1, f_lo);
      const int n_bhi = nseg > 1 ? run(s0 + sw - CW + 1 - cw, CW - 1, f_hi) : 0;
      // A segment that is neither the first of an overwriting pass nor the last adds its partial
      // sums with fire-and-forget reductions at L2 (red.add: no old value to wait for -- the
      // epilogue's load stalls were ~17% of the samples); the last segment needs the final values
      // for ||M||^2 and reads them back (relaxed loads: program order behind this thread's own
      // reductions on the same addresses). Otherwise: the chunk's M lines toward L2.
      const bool rmw = s > 0 || accumulate != 0;
      const bool red = rmw && !last && (TUNE & 1);
      if (rmw && !red) {
#pragma unroll
        for (int q = 0; q < CPT; ++q)
#pragma unroll
          for (int rr = 0; rr < R; ++rr)
            if (rr < rows)
              asm volatile("prefetch.global.L2 [%0];" ::"l"(M + (size_t)(r0 + rr) * out_ld + (cw - c_lo) + 32 * q + lane));
      }
      unsigned long long acc2[CPT][NP > 0 ? NP : 1];
      T accs[CPT][NS > 0 ? NS : 1];
#pragma unroll
      for (int q = 0; q < CPT; ++q) {
#pragma unroll
        for (int p = 0; p < (NP > 0 ? NP : 1); ++p) acc2[q][p] = 0ull;
#pragma unroll
        for (int p = 0; p < (NS > 0 ? NS : 1); ++p) accs[q][p] = T(0);
      }
      auto fma_rows = [&](int q, const T* xp, T l) {
        if constexpr (NP > 0) {
          const unsigned long long l2 = pack2((float)l, (float)l);
          const unsigned long long* xp2 = reinterpret_cast<const unsigned long long*>(xp);
#pragma unroll
          for (int p = 0; p < NP; ++p) acc2[q][p] = ffma2(xp2[p], l2, acc2[q][p]);
        }
        if constexpr (NS > 0) {
#pragma unroll
          for (int p = 0; p < NS; ++p) accs[q][p] = fma(xp[2 * NP + p], l, accs[q][p]);
        }
      };
      // interior shifts, kSegU per batch, batch i+1's lambda loads in flight while batch i is
      // consumed. off[u]: the warp-uniform source offset (m0 - s0) * RP of shift u.
      auto load_batch = [&](int i0, int (&off)[kSegU], T (&lv)[kSegU][CPT]) {
#pragma unroll
        for (int u = 0; u < kSegU; ++u) {
          int i = f_int + i0 + u;
          i = i >= k ? i - k : i;
          const bool in = i0 + u < c_int;
          const int2 jt = sJT[in ? i : f_int];  // broadcast
          unsigned m = (unsigned)(cw + jt.x);
          m = min(m, m - (unsigned)n);  // (cw + J) mod n
          off[u] = in ? (int)(m - (unsigned)s0) * RP : 0;
          const T* lrow = lam + (size_t)jt.y * lam_ld + (cw - c_lo) + lane;
#pragma unroll
          for (int q = 0; q < CPT; ++q) lv[u][q] = in ? ldg_nc_hint(lrow + 32 * q, pol_keep) : T(0);
        }
      };
      auto compute_batch = [&](const int (&off)[kSegU], const T (&lv)[kSegU][CPT]) {
#pragma unroll
        for (int u = 0; u < kSegU; ++u)
#pragma unroll
          for (int q = 0; q < CPT; ++q) fma_rows(q, xlane + off[u] + 32 * q * RP, lv[u][q]);
      };
      {
        int oA[kSegU], oB[kSegU];
        T lvA[kSegU][CPT], lvB[kSegU][CPT];
        if (c_int > 0) load_batch(0, oA, lvA);
        for (int i0 = 0; i0 < c_int; i0 += 2 * kSegU) {
          if (i0 + kSegU < c_int) load_batch(i0 + kSegU, oB, lvB);
          compute_batch(oA, lvA);
          if (i0 + kSegU >= c_int) break;
          if (i0 + 2 * kSegU < c_int) load_batch(i0 + 2 * kSegU, oA, lvA);
          compute_batch(oB, lvB);
        }
      }
      // boundary shifts: per-lane segment test; lanes outside read offset 0 with a zero lambda
      auto boundary = [&](int first, int cnt) {
        for (int e = 0; e < cnt; ++e) {
          int i = first + e;
          i = i >= k ? i - k : i;
          const int2 jt = sJT[i];
          const T* lrow = lam + (size_t)jt.y * lam_ld;
          T lv[CPT];
          unsigned l[CPT];
#pragma unroll
          for (int q = 0; q < CPT; ++q) {
            const int c = cw + 32 * q + lane;
            unsigned m = (unsigned)(c + jt.x);
            m = min(m, m - (unsigned)n);
            const unsigned d = m - (unsigned)s0;
            const bool ok = d < (unsigned)sw;
            l[q] = ok ? d : 0u;
            lv[q] = ok ? __ldg(lrow + (c - c_lo)) : T(0);
          }
#pragma unroll
          for (int q = 0; q < CPT; ++q) fma_rows(q, Xs + (size_t)l[q] * RP, lv[q]);
        }
      };
      boundary(f_lo, n_blo);
      boundary(f_hi, n_bhi);
      // M (+)= the segment's partial sums: the first segment applies `accumulate`, later ones
      // add (subtract for accumulate < 0); all old values are loaded before the first store
      T old[CPT][R];
#pragma unroll
      for (int q = 0; q < CPT; ++q)
#pragma unroll
        for (int rr = 0; rr < R; ++rr)
          old[q][rr] = (rr < rows && rmw && !red)
                           ? ld_relaxed(M + (size_t)(r0 + rr) * out_ld + (cw - c_lo) + 32 * q + lane)
                           : T(0);
#pragma unroll
      for (int q = 0; q < CPT; ++q)
#pragma unroll
        for (int rr = 0; rr < R; ++rr) {
          T a;
          if constexpr (NP > 0) {
            if (rr < 2 * NP) {
              const unsigned long long v = acc2[q][rr >> 1];
              a = (T)__uint_as_float((unsigned)(rr & 1 ? (v >> 32) : (v & 0xffffffffull)));
            } else {
              a = accs[q][rr - 2 * NP];
            }
          } else {
            a = accs[q][rr];
          }
          if (rr < rows) {
            T* mp = M + (size_t)(r0 + rr) * out_ld + (cw - c_lo) + 32 * q + lane;
            if (red) {
              red_add(mp, accumulate < 0 ? -a : a);
            } else {
              const T v = accumulate < 0 ? old[q][rr] - a : old[q][rr] + a;
              stg_hint(mp, v, pol_stream);
              if (last) msq += (double)v * (double)v;
            }
          }
        }
    }
  }
  if (xsq_partial != nullptr) {
    const double t = block_sum(xs, red);
    if (threadIdx.x == 0) xsq_partial[blockIdx.x] = t;
  }
  if (msq_partial != nullptr) {
    const double t = block_sum(msq, red);
    if (threadIdx.x == 0) msq_partial[blockIdx.x] = t;
  }
}

// ------------------------------------------------------------------------------------------
// K11h: the segmented gather over a small masked residual, staged as scaled f16 (fp32 only).
// The order-1 cycle product's second term dX . Bhat (dX = X with its kept cycles masked on load)
// is a small part of M whenever the kept cycles carry the operand (C5: 1.6% of ||A||_F), so --
// as in the C4 residual plan (mixed_f16.cu) -- dX is staged as 2^(15 - e_X) dX in f16 (e_X from
// ||X||_F: no entry can overflow, masked or not) and the kept diagonals of B as 2^(15 - e_B)
// lambda' in f16 (a k x n table made once per product); products are f16 x f16 with fp32
// accumulation (fma.rn.f32.f16), rescaled by 2^(e_X + e_B - 30) once per output and segment.
// Shared memory holds 8 rows x SW columns as one 16-byte vector per column: a warp's load of 32
// columns is 4 wavefronts for 256 FMAs (the fp32 kernel at R = 6: 6 for 192), plus one 64-byte
// lambda' wavefront per 16 loads (thread-order f16 table, 8 bytes per shift); the segment is twice as wide, so M is read-modified-written
// 3 times instead of 5 at n = 32768. Runs only when resid_small() holds (device-side decision;
// cycle_right_gather_seg is launched behind it as the fallback and returns at once otherwise).
// Accumulation order per output: segments ascending, in a segment the sorted interior run and
// then the two boundary runs -- independent of the row blocking, so row-sharded runs reproduce
// the single-device bits.
// ------------------------------------------------------------------------------------------
constexpr int kSegHR = 8;

__device__ __forceinline__ float fhfma_seg(unsigned short a, unsigned short b, float c) {
  float d;
  asm("fma.rn.f32.f16 %0, %1, %2, %3;" : "=f"(d) : "h"(a), "h"(b), "f"(c));
  return d;
}

// f16 lambda' table in the gather's thread order: within each 128-column chunk the four columns
// lane + 32 q (q < 4) of one lane sit together, lamh[t][chunk * 128 + lane * 4 + q] =
// f16(2^(15 - e_B) lam[t][chunk * 128 + 32 q + lane]), so a thread's four columns of one shift are
// ONE 8-byte load (a warp: 256 contiguous bytes) instead of four 2-byte loads.
__global__ void lam_seg_f16_kernel(const float* __restrict__ lam, size_t count, const double* __restrict__ fro2_b,
                                   unsigned short* __restrict__ out, const double* __restrict__ g_fro2,
                                   const double* __restrict__ g_kept) {
  if (g_fro2 != nullptr && !resid_small(g_fro2, g_kept)) return;
  const float s = ldexpf(1.f, 15 - f16_scale_exp(*fro2_b));
  const size_t nth = (size_t)gridDim.x * blockDim.x;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < count / 4; i += nth) {
    const size_t chunk = i >> 5, lane = i & 31;  // chunks run through the rows (n % 128 == 0)
    const float* src = lam + chunk * 128 + lane;
    uint2 o;
    o.x = pack_half2(s * src[0], s * src[32]);
    o.y = pack_half2(s * src[64], s * src[96]);
    *reinterpret_cast<uint2*>(out + chunk * 128 + lane * 4) = o;
  }
}
__device__ __forceinline__ uint2 ldg_nc_hint_u64(const unsigned short* a, unsigned long long pol) {
  uint2 v;
  asm volatile("ld.global.nc.L2::cache_hint.v2.u32 {%0, %1}, [%2], %3;" : "=r"(v.x), "=r"(v.y) : "l"(a), "l"(pol));
  return v;
}

template <int TUNE>
__global__ void __launch_bounds__(kSegThreads, 1)
    cycle_right_gather_seg_h(const float* __restrict__ X, const int* __restrict__ JA, int ka,
                             const unsigned short* __restrict__ lamh, const int* __restrict__ J, int k, int n,
                             int m_rows, int accumulate, float* __restrict__ M, double* __restrict__ msq_partial,
                             int SW, int row_off, int lam_ld, const double* __restrict__ g_fro2,
                             const double* __restrict__ g_kept, const double* __restrict__ fro2_b, int force) {
  if (!force && !resid_small(g_fro2, g_kept)) return;
  constexpr int R = kSegHR, CPT = 4;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  uint4* Xs = reinterpret_cast<uint4*>(smem_raw);  // column m of the segment: rows r0..r0+7 as f16
  int2* sJT = reinterpret_cast<int2*>(Xs + SW);   // (shift, lambda row), ascending shift
  __shared__ double red[32];
  const unsigned long long pol_keep = l2_policy_evict_last(), pol_stream = l2_policy_evict_first();
  const int e_x = f16_scale_exp(*g_fro2), e_b = f16_scale_exp(*fro2_b);
  const float sx = ldexpf(1.f, 15 - e_x), inv = ldexpf(1.f, e_x + e_b - 30);
  for (int t = threadIdx.x; t < k; t += blockDim.x) {
    const int j = J[t];
    int rank = 0;
    for (int u = 0; u < k; ++u) rank += J[u] < j;
    sJT[rank] = make_int2(j, t);
  }
  const int r0 = blockIdx.x * R;
  const int rows = min(R, m_rows - r0);
  const int nseg = (int)ceil_div(n, SW);
  double msq = 0.0;
  for (int s = 0; s < nseg; ++s) {
    const int s0 = s * SW, sw = min(SW, n - s0);
    __syncthreads();  // the previous segment's readers are done (and the sort is visible)
    // fill: coalesced 16-byte reads of 8 rows, 4 columns per thread step, scaled and packed
    for (int iv = threadIdx.x; iv < sw / 4; iv += blockDim.x) {
      float4 buf[R];
#pragma unroll
      for (int rr = 0; rr < R; ++rr)
        buf[rr] = rr < rows ? __ldg(reinterpret_cast<const float4*>(X + (size_t)(r0 + rr) * n + s0) + iv)
                            : float4{0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        float e[R];
#pragma unroll
        for (int rr = 0; rr < R; ++rr) e[rr] = sx * reinterpret_cast<const float*>(&buf[rr])[q];
        uint4 o;
        o.x = pack_half2(e[0], e[1]);
        o.y = pack_half2(e[2], e[3]);
        o.z = pack_half2(e[4], e[5]);
        o.w = pack_half2(e[6], e[7]);
        Xs[iv * 4 + q] = o;
      }
    }
    if (JA != nullptr) {
      __syncthreads();
      unsigned short* Xh = reinterpret_cast<unsigned short*>(Xs);
      for (int e = threadIdx.x; e < rows * ka; e += blockDim.x) {
        const int rr = e / ka, t = e - rr * ka;
        int m = (r0 + rr + row_off - JA[t]) % n;
        if (m < 0) m += n;
        APX_DCHECK(m >= 0 && m < n);
        if (m >= s0 && m < s0 + sw) Xh[(size_t)(m - s0) * R + rr] = 0;
      }
    }
    __syncthreads();
    const bool last = s == nseg - 1;
    if (threadIdx.x == 0 && s + 1 < nseg) {  // next segment's rows toward L2 while this one runs
      const int n1 = min(SW, n - (s0 + SW));
      for (int rr = 0; rr < rows; ++rr)
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(X + (size_t)(r0 + rr) * n + s0 + SW),
                     "r"((unsigned)(n1 * sizeof(float)))
                     : "memory");
    }
    const int lane = threadIdx.x & 31;
    constexpr int CW = 32 * CPT;
    const uint4* xlane = Xs + lane;
    for (int cw = (threadIdx.x >> 5) * CW; cw < n; cw += (blockDim.x >> 5) * CW) {
      // interior / boundary runs of the sorted shift table, as in cycle_right_gather_seg
      auto lower = [&](int v) -> int { return (k <= 256 && (TUNE & 2)) ? count_below(sJT, k, v) : lower_index(sJT, k, v, 0); };
      auto run = [&](int v, int len, int& first) -> int {
        v %= n;
        if (v < 0) v += n;
        first = lower(v);
        int cnt;
        if (v + len <= n) {
          cnt = lower(v + len) - first;
        } else {
          cnt = (k - first) + min(lower(v + len - n), first);
        }
        if (first >= k) first -= k;
        return cnt;
      };
      int f_int, f_lo, f_hi;
      const int c_int = run(s0 - cw, sw - CW + 1, f_int);
      const int n_blo = run(s0 - CW + 1 - cw, CW - 1, f_lo);
      const int n_bhi = nseg > 1 ? run(s0 + sw - CW + 1 - cw, CW - 1, f_hi) : 0;
      // red: a segment that is neither the first of an overwriting pass nor the last adds its
      // partial sums with fire-and-forget reductions at L2 (no old-value load to wait for); the
      // last segment needs the final values (||M||^2), so it reads them back (relaxed, from L2:
      // program order after this thread's own reductions on the same addresses)
      const bool rmw = s > 0 || accumulate != 0;
      const bool red = rmw && !last && (TUNE & 1);
      if (rmw && !red) {
#pragma unroll
        for (int q = 0; q < CPT; ++q)
#pragma unroll
          for (int rr = 0; rr < R; ++rr)
            if (rr < rows) asm volatile("prefetch.global.L2 [%0];" ::"l"(M + (size_t)(r0 + rr) * n + cw + 32 * q + lane));
      }
      float acc[CPT][R];
#pragma unroll
      for (int q = 0; q < CPT; ++q)
#pragma unroll
        for (int rr = 0; rr < R; ++rr) acc[q][rr] = 0.f;
      auto fma_rows = [&](int q, const uint4 x, unsigned short l) {
        acc[q][0] = fhfma_seg((unsigned short)(x.x & 0xffffu), l, acc[q][0]);
        acc[q][1] = fhfma_seg((unsigned short)(x.x >> 16), l, acc[q][1]);
        acc[q][2] = fhfma_seg((unsigned short)(x.y & 0xffffu), l, acc[q][2]);
        acc[q][3] = fhfma_seg((unsigned short)(x.y >> 16), l, acc[q][3]);
        acc[q][4] = fhfma_seg((unsigned short)(x.z & 0xffffu), l, acc[q][4]);
        acc[q][5] = fhfma_seg((unsigned short)(x.z >> 16), l, acc[q][5]);
        acc[q][6] = fhfma_seg((unsigned short)(x.w & 0xffffu), l, acc[q][6]);
        acc[q][7] = fhfma_seg((unsigned short)(x.w >> 16), l, acc[q][7]);
      };
      auto load_batch = [&](int i0, int (&off)[kSegU], uint2 (&lv)[kSegU]) {
#pragma unroll
        for (int u = 0; u < kSegU; ++u) {
          int i = f_int + i0 + u;
          i = i >= k ? i - k : i;
          const bool in = i0 + u < c_int;
          const int2 jt = sJT[in ? i : f_int];  // broadcast
          unsigned m = (unsigned)(cw + jt.x);
          m = min(m, m - (unsigned)n);  // (cw + J) mod n
          off[u] = in ? (int)(m - (unsigned)s0) : 0;
          lv[u] = in ? ldg_nc_hint_u64(lamh + (size_t)jt.y * lam_ld + cw + lane * 4, pol_keep) : uint2{0u, 0u};
        }
      };
      auto compute_batch = [&](const int (&off)[kSegU], const uint2 (&lv)[kSegU]) {
#pragma unroll
        for (int u = 0; u < kSegU; ++u) {
          APX_DCHECK(off[u] >= 0 && off[u] + 96 + lane < sw);
          fma_rows(0, xlane[off[u]], (unsigned short)(lv[u].x & 0xffffu));
          fma_rows(1, xlane[off[u] + 32], (unsigned short)(lv[u].x >> 16));
          fma_rows(2, xlane[off[u] + 64], (unsigned short)(lv[u].y & 0xffffu));
          fma_rows(3, xlane[off[u] + 96], (unsigned short)(lv[u].y >> 16));
        }
      };
      {
        int oA[kSegU], oB[kSegU];
        uint2 lvA[kSegU], lvB[kSegU];
        if (c_int > 0) load_batch(0, oA, lvA);
        for (int i0 = 0; i0 < c_int; i0 += 2 * kSegU) {
          if (i0 + kSegU < c_int) load_batch(i0 + kSegU, oB, lvB);
          compute_batch(oA, lvA);
          if (i0 + kSegU >= c_int) break;
          if (i0 + 2 * kSegU < c_int) load_batch(i0 + 2 * kSegU, oA, lvA);
          compute_batch(oB, lvB);
        }
      }
      auto boundary = [&](int first, int cnt) {
        for (int e = 0; e < cnt; ++e) {
          int i = first + e;
          i = i >= k ? i - k : i;
          const int2 jt = sJT[i];
          const unsigned short* lrow = lamh + (size_t)jt.y * lam_ld;
          unsigned short lv[CPT];
          unsigned l[CPT];
#pragma unroll
          for (int q = 0; q < CPT; ++q) {
            const int c = cw + 32 * q + lane;
            unsigned m = (unsigned)(c + jt.x);
            m = min(m, m - (unsigned)n);
            const unsigned d = m - (unsigned)s0;
            const bool ok = d < (unsigned)sw;
            l[q] = ok ? d : 0u;
            lv[q] = ok ? __ldg(lrow + cw + lane * 4 + q) : (unsigned short)0;
          }
#pragma unroll
          for (int q = 0; q < CPT; ++q) {
            APX_DCHECK(l[q] < (unsigned)sw);
            fma_rows(q, Xs[l[q]], lv[q]);
          }
        }
      };
      boundary(f_lo, n_blo);
      boundary(f_hi, n_bhi);
      // M (+)= the segment's partial sums, one column of the chunk at a time (8 old values in
      // flight per thread; the lines were prefetched into L2 at the chunk's start)
      if (red) {
#pragma unroll
        for (int q = 0; q < CPT; ++q)
#pragma unroll
          for (int rr = 0; rr < R; ++rr)
            if (rr < rows) {
              const float a = acc[q][rr] * inv;
              red_add(M + (size_t)(r0 + rr) * n + cw + 32 * q + lane, accumulate < 0 ? -a : a);
            }
      } else {
#pragma unroll
        for (int q = 0; q < CPT; ++q) {
          float old[R];
#pragma unroll
          for (int rr = 0; rr < R; ++rr)
            old[rr] = (rmw && rr < rows) ? ld_relaxed_f32(M + (size_t)(r0 + rr) * n + cw + 32 * q + lane) : 0.f;
#pragma unroll
          for (int rr = 0; rr < R; ++rr)
            if (rr < rows) {
              const float a = acc[q][rr] * inv;
              const float v = (accumulate < 0) ? old[rr] - a : old[rr] + a;
              stg_hint(M + (size_t)(r0 + rr) * n + cw + 32 * q + lane, v, pol_stream);
              if (last) msq += (double)v * (double)v;
            }
        }
      }
    }
  }
  if (msq_partial != nullptr) {
    const double t = block_sum(msq, red);
    if (threadIdx.x == 0) msq_partial[blockIdx.x] = t;
  }
}

// sum of |x|^2 over a dense array, per-block partials (for ||M||_F when no gather wrote M last)
template <typename T>
__global__ void __launch_bounds__(256) sumsq_partial_kernel(const T* __restrict__ x, size_t cnt,
                                                            double* __restrict__ partial) {
  __shared__ double red[32];
  double s = 0.0;
  const size_t tid = blockIdx.x * (size_t)blockDim.x + threadIdx.x, nth = (size_t)gridDim.x * blockDim.x;
  // 16-byte vectors, four in flight per thread (a scalar loop ran at a third of the HBM rate)
  using Vec = typename std::conditional<sizeof(T) == 4, float4, double2>::type;
  constexpr int V = 16 / sizeof(T);
  size_t head = 0;
  if (((uintptr_t)x & 15) == 0) {
    const size_t nv = cnt / V;
    const Vec* xv = reinterpret_cast<const Vec*>(x);
    size_t e = tid;
    for (; e + 3 * nth < nv; e += 4 * nth) {
      Vec v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) v[u] = __ldg(xv + e + u * nth);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const T* f = reinterpret_cast<const T*>(&v[u]);
#pragma unroll
        for (int q = 0; q < V; ++q) s = fma((double)f[q], (double)f[q], s);
      }
    }
    for (; e < nv; e += nth) {
      const Vec v = __ldg(xv + e);
      const T* f = reinterpret_cast<const T*>(&v);
#pragma unroll
      for (int q = 0; q < V; ++q) s = fma((double)f[q], (double)f[q], s);
    }
    head = nv * V;
  }
  for (size_t e = head + tid; e < cnt; e += nth) {
    const double v = (double)x[e];
    s += v * v;
  }
  s = block_sum(s, red);
  if (threadIdx.x == 0) partial[blockIdx.x] = s;
}

// ------------------------------------------------------------------------------------------
// host-side launchers
// ------------------------------------------------------------------------------------------
template <typename T>
static int set_smem(const void* fn, size_t bytes) {
  if (bytes > 48 * 1024) APX_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
  return OK;
}

static int energy_groups(int n, int* rows_per_chunk, int ctas_per_sm = 8) {
  const int cblocks = (int)ceil_div(n, 256);
  // one full wave of 8 CTAs per SM (launch bounds (256, 8)): rounding up left a 0.33-wave tail;
  // fewer CTAs per SM leave room for a concurrent latency-bound chain (the C4 residual plan's QR)
  int groups = std::max(1, (kNumSMs * ctas_per_sm) / cblocks);
  // at most 40 row groups: the finalize sums one column's groups per thread (n threads), so a
  // small n with many groups made it the slow part (53 us at n = 2048 with 128 groups)
  groups = std::max(1, std::min({groups, (int)ceil_div(n, 16), 40}));
  *rows_per_chunk = (int)ceil_div(n, groups);
  return (int)ceil_div(n, *rows_per_chunk);
}

// workspace of an energy pass with `groups` row groups (launch_cycle_energies' groups_override)
size_t cycle_energy_ws_groups(int n, int groups) {
  return (size_t)std::max(groups, 1) * n * sizeof(double) + ceil_div(n, 256) * sizeof(unsigned) + 256;
}

size_t cycle_energy_ws(int n) {
  int rpc;
  int g = energy_groups(n, &rpc);
  if (rows4_ok(n)) g = std::max(g, rows4_groups(n, &rpc));
  return (size_t)g * n * sizeof(double) + ceil_div(n, 256) * sizeof(unsigned) + 256;
}

template <typename T>
int launch_cycle_energies(const T* A, int n, double* energies, double* norms, double* fro2, double* partial,
                          cudaStream_t st, int ctas_per_sm, int groups_override, int rows4_ctas) {
  int rpc;
  int groups = energy_groups(n, &rpc, ctas_per_sm);
  if (groups_override > 0) {  // many short-lived CTAs (several waves), see cycle_energy_ws_groups
    rpc = (int)ceil_div(n, std::min(groups_override, n));
    groups = (int)ceil_div(n, rpc);
  }
  if (std::is_same<T, float>::value && rows4_ok(n) && groups_override <= 0) {
    groups = rows4_groups(n, &rpc, rows4_ctas);
    const size_t smem = rows4_smem(n);
    APX_CUDA(cudaFuncSetAttribute(cycle_energy_rows4_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    cycle_energy_rows4_kernel<<<(unsigned)groups, kEnThreads, smem, st>>>(reinterpret_cast<const float*>(A), n, rpc, partial);
    APX_LAUNCH_CHECK();
  } else {
    const unsigned cb = (unsigned)ceil_div(n, 256);
    dim3 grid(cb, (unsigned)groups);
    // separate finalize: the fused last-CTA reduce (counters != nullptr) measured 63 us vs 44 + 7
    cycle_energy_partial<T><<<grid, 256, 0, st>>>(A, n, rpc, partial, nullptr, energies, norms, n, 0);
    APX_LAUNCH_CHECK();
  }
  APX_CUDA(launch_pdl(cycle_energy_finalize, dim3((unsigned)ceil_div(n, 32)), dim3(256), 0, st, partial, n, groups,
                      energies, norms));
  APX_LAUNCH_CHECK();
  if (fro2) {
    sum_vector_kernel<<<1, 1024, 0, st>>>(energies, n, fro2);
    APX_LAUNCH_CHECK();
  }
  return OK;
}

// energies over a row block (local rows [0, m), global rows row_off + r) of an n x n operand:
// the partial vector a row-sharded product sums over ranks (no norms)
template <typename T>
int launch_cycle_energies_rows(const T* A, int m, int row_off, int n, double* energies, double* partial,
                               cudaStream_t st) {
  const unsigned cb = (unsigned)ceil_div(n, 256);
  const int groups = std::max(1, std::min({(kNumSMs * 8) / (int)cb, (int)ceil_div(m, 16), 40}));
  const int rpc = (int)ceil_div(m, groups);
  const int g = (int)ceil_div(m, rpc);
  cycle_energy_partial<T><<<dim3(cb, (unsigned)g), 256, 0, st>>>(A, n, rpc, partial, nullptr, energies, nullptr, m,
                                                                 row_off);
  APX_LAUNCH_CHECK();
  APX_CUDA(launch_pdl(cycle_energy_finalize, dim3((unsigned)ceil_div(n, 32)), dim3(256), 0, st, partial, n, g, energies,
                      (double*)nullptr));
  APX_LAUNCH_CHECK();
  return OK;
}

int launch_topk(const double* w, int n, int k, int* sel, cudaStream_t st, const double* kept_w, double kept_scale,
                double* kept, const double* tot_w, double* total) {
  if (k <= 0 && !kept && !total) return OK;
  APX_CUDA(launch_pdl(topk_select_kernel, dim3(1), dim3(kSelThreads), 0, st, w, n, k, sel, kept_w, kept_scale, kept,
                      tot_w, total));
  APX_LAUNCH_CHECK();
  return OK;
}

int launch_kept_energy(const double* norms, const int* sel, int k, double scale, double* out, cudaStream_t st) {
  kept_energy_kernel<<<1, 32, 0, st>>>(norms, sel, k, scale, out);
  APX_LAUNCH_CHECK();
  return OK;
}

template <typename T>
int launch_cycle_extract(const T* A, int n, const int* J, int k, T* lam, cudaStream_t st, bool aligned) {
  if (k <= 0) return OK;
  dim3 grid((unsigned)ceil_div(n, 256), (unsigned)ceil_div(k, kExtractT));
  if (aligned)
    APX_CUDA(launch_pdl(cycle_extract<T, true>, grid, dim3(256), 0, st, A, n, J, k, lam, n, 0));
  else
    APX_CUDA(launch_pdl(cycle_extract<T, false>, grid, dim3(256), 0, st, A, n, J, k, lam, n, 0));
  APX_LAUNCH_CHECK();
  return OK;
}

// left-layout lambdas of a row block (local rows [0, m), global row_off + i): k x m table
template <typename T>
int launch_cycle_extract_rows(const T* A, int m, int row_off, int n, const int* J, int k, T* lam, cudaStream_t st) {
  if (k <= 0) return OK;
  dim3 grid((unsigned)ceil_div(m, 256), (unsigned)ceil_div(k, kExtractT));
  cycle_extract<T, false><<<grid, 256, 0, st>>>(A, n, J, k, lam, m, row_off);
  APX_LAUNCH_CHECK();
  return OK;
}

template <typename T>
int launch_cycle_materialize(const T* lam, const int* J, int k, int n, T* out, cudaStream_t st) {
  cycle_materialize_kernel<T><<<kNumSMs * 4, 256, 0, st>>>(lam, J, k, n, out);
  APX_LAUNCH_CHECK();
  if (k > 0) {
    dim3 grid((unsigned)ceil_div(n, 256), (unsigned)k);
    cycle_scatter_kernel<T><<<grid, 256, 0, st>>>(lam, J, k, n, out);
    APX_LAUNCH_CHECK();
  }
  return OK;
}

constexpr size_t kSmemBudget = 200 * 1024;

template <typename T, int W>
static int left_gather_w(const T* X, const T* lam, const int* J, int k, int n, int acc, T* M, cudaStream_t st,
                         int r_lo = 0, int r_hi = -1, int lam_ld = -1) {
  if (r_hi < 0) r_hi = n;
  if (lam_ld < 0) lam_ld = n;
  constexpr int S = (W == 1) ? 1 : W + 1;
  const size_t smem = (size_t)n * S * sizeof(T) + (size_t)std::max(k, 1) * sizeof(int);
  APX_TRY(set_smem<T>((const void*)cycle_left_gather<T, W>, smem));
  const int strips = (int)ceil_div(n, W);
  int groups = 1;
  const int rows = r_hi - r_lo;
  if (strips < 2 * kNumSMs) groups = std::min<int>((int)ceil_div(2 * kNumSMs, strips), std::max(1, rows / kLeftThreads));
  dim3 grid((unsigned)strips, (unsigned)groups);
  cycle_left_gather<T, W><<<grid, kLeftThreads, smem, st>>>(X, lam, J, k, n, acc, M, r_lo, r_hi, lam_ld);
  APX_LAUNCH_CHECK();
  return OK;
}

__global__ void negate_shifts_kernel(const int* __restrict__ J, int k, int n, int* __restrict__ out) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < k) out[t] = J[t] == 0 ? 0 : n - J[t];
}

int launch_negate_shifts(const int* J, int k, int n, int* out, cudaStream_t st) {
  if (k <= 0) return OK;
  negate_shifts_kernel<<<(unsigned)ceil_div(k, 256), 256, 0, st>>>(J, k, n, out);
  APX_LAUNCH_CHECK();
  return OK;
}

static int left_strip_width(int n, size_t elem) {
  const size_t per_col = (size_t)n * elem;
  int w = 1;
  while (w < 8 && (size_t)(2 * w + 1) * per_col <= kSmemBudget) w *= 2;
  return w;
}

bool left_via_transpose(int n, size_t elem, int k) {
  return left_strip_width(n, elem) <= 2 && (n % (kGatherThreads * APX_GATHER_CPT)) == 0 && k > 0;
}

template <typename T>
int launch_cycle_left_gather(const T* X, const T* lam, const int* J, int k, int n, int accumulate, T* M,
                             cudaStream_t st) {
  const size_t per_col = (size_t)n * sizeof(T);
  int w = 1;
  while (w < 8 && (size_t)(2 * w + 1) * per_col <= kSmemBudget) w *= 2;
  APX_REQUIRE((size_t)(w == 1 ? 1 : w + 1) * per_col <= 227 * 1024, "n=%d too large for the left gather strip", n);
  switch (w) {
    case 1: return left_gather_w<T, 1>(X, lam, J, k, n, accumulate, M, st);
    case 2: return left_gather_w<T, 2>(X, lam, J, k, n, accumulate, M, st);
    case 4: return left_gather_w<T, 4>(X, lam, J, k, n, accumulate, M, st);
    default: return left_gather_w<T, 8>(X, lam, J, k, n, accumulate, M, st);
  }
}

// output rows [r_lo, r_hi) of Ahat . X into M_rows ((r_hi - r_lo) x n); lam: k x (r_hi - r_lo)
// left-layout table of those rows. Strip path only (left_via_transpose false).
template <typename T>
int launch_cycle_left_gather_rows(const T* X, const T* lam, const int* J, int k, int n, int r_lo, int r_hi, T* M_rows,
                                  cudaStream_t st) {
  const size_t per_col = (size_t)n * sizeof(T);
  int w = 1;
  while (w < 8 && (size_t)(2 * w + 1) * per_col <= kSmemBudget) w *= 2;
  APX_REQUIRE((size_t)(w == 1 ? 1 : w + 1) * per_col <= 227 * 1024, "n=%d too large for the left gather strip", n);
  const int ld = r_hi - r_lo;
  switch (w) {
    case 1: return left_gather_w<T, 1>(X, lam, J, k, n, 0, M_rows, st, r_lo, r_hi, ld);
    case 2: return left_gather_w<T, 2>(X, lam, J, k, n, 0, M_rows, st, r_lo, r_hi, ld);
    case 4: return left_gather_w<T, 4>(X, lam, J, k, n, 0, M_rows, st, r_lo, r_hi, ld);
    default: return left_gather_w<T, 8>(X, lam, J, k, n, 0, M_rows, st, r_lo, r_hi, ld);
  }
}

template <typename T, int R>
static int right_gather_r(const T* X, const int* JA, int ka, const T* lam, const int* J, int k, int n, int m_rows,
                          int acc, T* M, double* msq_partial, double* xsq_partial, bool lam_padded, int max_ctas,
                          int* ticket, int col_chunks, int trunc, int* ready, bool x_early, int row_off,
                          cudaStream_t st, const int* skip_if = nullptr) {
  constexpr int U = APX_GATHER_U, CPT = APX_GATHER_CPT;
  const int kp = (int)ceil_div(std::max(k, 1), U) * U;
  const size_t smem = (size_t)gather_pitch(R, sizeof(T)) * n * sizeof(T) + (size_t)kp * sizeof(int);
  int blocks = (int)ceil_div(m_rows, R);
  if (max_ctas > 0 && ticket) {
    // x_early: the caller zeroed the ticket before the previous kernel (a memset here would sit
    // between that kernel and this programmatic dependent launch)
    if (!x_early) APX_CUDA(cudaMemsetAsync(ticket, 0, sizeof(int), st));
    blocks = std::min(blocks, max_ctas);
  } else {
    ticket = nullptr;
  }
  const int threads = n >= kGatherThreads ? kGatherThreads : ((n + 31) / 32) * 32;
  const bool fast = lam_padded && (n % (threads * CPT)) == 0;
  // column chunks: more CTAs for short inputs (few row blocks); partial sums are per row block
  int chunks = 1;
  if (fast && !ticket && col_chunks > 1 && msq_partial == nullptr && xsq_partial == nullptr)
    chunks = std::min(col_chunks, n / (threads * CPT));
  APX_REQUIRE(ready == nullptr || chunks == 1, "right gather: ready flags need whole-row blocks");
  const dim3 grid((unsigned)blocks, (unsigned)chunks);
  auto go = [&](auto kern) -> int {
    APX_TRY(set_smem<T>((const void*)kern, smem));
    if (x_early) {
      APX_CUDA(launch_pdl(kern, grid, dim3(threads), smem, st, X, JA, ka, lam, J, k, n, m_rows, acc, M, msq_partial,
                          xsq_partial, ticket, ready, 1, row_off, skip_if));
    } else {
      kern<<<grid, threads, smem, st>>>(X, JA, ka, lam, J, k, n, m_rows, acc, M, msq_partial, xsq_partial, ticket,
                                        ready, 0, row_off, skip_if);
    }
    APX_LAUNCH_CHECK();
    return OK;
  };
  if (fast) {
    if (trunc == 1 && sizeof(T) == 4) return go(cycle_right_gather<T, R, true, 1>);
    if (trunc == 2 && sizeof(T) == 4) return go(cycle_right_gather<T, R, true, 2>);
    return go(cycle_right_gather<T, R, true>);
  }
  if (trunc == 1 && sizeof(T) == 4) return go(cycle_right_gather<T, R, false, 1>);
  if (trunc == 2 && sizeof(T) == 4) return go(cycle_right_gather<T, R, false, 2>);
  return go(cycle_right_gather<T, R, false>);
}

int right_gather_rows(int n, size_t elem, int k) {
  // fp32: up to 8 rows (even counts keep the pairs packed); fp64: 4 rows, so two CTAs share an SM
  // (C2, n = 2048: 8 rows left one 16-warp CTA per SM latency-bound, 0.28 -> 0.25 ms per product)
  int r = elem == 8 ? 4 : 8;
  while (r > 1 && (size_t)gather_pitch(r, elem) * n * elem + (size_t)(k + 8) * sizeof(int) > kSmemBudget)
    r -= (r > 2 ? 2 : 1);
  return r;
}

// Segmented gather (K11s) for the plain (non-persistent, non-TF32) call when a whole row fits at
// most twice: R rows over column segments of width SW. APX_SEG_R overrides R (tuning).
static int seg_rows(size_t elem) {
  static const int env = [] {
    const char* e = getenv("APX_SEG_R");
    return e ? atoi(e) : 0;
  }();
  if (env == 2 || env == 4 || env == 6 || env == 8) return env;
  return elem == 8 ? 4 : 6;
}
static int seg_width(int n, size_t elem, int k, int R) {
  const size_t budget = kSmemBudget - (size_t)2 * std::max(k, 1) * sizeof(int);
  const int64_t maxw = (int64_t)(budget / ((size_t)gather_pitch(R, elem) * elem)) & ~int64_t(31);
  const int64_t nseg = ceil_div(n, maxw);
  return (int)(ceil_div(ceil_div(n, nseg), 32) * 32);
}
int right_gather_seg_rows(int n, size_t elem, int k) {
  if (right_gather_rows(n, elem, k) > 2 || n % kSegThreads != 0 || k <= 0) return 0;
  return seg_rows(elem);
}
int right_gather_rows_plain(int n, size_t elem, int k) {
  const int r = right_gather_seg_rows(n, elem, k);
  return r > 0 ? r : right_gather_rows(n, elem, k);
}

// epilogue / search variant of the segmented gathers (TUNE = 3: red.add epilogue on the middle
// segments + lane-parallel shift search; 0: read-modify-write everywhere + binary search);
// APX_SEG_TUNE (fp32/fp64 kernel) and APX_SEGH_TUNE (f16-staged kernel) = 0 / 1 pick one for A/B
static int seg_tune(int fp32_kernel) {
  const char* e = getenv(fp32_kernel ? "APX_SEG_TUNE" : "APX_SEGH_TUNE");
  if (e) return atoi(e) != 0;
  // same-box A/B at C5 (n = 32768, k = 128): fp32 kernel 60.68 ms (0) vs 60.85 (3) per product --
  // it sits at 78% of the L1 data pipe either way; f16-staged kernel 52.5 (0) vs 50.1 (3)
  return fp32_kernel ? 0 : 1;
}

template <typename T, int R>
static int right_gather_seg_r(const T* X, const int* JA, int ka, const T* lam, const int* J, int k, int n,
                              int m_rows, int acc, T* M, double* msq_partial, double* xsq_partial, cudaStream_t st,
                              int row_off = 0, int c_lo = 0, int c_hi = -1, int lam_ld = -1, int out_ld = -1,
                              const double* g_fro2 = nullptr, const double* g_kept = nullptr) {
  if (c_hi < 0) c_hi = n;
  if (lam_ld < 0) lam_ld = n;
  if (out_ld < 0) out_ld = n;
  const int SW = seg_width(n, sizeof(T), k, R);
  const size_t smem = (size_t)gather_pitch(R, sizeof(T)) * SW * sizeof(T) + (size_t)2 * k * sizeof(int);
  auto kern = seg_tune(1) ? cycle_right_gather_seg<T, R, 3> : cycle_right_gather_seg<T, R, 0>;
  APX_TRY(set_smem<T>((const void*)kern, smem));
  kern<<<(unsigned)ceil_div(m_rows, R), kSegThreads, smem, st>>>(X, JA, ka, lam, J, k, n, m_rows, acc, M, msq_partial,
                                                                 xsq_partial, SW, row_off, c_lo, c_hi, lam_ld, out_ld, g_fro2, g_kept);
  APX_LAUNCH_CHECK();
  return OK;
}

// ---- f16-staged residual gather (K11h) ----
// APX_SEG_F16: 0 = never (fp32 segmented gather only), 1 = device-side rule (default), 2 = always
static int seg_f16_mode() {
  const char* e = getenv("APX_SEG_F16");
  const int v = e ? atoi(e) : 1;
  return v < 0 || v > 2 ? 1 : v;
}
bool right_gather_seg_f16_ok(int n, size_t elem, int k) {
  return elem == 4 && seg_f16_mode() != 0 && right_gather_seg_rows(n, elem, k) > 0 && n % (32 * 4) == 0;
}
size_t right_gather_seg_f16_ws(int n, int k) { return (size_t)std::max(k, 1) * n * sizeof(unsigned short) + 16; }

// M (+)= (X masked by JA) . Bhat over the segmented path, f16-staged when the residual is small
// (decided on the device from *fro2_x and *kept_x), else the fp32 segmented gather. msq_partial
// gets one partial per fp32 row block (right_gather_rows_plain rows); the f16 kernel fills the
// first ceil(m_rows / 8) of them and the rest stay zero.
int launch_cycle_right_gather_seg_f16(const float* X, const int* JA, int ka, const float* lam, const int* J, int k,
                                      int n, int m_rows, int accumulate, float* M, double* msq_partial,
                                      cudaStream_t st, int row_off, unsigned short* lamh, const double* fro2_x,
                                      const double* kept_x, const double* fro2_b) {
  const int mode = seg_f16_mode();
  APX_REQUIRE(right_gather_seg_f16_ok(n, 4, k) && JA != nullptr && lamh != nullptr, "seg f16 gather: bad call");
  const int R32 = right_gather_seg_rows(n, 4, k);
  if (msq_partial) APX_CUDA(cudaMemsetAsync(msq_partial, 0, ceil_div(m_rows, R32) * sizeof(double), st));
  const size_t cnt = (size_t)k * n;
  lam_seg_f16_kernel<<<(unsigned)std::min<size_t>(ceil_div(cnt / 4, (size_t)256), (size_t)kNumSMs * 8), 256, 0, st>>>(
      lam, cnt, fro2_b, lamh, mode == 2 ? nullptr : fro2_x, kept_x);
  APX_LAUNCH_CHECK();
  const size_t budget = 216 * 1024 - (size_t)std::max(k, 1) * sizeof(int2);
  const int64_t maxw = (int64_t)(budget / 16) & ~int64_t(127);
  const int64_t nseg = ceil_div(n, maxw);
  const int SW = (int)(ceil_div(ceil_div(n, nseg), 128) * 128);
  const size_t smem = (size_t)SW * 16 + (size_t)k * sizeof(int2);
  auto kern = seg_tune(0) ? cycle_right_gather_seg_h<3> : cycle_right_gather_seg_h<0>;
  APX_TRY(set_smem<float>((const void*)kern, smem));
  kern<<<(unsigned)ceil_div(m_rows, kSegHR), kSegThreads, smem, st>>>(
      X, JA, ka, lamh, J, k, n, m_rows, accumulate, M, msq_partial, SW, row_off, n, fro2_x, kept_x, fro2_b,
      mode == 2 ? 1 : 0);
  APX_LAUNCH_CHECK();
  if (mode == 2) return OK;
#define APX_SEGF(RV)                                                                                               \
  return right_gather_seg_r<float, RV>(X, JA, ka, lam, J, k, n, m_rows, accumulate, M, msq_partial, nullptr, st, \
                                       row_off, 0, -1, -1, -1, fro2_x, kept_x)
  switch (R32) {
    case 2: APX_SEGF(2);
    case 4: APX_SEGF(4);
    case 6: APX_SEGF(6);
    default: APX_SEGF(8);
  }
#undef APX_SEGF
}

// lam: the column-aligned table (cycle_extract<T, true>), k x n, or (lam_padded) ceil(k/8)*8 x n
// with zero rows past k -- enables the fast path. accumulate: 0 M = X.Bhat, 1 M += X.Bhat,
// -1 M -= X.Bhat. max_ctas + ticket: persistent grid; col_chunks: split the columns over CTAs;
// tf32_operands (fp32): 1 = X and lambda truncated to TF32, 2 = lambda - tf32(lambda) (see
// cycle_right_gather).
template <typename T>
int launch_cycle_right_gather(const T* X, const int* JA, int ka, const T* lam, const int* J, int k, int n,
                              int m_rows, int accumulate, T* M, double* msq_partial, double* xsq_partial,
                              cudaStream_t st, bool lam_padded, int max_ctas, int* ticket, int col_chunks,
                              int tf32_operands, int* ready, bool x_early, int row_off, const int* skip_if) {
  const int rs = right_gather_seg_rows(n, sizeof(T), k);
  if (rs > 0 && !(max_ctas > 0 && ticket) && ready == nullptr && !(tf32_operands && sizeof(T) == 4)) {
    switch (rs) {
      case 2: return right_gather_seg_r<T, 2>(X, JA, ka, lam, J, k, n, m_rows, accumulate, M, msq_partial, xsq_partial, st,
                                              row_off);
      case 4: return right_gather_seg_r<T, 4>(X, JA, ka, lam, J, k, n, m_rows, accumulate, M, msq_partial, xsq_partial, st,
                                              row_off);
      case 6: return right_gather_seg_r<T, 6>(X, JA, ka, lam, J, k, n, m_rows, accumulate, M, msq_partial, xsq_partial, st,
                                              row_off);
      default: return right_gather_seg_r<T, 8>(X, JA, ka, lam, J, k, n, m_rows, accumulate, M, msq_partial, xsq_partial, st,
                                              row_off);
    }
  }
  const int r = right_gather_rows(n, sizeof(T), k);
  APX_REQUIRE((size_t)n * sizeof(T) + (size_t)(k + 8) * sizeof(int) <= 227 * 1024,
              "n=%d too large for the right gather row block", n);
#define APX_RG(RV) \
  return right_gather_r<T, RV>(X, JA, ka, lam, J, k, n, m_rows, accumulate, M, msq_partial, xsq_partial, lam_padded, \
                               max_ctas, ticket, col_chunks, tf32_operands, ready, x_early, row_off, st, skip_if)
  switch (r) {
    case 1: APX_RG(1);
    case 2: APX_RG(2);
    case 3: APX_RG(3);
    case 4: APX_RG(4);
    case 5: APX_RG(5);
    case 6: APX_RG(6);
    case 7: APX_RG(7);
    default: APX_RG(8);
  }
#undef APX_RG
}

// Output columns [c_lo, c_hi) of X . Bhat for all m_rows rows of X, through the segmented gather
// (any n that is a multiple of 512; c_lo, c_hi multiples of its 32 * CPT-column chunks):
// lam: k x (c_hi - c_lo) column-aligned table of those columns; M: m_rows x (c_hi - c_lo).
template <typename T>
int launch_cycle_right_gather_cols(const T* X, const T* lam, const int* J, int k, int n, int m_rows, int c_lo,
                                   int c_hi, T* M, cudaStream_t st) {
  constexpr int CW = 32 * seg_cpt<T>();
  APX_REQUIRE(n % kSegThreads == 0 && c_lo % CW == 0 && c_hi % CW == 0 && 0 <= c_lo && c_lo < c_hi && c_hi <= n,
              "column-block gather needs n %% %d == 0 and %d-aligned blocks, got n=%d [%d, %d)", kSegThreads, CW, n,
              c_lo, c_hi);
  const int w = c_hi - c_lo;
  switch (seg_rows(sizeof(T))) {
    case 2: return right_gather_seg_r<T, 2>(X, nullptr, 0, lam, J, k, n, m_rows, 0, M, nullptr, nullptr, st, 0, c_lo, c_hi, w, w);
    case 4: return right_gather_seg_r<T, 4>(X, nullptr, 0, lam, J, k, n, m_rows, 0, M, nullptr, nullptr, st, 0, c_lo, c_hi, w, w);
    case 6: return right_gather_seg_r<T, 6>(X, nullptr, 0, lam, J, k, n, m_rows, 0, M, nullptr, nullptr, st, 0, c_lo, c_hi, w, w);
    default: return right_gather_seg_r<T, 8>(X, nullptr, 0, lam, J, k, n, m_rows, 0, M, nullptr, nullptr, st, 0, c_lo, c_hi, w, w);
  }
}

template <typename T>
int launch_sumsq(const T* x, size_t cnt, double* partial, int* nparts, cudaStream_t st) {
  const int blocks = kNumSMs * 4;
  sumsq_partial_kernel<T><<<blocks, 256, 0, st>>>(x, cnt, partial);
  APX_LAUNCH_CHECK();
  *nparts = blocks;
  return OK;
}

int launch_sum_vector(const double* v, int n, double* out, cudaStream_t st) {
  sum_vector_kernel<<<1, 1024, 0, st>>>(v, n, out);
  APX_LAUNCH_CHECK();
  return OK;
}

#define APX_INST(T)                                                                                            \
  template int launch_cycle_energies<T>(const T*, int, double*, double*, double*, double*, cudaStream_t, int, int, int);     \
  template int launch_cycle_extract<T>(const T*, int, const int*, int, T*, cudaStream_t, bool);                   \
  template int launch_cycle_materialize<T>(const T*, const int*, int, int, T*, cudaStream_t);                 \
  template int launch_cycle_left_gather<T>(const T*, const T*, const int*, int, int, int, T*, cudaStream_t);  \
  template int launch_cycle_right_gather<T>(const T*, const int*, int, const T*, const int*, int, int, int, int, T*, \
                                            double*, double*, cudaStream_t, bool, int, int*, int, int, int*, bool, int, const int*); \
  template int launch_sumsq<T>(const T*, size_t, double*, int*, cudaStream_t);                               \
  template int launch_cycle_energies_rows<T>(const T*, int, int, int, double*, double*, cudaStream_t);       \
  template int launch_cycle_extract_rows<T>(const T*, int, int, int, const int*, int, T*, cudaStream_t);      \
  template int launch_cycle_left_gather_rows<T>(const T*, const T*, const int*, int, int, int, int, T*, cudaStream_t); \
  template int launch_cycle_right_gather_cols<T>(const T*, const T*, const int*, int, int, int, int, int, T*, cudaStream_t);
APX_INST(float)
APX_INST(double)

}  // namespace apx
