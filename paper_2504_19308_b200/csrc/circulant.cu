// Circulant decomposition A = sum_k R_k D^k and its truncated first-order product
// (reference circulant.py), plus the unitary DFT and cycle-layout primitives of core.py.
//
//   decompose   S[t][j] = (1/n) sum_i A[(i+j)%n][i] w^{-ti}   (circulant.py:73-91: W applied to
//               the right cycle layout, / sqrt(n)); magnitudes[t] = ||S[t,:]||_2
//   left        term1[:, c] = W* sum_t diag(L_t) C^t (W B[:, c]),  L_t = fft(S_A[t])  (:136-147)
//   right       term2[r, :] = conj(W* sum_t C^{-t} diag(conj L_t) W conj(dA[r, :]))     (:150-161)
//               with dA[r, c] = A[r, c] - sum_t S_A[t][(r-c)%n] w^{tc} formed on the fly (:116-127,197)
// Every length-n transform runs in shared memory (fft.cuh); term1 is column-local and term2
// row-local, so each CTA owns one column (left) or one row (right) end to end.
#include "../../include/apx.h"
#include "common.cuh"
#include "fft.cuh"
#include "fft16.cuh"
#include <type_traits>
#include "kernels.cuh"

namespace apx {

__global__ void roots_kernel(double2* roots, int n) {
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
    double s, c;
    sincospi(2.0 * (double)k / (double)n, &s, &c);
    roots[k] = make_double2(c, -s);  // exp(-2 pi i k / n)
  }
}

void launch_roots(double2* roots, int n, cudaStream_t st) {
  roots_kernel<<<(unsigned)std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, 256), 1024)), 256, 0, st>>>(roots, n);
}

template <typename T>
__device__ __forceinline__ double2 ld_c(const T* p, size_t i);
template <>
__device__ __forceinline__ double2 ld_c<double>(const double* p, size_t i) {
  return make_double2(__ldg(p + i), 0.0);
}
template <>
__device__ __forceinline__ double2 ld_c<double2>(const double2* p, size_t i) {
  return __ldg(p + i);
}

// (t * c) mod n for 0 <= t, c < n: a mask for power-of-two n, 32-bit arithmetic while n^2 < 2^32
__device__ __forceinline__ int mulmod_n(int t, int c, int n) {
  if ((n & (n - 1)) == 0) return (t * c) & (n - 1);
  if (n < 65536) return (int)(((unsigned)t * (unsigned)c) % (unsigned)n);
  return (int)(((long long)t * c) % n);
}

static size_t fft_smem_bytes(int n, int buffers) {
  return (size_t)(buffers + (is_pow2(n) ? 0 : 1)) * n * sizeof(double2);
}

// ---------------------------------------------------------------------------------------------
// skew: X[j][i] = A[(i+j)%n][i] (row j = cycle j in the right layout, core.py:113). The diagonal
// read of the cycle layout touches one element per row of A -- one DRAM sector per element -- so
// it is done once, tile by tile: a 32 x 32 tile of X needs a 63-row parallelogram of A whose
// rows are contiguous column segments (coalesced reads), staged in shared memory and written
// back as contiguous rows of X.
// ---------------------------------------------------------------------------------------------
// [j_lo, j_hi): the cycle rows to produce (a rank's share in the sharded product); X holds them
// from row j_lo on.
template <typename T>
__global__ void __launch_bounds__(256) circ_skew_kernel(const T* __restrict__ A, int n, T* __restrict__ X,
                                                        int j_lo = 0, int j_hi = -1) {
  __shared__ T tile[32][33];
  if (j_hi < 0) j_hi = n;
  const int i0 = blockIdx.x * 32, j0 = j_lo + blockIdx.y * 32;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int d = warp; d < 63; d += 8) {  // source row r = i0 + j0 + d, column i0 + lane, j = d - lane
    const int jj = d - lane;
    if (jj < 0 || jj >= 32 || i0 + lane >= n || j0 + jj >= j_hi) continue;
    int r = i0 + j0 + d;
    r %= n;
    tile[jj][lane] = A[(size_t)r * n + i0 + lane];
  }
  __syncthreads();
  for (int jj = warp; jj < 32; jj += 8)
    if (j0 + jj < j_hi && i0 + lane < n) X[(size_t)(j0 + jj - j_lo) * n + i0 + lane] = tile[jj][lane];
}

// ---------------------------------------------------------------------------------------------
// decompose: CTA handles cycles [j0, j0 + cpc); per cycle: the (contiguous) row j of the skewed
// copy, FFT, scale, store row j of S^T, and fold |S[t][j]|^2 into a per-CTA partial of the
// magnitudes.
// ---------------------------------------------------------------------------------------------
template <typename T>
__global__ void __launch_bounds__(512) circ_decompose_rows_kernel(const T* __restrict__ X, int n, int cpc,
                                                                  const double2* __restrict__ roots,
                                                                  double2* __restrict__ St,
                                                                  double* __restrict__ mag2_part, int b_off = 0,
                                                                  int j_base = 0, int direct = 0) {
  // b_off / j_base (sharded product): this launch is CTA-blocks [b_off, ...) of the full grid, and
  // X, St hold rows from cycle j_base on; the partials land in the full-grid slots (the caller
  // sums the zero-padded slot arrays over ranks, so mag_finalize sees the single-device layout)
  // direct (real operands, n <= 4096): X is the operand A itself and the cycle rows are read off
  // its diagonals -- no skewed copy (whose parallelogram tiles read A twice and wrote X once)
  if (!direct) X -= (size_t)j_base * n;
  St -= (size_t)j_base * n;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double2* x = reinterpret_cast<double2*>(smem_raw);
  double2* scratch = x + n;
  double* m2 = reinterpret_cast<double*>(scratch + (is_pow2(n) ? 0 : n));
  for (int t = threadIdx.x; t < n; t += blockDim.x) m2[t] = 0.0;
  const double inv_n = 1.0 / n;
  const int blk = blockIdx.x + b_off;
  const int j0 = blk * cpc, j1 = min(n, j0 + cpc);
  if constexpr (std::is_same<T, double>::value) {
    // real rows in pairs: x_j + i x_{j+1} through ONE transform Z, split as
    // F_j[t] = (Z[t] + conj Z[-t]) / 2, F_{j+1}[t] = (Z[t] - conj Z[-t]) / 2i; the next pair's
    // loads are in flight (registers) while the current pair is transformed
    if (n <= 8 * 512) {
      double nx0[8], nx1[8];
      // direct: the thread's unit u is ROW r of A, which holds x_j[(r - j) mod n] and, one column
      // to the left, x_{j+1}[(r - j - 1) mod n] (usually one 32-byte sector for both)
      auto load_pair = [&](int j) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int i = threadIdx.x + u * blockDim.x;
          if (direct) {
            int c = i - j;
            if (c < 0) c += n;
            const int c1 = c == 0 ? n - 1 : c - 1;
            nx0[u] = (i < n && j < j1) ? __ldg(X + (size_t)i * n + c) : 0.0;
            nx1[u] = (i < n && j + 1 < j1) ? __ldg(X + (size_t)i * n + c1) : 0.0;
          } else {
            nx0[u] = (i < n && j < j1) ? __ldg(X + (size_t)j * n + i) : 0.0;
            nx1[u] = (i < n && j + 1 < j1) ? __ldg(X + (size_t)(j + 1) * n + i) : 0.0;
          }
        }
      };
      load_pair(j0);
      for (int j = j0; j < j1; j += 2) {
        if (direct) {
          double* xd = reinterpret_cast<double*>(x);
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const int r = threadIdx.x + u * blockDim.x;
            if (r < n) {
              int c = r - j;
              if (c < 0) c += n;
              const int c1 = c == 0 ? n - 1 : c - 1;
              xd[2 * fsw(c, n)] = nx0[u];
              xd[2 * fsw(c1, n) + 1] = nx1[u];
            }
          }
        } else {
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const int i = threadIdx.x + u * blockDim.x;
            if (i < n) x[fsw(i, n)] = make_double2(nx0[u], nx1[u]);
          }
        }
        __syncthreads();
        if (j + 2 < j1) load_pair(j + 2);
        fft_block(x, scratch, n, roots, false);
        const bool two = j + 1 < j1;
        const double h = 0.5 * inv_n;
        for (int t = threadIdx.x; t < n; t += blockDim.x) {
          const double2 z = x[fsw(t, n)], zm = x[fsw(t == 0 ? 0 : n - t, n)];
          const double2 v0 = make_double2(h * (z.x + zm.x), h * (z.y - zm.y));
          St[(size_t)j * n + t] = v0;
          double a = fma(v0.x, v0.x, fma(v0.y, v0.y, m2[t]));
          if (two) {
            const double2 v1 = make_double2(h * (z.y + zm.y), h * (zm.x - z.x));
            St[(size_t)(j + 1) * n + t] = v1;
            a = fma(v1.x, v1.x, fma(v1.y, v1.y, a));
          }
          m2[t] = a;
        }
        __syncthreads();
      }
      for (int t = threadIdx.x; t < n; t += blockDim.x) mag2_part[(size_t)blk * n + t] = m2[t];
      return;
    }
  }
  for (int j = j0; j < j1; ++j) {
    for (int i = threadIdx.x; i < n; i += blockDim.x) x[fsw(i, n)] = ld_c<T>(X, (size_t)j * n + i);
    __syncthreads();
    fft_block(x, scratch, n, roots, false);
    for (int t = threadIdx.x; t < n; t += blockDim.x) {
      const double2 v = cscale(x[fsw(t, n)], inv_n);
      St[(size_t)j * n + t] = v;
      m2[t] = fma(v.x, v.x, fma(v.y, v.y, m2[t]));
    }
    __syncthreads();
  }
  for (int t = threadIdx.x; t < n; t += blockDim.x) mag2_part[(size_t)blk * n + t] = m2[t];
}

// The decomposition for real operands at n = 4096 on the radix-16 transform: the two halves of
// the CTA take alternate cycle pairs of the CTA's range [j0, j1). A pair (x_j, x_{j+1}) is staged
// from A's diagonals exactly as the direct path of circ_decompose_rows_kernel (thread unit = row
// i of A: x_j[(i - j) mod n] and x_{j+1}[(i - j - 1) mod n]), read back as Z[t + 256 m] into the
// transform's registers, transformed, and split F_j = (Z[t] + conj Z[-t]) / 2n, F_{j+1} =
// (Z[t] - conj Z[-t]) / 2in with the conjugate partners read from the plain-order copy; each thread
// keeps the magnitude partials of its 16 frequencies t + 256 m in registers, and the two halves'
// partials are added (half 0 + half 1) into the CTA's slot of mag2_part. Same CTA grid and slots as
// circ_decompose_rows_kernel (b_off / j_base for the sharded product).
__global__ void __launch_bounds__(512) circ_decompose_r16_kernel(const double* __restrict__ A, int cpc,
                                                                 const double2* __restrict__ roots,
                                                                 double2* __restrict__ St,
                                                                 double* __restrict__ mag2_part, int b_off,
                                                                 int j_base) {
  constexpr int n = 4096;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int tid = threadIdx.x, half = tid >> 8, t = tid & 255, bar = 1 + half;
  double2* buf = reinterpret_cast<double2*>(smem_raw) + (size_t)half * kFFT16Buf;
  double* bufd = reinterpret_cast<double*>(buf);
  St -= (size_t)j_base * n;
  const int blk = blockIdx.x + b_off;
  const int j0 = blk * cpc, j1 = min(n, j0 + cpc);
  const double h = 0.5 / n;
  double m2[16];
#pragma unroll
  for (int m = 0; m < 16; ++m) m2[m] = 0.0;
  for (int j = j0 + 2 * half; j < j1; j += 4) {
    {
      // all 32 loads in flight before the first store (a prefetch of the next pair spilled)
      double xr[16], xi[16];
#pragma unroll
      for (int m = 0; m < 16; ++m) {
        const int i = t + 256 * m;
        const int c = (i - j) & (n - 1), c1 = (c - 1) & (n - 1);
        xr[m] = __ldg(A + (size_t)i * n + c);
        xi[m] = j + 1 < j1 ? __ldg(A + (size_t)i * n + c1) : 0.0;
      }
#pragma unroll
      for (int m = 0; m < 16; ++m) {
        const int i = t + 256 * m;
        const int c = (i - j) & (n - 1), c1 = (c - 1) & (n - 1);
        bufd[2 * c] = xr[m];
        bufd[2 * c1 + 1] = xi[m];
      }
    }
    named_bar(bar, 256);
    double2 v[16];
#pragma unroll
    for (int m = 0; m < 16; ++m) v[m] = buf[t + 256 * m];
    named_bar(bar, 256);  // every read of the staged pair done before the transform writes
    fft4096_r16<false>(v, buf, roots, t, bar);
#pragma unroll
    for (int m = 0; m < 16; ++m) buf[t + 256 * m] = v[m];
    named_bar(bar, 256);
    const bool two = j + 1 < j1;
#pragma unroll
    for (int m = 0; m < 16; ++m) {
      const int tau = t + 256 * m;
      const double2 z = v[m], zm = buf[(n - tau) & (n - 1)];
      const double2 f0 = make_double2(h * (z.x + zm.x), h * (z.y - zm.y));
      St[(size_t)j * n + tau] = f0;
      double a = fma(f0.x, f0.x, fma(f0.y, f0.y, m2[m]));
      if (two) {
        const double2 f1 = make_double2(h * (z.y + zm.y), h * (zm.x - z.x));
        St[(size_t)(j + 1) * n + tau] = f1;
        a = fma(f1.x, f1.x, fma(f1.y, f1.y, a));
      }
      m2[m] = a;
    }
    named_bar(bar, 256);  // the conjugate-partner reads done before the next pair is staged
  }
  __syncthreads();
  double* other = reinterpret_cast<double*>(smem_raw);  // half 1's partials, then half 0 adds
  if (half == 1) {
#pragma unroll
    for (int m = 0; m < 16; ++m) other[t + 256 * m] = m2[m];
  }
  __syncthreads();
  if (half == 0) {
#pragma unroll
    for (int m = 0; m < 16; ++m) mag2_part[(size_t)blk * n + t + 256 * m] = m2[m] + other[t + 256 * m];
  }
}

// decomposition launch shared by the single-device and the sharded plans: the radix-16 kernel for
// real operands at n = 4096 (APX_CIRC_R16=0 selects circ_decompose_rows_kernel)
template <typename T>
static int launch_decompose_rows(const T* X, int n, int cpc, const double2* roots, double2* St, double* mag2_part,
                                 int blocks, int b_off, int j_base, int direct, cudaStream_t st) {
  static const bool r16_off = getenv("APX_CIRC_R16") != nullptr && atoi(getenv("APX_CIRC_R16")) == 0;
  if (std::is_same<T, double>::value && n == 4096 && direct && !r16_off) {
    const size_t smem = (size_t)2 * kFFT16Buf * sizeof(double2);
    APX_CUDA(cudaFuncSetAttribute(circ_decompose_r16_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    circ_decompose_r16_kernel<<<blocks, 512, smem, st>>>(reinterpret_cast<const double*>(X), cpc, roots, St,
                                                          mag2_part, b_off, j_base);
    APX_LAUNCH_CHECK();
    return OK;
  }
  const size_t smem = fft_smem_bytes(n, 1) + (size_t)n * sizeof(double);
  auto fn = circ_decompose_rows_kernel<T>;
  APX_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  fn<<<blocks, 512, smem, st>>>(X, n, cpc, roots, St, mag2_part, b_off, j_base, direct);
  APX_LAUNCH_CHECK();
  return OK;
}

// mag[t] = sqrt(sum_p part[p][t]): a CTA covers 32 columns with 8 slices of the parts (slice s:
// parts s, s+8, ...), combined in slice order -- a fixed order, 8x the loads in flight of a
// column-per-thread loop over all parts (which was latency-bound: 33 us at n = 4096)
__global__ void __launch_bounds__(256) mag_finalize_kernel(const double* __restrict__ part, int parts, int n,
                                                           double* __restrict__ mag) {
  __shared__ double acc_s[8][33];
  const int jx = threadIdx.x & 31, sl = threadIdx.x >> 5;
  const int t = blockIdx.x * 32 + jx;
  double a = 0.0;
  if (t < n)
    for (int q = sl; q < parts; q += 8) a += part[(size_t)q * n + t];
  acc_s[sl][jx] = a;
  __syncthreads();
  if (sl == 0 && t < n) {
    double e = 0.0;
#pragma unroll
    for (int q = 0; q < 8; ++q) e += acc_s[q][jx];
    mag[t] = sqrt(e);
  }
}

// Selected spectrum rows from S^T: Ssel[q] = S[sel[q]], L[q] = fft(S[sel[q]]) (unnormalised, :145)
// rows_in (sharded product): S is already the k x n table of selected rows (row q contiguous).
__global__ void __launch_bounds__(512) circ_spectra_kernel(const double2* __restrict__ S, int n,
                                                           const int* __restrict__ sel,
                                                           const double2* __restrict__ roots,
                                                           double2* __restrict__ Ssel, double2* __restrict__ L,
                                                           int rows_in, double scale) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double2* x = reinterpret_cast<double2*>(smem_raw);
  double2* scratch = x + n;
  const int q = blockIdx.x;
  const int t = sel[q];
  // row t of S = column t of S^T (strided; 8 loads per thread in flight)
  for (int i0 = threadIdx.x; i0 < n; i0 += 8 * blockDim.x) {
    double2 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int i = i0 + u * blockDim.x;
      v[u] = i < n ? __ldg(rows_in ? S + (size_t)q * n + i : S + (size_t)i * n + t) : make_double2(0.0, 0.0);
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int i = i0 + u * blockDim.x;
      if (i < n) {
        x[fsw(i, n)] = v[u];
        if (Ssel) Ssel[(size_t)q * n + i] = v[u];
      }
    }
  }
  __syncthreads();
  fft_block(x, scratch, n, roots, false);
  for (int i = threadIdx.x; i < n; i += blockDim.x) L[(size_t)q * n + i] = cscale(x[fsw(i, n)], scale);
}

// ---------------------------------------------------------------------------------------------
// term1, one column per CTA: FB = W B[:,c]; acc[p] = sum_t L_t[p] FB[(p - t) % n]; M[:,c] = W* acc
// ---------------------------------------------------------------------------------------------
template <typename T>
__global__ void __launch_bounds__(512) circ_left_kernel(const T* __restrict__ B, int n, const double2* __restrict__ L,
                                                        const int* __restrict__ sel, int k,
                                                        const double2* __restrict__ roots, double2* __restrict__ M) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double2* x = reinterpret_cast<double2*>(smem_raw);
  double2* y = x + n;
  double2* scratch = y + n;
  int* s_sel = reinterpret_cast<int*>(scratch + (is_pow2(n) ? 0 : n));
  for (int q = threadIdx.x; q < k; q += blockDim.x) s_sel[q] = sel[q];
  sel = s_sel;
  const int c = blockIdx.x;
  const double rs = rsqrt((double)n);
  // column c of B: strided, so 8 loads per thread are issued before the first store
  for (int p0 = threadIdx.x; p0 < n; p0 += 8 * blockDim.x) {
    double2 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int p = p0 + u * blockDim.x;
      v[u] = p < n ? ld_c<T>(B, (size_t)p * n + c) : make_double2(0.0, 0.0);
    }
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (p0 + u * blockDim.x < n) x[fsw(p0 + u * blockDim.x, n)] = v[u];
  }
  __syncthreads();
  fft_block(x, scratch, n, roots, false);
  for (int p = threadIdx.x; p < n; p += blockDim.x) {
    double2 acc = make_double2(0.0, 0.0), acc2 = make_double2(0.0, 0.0);
    int q = 0;
    for (; q + 4 <= k; q += 4) {
      double2 lv[4], xv[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        int src = p - sel[q + u];
        if (src < 0) src += n;
        lv[u] = __ldg(L + (size_t)(q + u) * n + p);
        xv[u] = x[fsw(src, n)];
      }
#pragma unroll
      for (int u = 0; u < 4; u += 2) {
        acc = cmac(acc, lv[u], xv[u]);
        acc2 = cmac(acc2, lv[u + 1], xv[u + 1]);
      }
    }
    for (; q < k; ++q) {
      int src = p - sel[q];
      if (src < 0) src += n;
      acc = cmac(acc, __ldg(L + (size_t)q * n + p), x[fsw(src, n)]);
    }
    y[fsw(p, n)] = cadd(acc, acc2);
  }
  __syncthreads();
  fft_block(y, scratch, n, roots, true);
  for (int p = threadIdx.x; p < n; p += blockDim.x) M[(size_t)p * n + c] = y[fsw(p, n)];
}

// ---------------------------------------------------------------------------------------------
// Two columns (left) / two rows (right) per CTA, n <= kPP * 512: every L_t load of the weighted
// gather-sum serves both transforms, neighbouring B columns share DRAM sectors, and the two
// rows' Ahat terms read adjacent S_t entries. The gather-sum results stay in registers (kPP
// complex per thread per transform) until every thread has read its inputs; the input buffers
// are then reused for the inverse transforms, so two transforms fit the shared memory of one.
// ---------------------------------------------------------------------------------------------
constexpr int kPP = 8;

template <typename T>
// col_base / col_end / ldm (sharded product): the CTA pairs cover columns [col_base, col_end) of
// term1 (col_base even: the same pairs as the full grid), written to an n x (col_end - col_base)
// block with leading dimension ldm.
__global__ void __launch_bounds__(512) circ_left2_kernel(const T* __restrict__ B, int n, const double2* __restrict__ L,
                                                         const int* __restrict__ sel, int k,
                                                         const double2* __restrict__ roots, double2* __restrict__ M,
                                                         int col_base = 0, int col_end = -1, int64_t ldm = -1,
                                                         int stage_l = 0) {
  if (col_end < 0) col_end = n;
  if (ldm < 0) ldm = n;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double2* x0 = reinterpret_cast<double2*>(smem_raw);
  double2* x1 = x0 + n;
  double2* scratch = x1 + n;
  int* s_sel = reinterpret_cast<int*>(scratch + (is_pow2(n) ? 0 : n));
  for (int q = threadIdx.x; q < k; q += blockDim.x) s_sel[q] = sel[q];
  // stage_l (n == 2 * kPP/2 * blockDim): the L_t rows reach shared memory by bulk async copies, in
  // half rows (positions i < kPP/2 of every thread lie in the first half), double-buffered and
  // started before the transform, so the gather's L reads are conflict-free shared loads instead
  // of L2 round trips (its largest stall). Stage s = (term s / 2, half s % 2) uses buffer s % 2.
  const int half = n / 2;
  double2* Lb = reinterpret_cast<double2*>(
      (reinterpret_cast<uintptr_t>(s_sel + k) + 127) & ~static_cast<uintptr_t>(127));
  uint64_t* lbar = reinterpret_cast<uint64_t*>(Lb + 2 * half);
  const bool stage = stage_l && k > 0;
  auto issue = [&](int st) {
    const uint32_t bytes = (uint32_t)(half * sizeof(double2));
    const uint32_t bar = (uint32_t)__cvta_generic_to_shared(&lbar[st & 1]);
    const uint32_t dst = (uint32_t)__cvta_generic_to_shared(Lb + (st & 1) * half);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                 "l"(L + (size_t)(st >> 1) * n + (st & 1) * half), "r"(bytes), "r"(bar)
                 : "memory");
  };
  if (stage && threadIdx.x == 0) {
    for (int b = 0; b < 2; ++b)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&lbar[b])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    issue(0);
    if (2 * k > 1) issue(1);
  }
  const int c0 = col_base + 2 * blockIdx.x;
  const bool two = c0 + 1 < col_end;
  const double rs = rsqrt((double)n);
  // real B: the two columns travel as one complex sequence b0 + i b1 through ONE forward
  // transform Z, split afterwards as FB0[p] = (Z[p] + conj Z[-p]) / 2, FB1[p] = (Z[p] - conj Z[-p]) / 2i
  constexpr bool kPack = std::is_same<T, double>::value;
  // the two real columns of a row are one 16-byte load (c0 even, n even)
  const bool pair_ld = kPack && two && (n & 1) == 0;
  for (int p0 = threadIdx.x; p0 < n; p0 += 4 * blockDim.x) {
    double2 v0[4], v1[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int p = p0 + u * blockDim.x;
      if (pair_ld) {
        const double2 b2 = p < n ? __ldg(reinterpret_cast<const double2*>(B + (size_t)p * n + c0))
                                 : make_double2(0.0, 0.0);
        v0[u] = make_double2(b2.x, 0.0);
        v1[u] = make_double2(b2.y, 0.0);
      } else {
        v0[u] = p < n ? ld_c<T>(B, (size_t)p * n + c0) : make_double2(0.0, 0.0);
        v1[u] = (p < n && two) ? ld_c<T>(B, (size_t)p * n + c0 + 1) : make_double2(0.0, 0.0);
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int p = p0 + u * blockDim.x;
      if (p < n) {
        if constexpr (kPack) {
          x0[fsw(p, n)] = make_double2(v0[u].x, v1[u].x);
        } else {
          x0[fsw(p, n)] = v0[u];
          x1[fsw(p, n)] = v1[u];
        }
      }
    }
  }
  __syncthreads();
  // forward transforms end in plain order (fft_linear_ok): the shifted gathers below read
  // unaligned runs, which the swizzle split over bank groups
  const bool lin = fft_linear_ok(n);
  auto ix = [&](int i) { return lin ? i : fsw(i, n); };
  fft_block(x0, scratch, n, roots, false, true);
  if constexpr (kPack) {
    double2 f0[kPP];  // FB1 goes straight to x1; FB0 waits in registers until every Z read is done
#pragma unroll
    for (int i = 0; i < kPP; ++i) {
      const int p = threadIdx.x + i * blockDim.x;
      if (p < n) {
        const double2 z = x0[ix(p)], zm = x0[ix(p == 0 ? 0 : n - p)];
        f0[i] = make_double2(0.5 * (z.x + zm.x), 0.5 * (z.y - zm.y));
        x1[ix(p)] = make_double2(0.5 * (z.y + zm.y), 0.5 * (zm.x - z.x));
      }
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < kPP; ++i) {
      const int p = threadIdx.x + i * blockDim.x;
      if (p < n) x0[ix(p)] = f0[i];
    }
    __syncthreads();
  } else {
    fft_block(x1, scratch, n, roots, false, true);
  }
  // term-major: the kPP positions' L_t loads (L2) of one term are independent, so all are in
  // flight together (position-major, each thread waited one L2 latency per term and position);
  // every position still sums its terms in ascending order
  double2 y0[kPP], y1[kPP];
#pragma unroll
  for (int i = 0; i < kPP; ++i) y0[i] = y1[i] = make_double2(0.0, 0.0);
  if (stage) {
    auto half_terms = [&](const double2* Lh, int sq, auto ibase) {
      constexpr int I0 = decltype(ibase)::value;
#pragma unroll
      for (int i = I0; i < I0 + kPP / 2; ++i) {
        const int p = threadIdx.x + i * blockDim.x;
        int src = p - sq;
        if (src < 0) src += n;
        APX_DCHECK(src >= 0 && src < n && p - I0 * (int)blockDim.x < half);
        const double2 l = Lh[p - I0 * blockDim.x];
        y0[i] = cmac(y0[i], l, x0[ix(src)]);
        y1[i] = cmac(y1[i], l, x1[ix(src)]);
      }
    };
    for (int st = 0; st < 2 * k; ++st) {
      const int b = st & 1;
      const uint32_t bar = (uint32_t)__cvta_generic_to_shared(&lbar[b]);
      const uint32_t ph = (uint32_t)((st >> 1) & 1);
      asm volatile(
          "{\n.reg .pred p;\nLW_%=:\n"
          "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
          "@!p bra LW_%=;\n}\n" ::"r"(bar),
          "r"(ph)
          : "memory");
      const int sq = s_sel[st >> 1];
      if (b == 0)
        half_terms(Lb, sq, std::integral_constant<int, 0>());
      else
        half_terms(Lb + half, sq, std::integral_constant<int, kPP / 2>());
      __syncthreads();  // buffer b drained
      if (threadIdx.x == 0 && st + 2 < 2 * k) issue(st + 2);
    }
  }
  for (int q = 0; q < k && !stage; ++q) {
    const int sq = s_sel[q];
    const double2* Lq = L + (size_t)q * n;
    double2 l[kPP];
#pragma unroll
    for (int i = 0; i < kPP; ++i) {
      const int p = threadIdx.x + i * blockDim.x;
      l[i] = p < n ? __ldg(Lq + p) : make_double2(0.0, 0.0);
    }
#pragma unroll
    for (int i = 0; i < kPP; ++i) {
      const int p = threadIdx.x + i * blockDim.x;
      if (p < n) {
        int src = p - sq;
        if (src < 0) src += n;
        APX_DCHECK(src >= 0 && src < n && sq >= 0 && sq < n);
        y0[i] = cmac(y0[i], l[i], x0[ix(src)]);
        y1[i] = cmac(y1[i], l[i], x1[ix(src)]);
      }
    }
  }
  __syncthreads();  // every gather read of x0 / x1 is done: reuse them for the inverse transforms
#pragma unroll
  for (int i = 0; i < kPP; ++i) {
    const int p = threadIdx.x + i * blockDim.x;
    if (p < n) {
      x0[fsw(p, n)] = y0[i];
      x1[fsw(p, n)] = y1[i];
    }
  }
  __syncthreads();
  fft_block(x0, scratch, n, roots, true);
  fft_block(x1, scratch, n, roots, true);
  // the two complex outputs of a row are adjacent: one 32-byte store (STG.256) when aligned
  const bool pair_st = two && ((ldm | (c0 - col_base)) & 1) == 0 && ((uintptr_t)M & 31) == 0;
  for (int p = threadIdx.x; p < n; p += blockDim.x) {
    double2* dst = M + (size_t)p * ldm + (c0 - col_base);
    const double2 a = x0[fsw(p, n)], b = x1[fsw(p, n)];
    if (pair_st) {
      asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(dst), "d"(a.x), "d"(a.y), "d"(b.x), "d"(b.y)
                   : "memory");
    } else {
      dst[0] = a;
      if (two) dst[1] = b;
    }
  }
}

// ---------------------------------------------------------------------------------------------
// term1 for n = 4096, real B, two columns per CTA on the radix-16 transform (fft16.cuh):
//   1. the first half of the CTA (256 threads) packs the two real columns as Z = b0 + i b1 and runs
//      one forward fft4096_r16 from the global loads; Z goes to shared memory in plain order;
//   2. all 512 threads gather for positions p = tid + 512 i: with q = p - s_t, P = sum_t L_t[p] Z[q]
//      and N = sum_t L_t[p] conj Z[-q], so FB0 . L = (P + N) / 2 and FB1 . L = (P - N) / 2i -- the
//      split of Z into FB0 and FB1 needs no pass of its own;
//   3. each half runs the inverse transform of one column and writes it from its registers.
// Shared traffic per column ~1.6 MB against ~2.2 MB for circ_left2_kernel (each transform: two
// exchanges instead of bit reversal plus four radix-8 passes). (Four columns per CTA, which would
// halve the L_t traffic, needs 64 accumulator doubles per thread and spilled.)
// ---------------------------------------------------------------------------------------------
// col_base / col_end / ldm (sharded product, as circ_left2_kernel): the CTA pairs cover columns
// [col_base, col_end) (col_base even: the full grid's pairs), written to an n x (col_end - col_base)
// block with leading dimension ldm.
__global__ void __launch_bounds__(512) circ_left2_r16_kernel(const double* __restrict__ B, const double2* __restrict__ L,
                                                             const int* __restrict__ sel, int k,
                                                             const double2* __restrict__ roots, double2* __restrict__ M,
                                                             int col_base, int col_end, int64_t ldm) {
  constexpr int n = 4096;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double2* buf0 = reinterpret_cast<double2*>(smem_raw);
  double2* buf1 = buf0 + kFFT16Buf;
  int* s_sel = reinterpret_cast<int*>(buf1 + kFFT16Buf);
  const int tid = threadIdx.x, half = tid >> 8, t = tid & 255;
  for (int q = tid; q < k; q += blockDim.x) s_sel[q] = sel[q];
  const int c0 = col_base + 2 * blockIdx.x;
  if (half == 0) {
    // columns c0, c0 + 1 of rows t + 256 m: one 16-byte load per row
    double2 v[16];
#pragma unroll
    for (int m = 0; m < 16; ++m) v[m] = __ldg(reinterpret_cast<const double2*>(B + (size_t)(t + 256 * m) * n + c0));
    fft4096_r16<false>(v, buf0, roots, t, 1);
#pragma unroll
    for (int m = 0; m < 16; ++m) buf1[t + 256 * m] = v[m];
  }
  __syncthreads();
  double2 P[kPP], N[kPP];
#pragma unroll
  for (int i = 0; i < kPP; ++i) P[i] = N[i] = make_double2(0.0, 0.0);
  for (int q = 0; q < k; ++q) {
    const int sq = s_sel[q];
    const double2* Lq = L + (size_t)q * n;
    double2 l[kPP];
#pragma unroll
    for (int i = 0; i < kPP; ++i) l[i] = __ldg(Lq + tid + 512 * i);
#pragma unroll
    for (int i = 0; i < kPP; ++i) {
      const int p = tid + 512 * i;
      const int src = (p - sq) & (n - 1), neg = (n - src) & (n - 1);
      P[i] = cmac(P[i], l[i], buf1[src]);
      N[i] = cmacc(N[i], l[i], buf1[neg]);  // l * conj(Z[-q])
    }
  }
  __syncthreads();  // every Z read done: the buffers take the two columns' gather results
#pragma unroll
  for (int i = 0; i < kPP; ++i) {
    const int p = tid + 512 * i;
    // FB0 . L = (P + N) / 2 -> column c0; FB1 . L = (P - N) / 2i -> column c0 + 1
    buf0[p] = make_double2(0.5 * (P[i].x + N[i].x), 0.5 * (P[i].y + N[i].y));
    buf1[p] = make_double2(0.5 * (P[i].y - N[i].y), -0.5 * (P[i].x - N[i].x));
  }
  __syncthreads();
  double2* xb = half ? buf1 : buf0;
  double2 v[16];
#pragma unroll
  for (int m = 0; m < 16; ++m) v[m] = xb[t + 256 * m];
  fft4096_r16<true>(v, xb, roots, t, 1 + half);
  // the two columns leave through shared memory as (row, col pair) = 32 contiguous bytes, one
  // st.global.v4.f64 per row (a 16-byte store per column and row -- 32 scattered sectors per warp
  // instruction -- held the kernel in LSU throttle and store drain)
  __syncthreads();  // both halves' transforms done with buf0 / buf1
  double2* o = buf0;  // [n][2] across buf0 and buf1 (contiguous, 2 * kFFT16Buf >= 2n)
#pragma unroll
  for (int m = 0; m < 16; ++m) o[2 * (t + 256 * m) + half] = v[m];
  __syncthreads();
  const bool two = c0 + 1 < col_end;
  const bool pair_st = two && ((ldm | (c0 - col_base)) & 1) == 0 && ((uintptr_t)M & 31) == 0;
#pragma unroll
  for (int i = 0; i < kPP; ++i) {
    const int p = tid + 512 * i;
    const double2 a = o[2 * p], b = o[2 * p + 1];
    double2* dst = M + (size_t)p * ldm + (c0 - col_base);
    if (pair_st) {
      asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(dst), "d"(a.x), "d"(a.y), "d"(b.x), "d"(b.y)
                   : "memory");
    } else {
      dst[0] = a;
      if (two) dst[1] = b;
    }
  }
}

// term2 for n = 4096 on the radix-16 transform, two rows per CTA, from the precomputed conj(dA)
// rows (big_dA_win_kernel): each half transforms one row from its global loads, both rows go to
// shared memory in plain order, all 512 threads gather (y += x[(p + s) mod n] conj L_s[(p + s) mod n]
// for both rows, one L load per pair), each half inverse-transforms one row and adds conj of it onto
// M's row straight from its registers (coalesced over t), with one ||M||^2 partial per CTA.
__global__ void __launch_bounds__(512) circ_right2_r16_kernel(const double2* __restrict__ Xpre,
                                                              const double2* __restrict__ LB,
                                                              const int* __restrict__ selB, int kb,
                                                              const double2* __restrict__ roots,
                                                              double2* __restrict__ M, double* __restrict__ msq_part,
                                                              int row_base, int row_end) {
  // row_base / row_end (sharded product, as circ_right2_kernel): the CTA pairs cover rows
  // [row_base, row_end) of term2; M and Xpre hold them from row row_base on
  constexpr int n = 4096;
  M -= (size_t)row_base * n;
  Xpre -= (size_t)row_base * n;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double2* buf0 = reinterpret_cast<double2*>(smem_raw);
  double2* buf1 = buf0 + kFFT16Buf;
  int* sB = reinterpret_cast<int*>(buf1 + kFFT16Buf);
  __shared__ double red[32];
  const int tid = threadIdx.x, half = tid >> 8, t = tid & 255;
  for (int q = tid; q < kb; q += blockDim.x) sB[q] = selB[q];
  const int row = row_base + 2 * blockIdx.x + half;
  const bool live = row < row_end;  // an odd row count leaves the last CTA's second row empty
  double2* xb = half ? buf1 : buf0;
  // the epilogue's read-modify-write of M (term1, DRAM-resident by now): pull the row toward L2
  if (t == 0 && live && ((uintptr_t)(M + (size_t)row * n) & 15) == 0)
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(M + (size_t)row * n),
                 "r"((unsigned)(n * sizeof(double2)))
                 : "memory");
  double2 v[16];
#pragma unroll
  for (int m = 0; m < 16; ++m) v[m] = live ? __ldg(Xpre + (size_t)row * n + t + 256 * m) : make_double2(0.0, 0.0);
  fft4096_r16<false>(v, xb, roots, t, 1 + half);
#pragma unroll
  for (int m = 0; m < 16; ++m) xb[t + 256 * m] = v[m];
  __syncthreads();
  double2 y0[kPP], y1[kPP];
#pragma unroll
  for (int i = 0; i < kPP; ++i) y0[i] = y1[i] = make_double2(0.0, 0.0);
  for (int q = 0; q < kb; ++q) {
    const int sq = sB[q];
    const double2* Lq = LB + (size_t)q * n;
    // two half-batches of L loads in flight (as circ_right2_kernel)
#pragma unroll
    for (int h = 0; h < kPP; h += kPP / 2) {
      double2 l[kPP];
#pragma unroll
      for (int i = h; i < h + kPP / 2; ++i) l[i] = __ldg(Lq + ((tid + 512 * i + sq) & (n - 1)));
#pragma unroll
      for (int i = h; i < h + kPP / 2; ++i) {
        const int src = (tid + 512 * i + sq) & (n - 1);
        y0[i] = cmacc(y0[i], buf0[src], l[i]);
        y1[i] = cmacc(y1[i], buf1[src], l[i]);
      }
    }
  }
  __syncthreads();  // every gather read done
#pragma unroll
  for (int i = 0; i < kPP; ++i) {
    buf0[tid + 512 * i] = y0[i];
    buf1[tid + 512 * i] = y1[i];
  }
  __syncthreads();
#pragma unroll
  for (int m = 0; m < 16; ++m) v[m] = xb[t + 256 * m];
  fft4096_r16<true>(v, xb, roots, t, 1 + half);
  double msq = 0.0;
  double2* mr = M + (size_t)row * n;
  if (live) {
#pragma unroll
    for (int m = 0; m < 16; ++m) {
      const double2 o = mr[t + 256 * m];
      const double2 nv = make_double2(o.x + v[m].x, o.y - v[m].y);  // + conj
      mr[t + 256 * m] = nv;
      msq = fma(nv.x, nv.x, fma(nv.y, nv.y, msq));
    }
  }
  msq = block_sum(msq, red);
  if (tid == 0 && msq_part) msq_part[blockIdx.x] = msq;
}

template <typename T>
__global__ void __launch_bounds__(512) circ_right2_kernel(const T* __restrict__ A, int n,
                                                          const double2* __restrict__ SselA,
                                                          const int* __restrict__ selA, int ka,
                                                          const double2* __restrict__ LB, const int* __restrict__ selB,
                                                          int kb, const double2* __restrict__ roots,
                                                          double2* __restrict__ M,
                                                          const double2* __restrict__ Xpre, int row_base = 0,
                                                          int row_end = -1, int lin_out = 0,
                                                          double* __restrict__ msq_part = nullptr) {
  // [row_base, row_end) (sharded product): the CTA pairs cover these rows of term2; M and Xpre
  // hold them from row row_base on (A is the full operand)
  if (row_end < 0) row_end = n;
  M -= (size_t)row_base * n;
  if (Xpre) Xpre -= (size_t)row_base * n;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double2* x0 = reinterpret_cast<double2*>(smem_raw);
  double2* x1 = x0 + n;
  double2* scratch = x1 + n;
  int* sA = reinterpret_cast<int*>(scratch + (is_pow2(n) ? 0 : n));
  int* sB = sA + ka;
  for (int q = threadIdx.x; q < ka; q += blockDim.x) sA[q] = selA[q];
  for (int q = threadIdx.x; q < kb; q += blockDim.x) sB[q] = selB[q];
  __syncthreads();
  const int r0 = row_base + 2 * blockIdx.x;
  const bool two = r0 + 1 < row_end;
  const double rs = rsqrt((double)n);
  // the epilogue's read-modify-write of M (term1, DRAM-resident by now): pull both rows toward
  // L2 while the transforms run
  if (threadIdx.x < 2 && r0 + (int)threadIdx.x < row_end && ((uintptr_t)M & 15) == 0)
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(M + (size_t)(r0 + threadIdx.x) * n),
                 "r"((unsigned)(n * sizeof(double2)))
                 : "memory");
  if (Xpre != nullptr) {
    // conj(dA) rows precomputed by big_dA_kernel (16-row blocks share every S_t and twiddle load:
    // formed here, two rows per CTA, the S_t reads from L2 were the kernel's largest stall)
    for (int c = threadIdx.x; c < n; c += blockDim.x) {
      x0[fsw(c, n)] = __ldg(Xpre + (size_t)r0 * n + c);
      x1[fsw(c, n)] = two ? __ldg(Xpre + (size_t)(r0 + 1) * n + c) : make_double2(0.0, 0.0);
    }
  } else {
    // Ahat[r][c] = sum_t S_t[(r - c) % n] * w^{t c} at the thread's columns c_i = tid + i * nt:
    // rows r0, r0+1 read S_t[d], S_t[d+1]; the twiddle of c_{i+1} is the one of c_i times
    // w^{t nt}, so each term takes two table loads per thread instead of one per column (the
    // table index t c mod n scatters the lanes over the table: one sector per lane)
    const int nt = blockDim.x;
    double2 h0[kPP], h1[kPP];
#pragma unroll
    for (int i = 0; i < kPP; ++i) h0[i] = h1[i] = make_double2(0.0, 0.0);
    for (int q = 0; q < ka; ++q) {
      double2 w = cconj(__ldg(roots + mulmod_n(sA[q], threadIdx.x, n)));  // exp(+2 pi i t c / n)
      const double2 stp = cconj(__ldg(roots + mulmod_n(sA[q], nt % n, n)));
      const double2* Sq = SselA + (size_t)q * n;
#pragma unroll
      for (int i = 0; i < kPP; ++i) {
        const int c = threadIdx.x + i * nt;
        if (c < n) {
          int d = r0 - c;
          if (d < 0) d += n;
          const int d1 = d + 1 == n ? 0 : d + 1;
          h0[i] = cadd(h0[i], cmul(__ldg(Sq + d), w));
          h1[i] = cadd(h1[i], cmul(__ldg(Sq + d1), w));
          w = cmul(w, stp);
        }
      }
    }
#pragma unroll
    for (int i = 0; i < kPP; ++i) {
      const int c = threadIdx.x + i * nt;
      if (c < n) {
        x0[fsw(c, n)] = cconj(csub(ld_c<T>(A, (size_t)r0 * n + c), h0[i]));
        x1[fsw(c, n)] = two ? cconj(csub(ld_c<T>(A, (size_t)(r0 + 1) * n + c), h1[i])) : make_double2(0.0, 0.0);
      }
    }
  }
  __syncthreads();
  // lin_out: the forward transforms end in plain order (fft_linear_ok) so the shifted gathers below
  // read unaligned runs conflict-free (the XOR swizzle splits them over bank groups)
  const bool lin = lin_out && fft_linear_ok(n);
  fft_block(x0, scratch, n, roots, false, lin);
  fft_block(x1, scratch, n, roots, false, lin);
  // term-major (see circ_left2_kernel): kPP independent L_t loads in flight per term
  double2 y0[kPP], y1[kPP];
#pragma unroll
  for (int i = 0; i < kPP; ++i) y0[i] = y1[i] = make_double2(0.0, 0.0);
  for (int q = 0; q < kb; ++q) {
    const int sq = sB[q];
    const double2* Lq = LB + (size_t)q * n;
    // two half-batches of loads (a full batch of kPP spilled at the 128-register bound)
#pragma unroll
    for (int h = 0; h < kPP; h += kPP / 2) {
      double2 l[kPP];
#pragma unroll
      for (int i = h; i < h + kPP / 2; ++i) {
        const int p = threadIdx.x + i * blockDim.x;
        int src = p + sq;
        if (src >= n) src -= n;
        l[i] = p < n ? __ldg(Lq + src) : make_double2(0.0, 0.0);
      }
#pragma unroll
      for (int i = h; i < h + kPP / 2; ++i) {
        const int p = threadIdx.x + i * blockDim.x;
        if (p < n) {
          int src = p + sq;
          if (src >= n) src -= n;
          APX_DCHECK(src >= 0 && src < n);
          const int sx = lin ? src : fsw(src, n);
          y0[i] = cmacc(y0[i], x0[sx], l[i]);
          y1[i] = cmacc(y1[i], x1[sx], l[i]);
        }
      }
    }
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < kPP; ++i) {
    const int p = threadIdx.x + i * blockDim.x;
    if (p < n) {
      x0[fsw(p, n)] = y0[i];
      x1[fsw(p, n)] = y1[i];
    }
  }
  __syncthreads();
  fft_block(x0, scratch, n, roots, true);
  fft_block(x1, scratch, n, roots, true);
  double msq = 0.0;  // ||M||^2 of the two finished rows (msq_part: one fixed-order partial per CTA)
  for (int c = threadIdx.x; c < n; c += blockDim.x) {
    double2* pm = M + (size_t)r0 * n + c;
    const double2 v0 = cadd(*pm, cconj(x0[fsw(c, n)]));
    *pm = v0;
    msq = fma(v0.x, v0.x, fma(v0.y, v0.y, msq));
    if (two) {
      const double2 v1 = cadd(pm[n], cconj(x1[fsw(c, n)]));
      pm[n] = v1;
      msq = fma(v1.x, v1.x, fma(v1.y, v1.y, msq));
    }
  }
  if (msq_part != nullptr) {
    __shared__ double red[32];
    msq = block_sum(msq, red);
    if (threadIdx.x == 0) msq_part[blockIdx.x] = msq;
  }
}

// ---------------------------------------------------------------------------------------------
// term2, one row per CTA: x = W conj(dA[r,:]); a[p] = sum_t conj(L_t[(p+t)%n]) x[(p+t)%n];
// M[r,:] += conj(W* a). dA's row is formed on the fly from the selected spectra of A.
// ---------------------------------------------------------------------------------------------
template <typename T>
__global__ void __launch_bounds__(512) circ_right_kernel(const T* __restrict__ A, int n,
                                                         const double2* __restrict__ SselA,
                                                         const int* __restrict__ selA, int ka,
                                                         const double2* __restrict__ LB, const int* __restrict__ selB,
                                                         int kb, const double2* __restrict__ roots,
                                                         double2* __restrict__ M) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double2* x = reinterpret_cast<double2*>(smem_raw);
  double2* y = x + n;
  double2* scratch = y + n;
  // the selections, staged once: every term's index math needs them (a global load each time
  // put two dependent loads on every term's critical path)
  int* sA = reinterpret_cast<int*>(scratch + (is_pow2(n) ? 0 : n));
  int* sB = sA + ka;
  for (int q = threadIdx.x; q < ka; q += blockDim.x) sA[q] = selA[q];
  for (int q = threadIdx.x; q < kb; q += blockDim.x) sB[q] = selB[q];
  selA = sA;
  selB = sB;
  __syncthreads();
  const int r = blockIdx.x;
  const double rs = rsqrt((double)n);
  for (int c = threadIdx.x; c < n; c += blockDim.x) {
    // Ahat[r][c] = sum_t S_t[(r - c) % n] * w^{t c}, ascending t (circulant_materialize order)
    double2 ah = make_double2(0.0, 0.0), ah2 = make_double2(0.0, 0.0);
    int d = r - c;
    if (d < 0) d += n;
    // four terms' loads in flight at a time, two accumulators (even / odd q)
    int q = 0;
    for (; q + 4 <= ka; q += 4) {
      double2 w[4], sv[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        w[u] = __ldg(roots + mulmod_n(selA[q + u], c, n));
        sv[u] = __ldg(SselA + (size_t)(q + u) * n + d);
      }
#pragma unroll
      for (int u = 0; u < 4; u += 2) {
        ah = cadd(ah, cmul(sv[u], cconj(w[u])));  // exp(+2 pi i t c / n)
        ah2 = cadd(ah2, cmul(sv[u + 1], cconj(w[u + 1])));
      }
    }
    for (; q < ka; ++q)
      ah = cadd(ah, cmul(__ldg(SselA + (size_t)q * n + d), cconj(__ldg(roots + mulmod_n(selA[q], c, n)))));
    ah = cadd(ah, ah2);
    const double2 a = ld_c<T>(A, (size_t)r * n + c);
    x[fsw(c, n)] = cconj(csub(a, ah));
  }
  __syncthreads();
  fft_block(x, scratch, n, roots, false);
  for (int p = threadIdx.x; p < n; p += blockDim.x) {
    double2 acc = make_double2(0.0, 0.0), acc2 = make_double2(0.0, 0.0);
    int q = 0;
    for (; q + 4 <= kb; q += 4) {
      double2 lv[4], xv[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        int src = p + selB[q + u];
        if (src >= n) src -= n;
        lv[u] = __ldg(LB + (size_t)(q + u) * n + src);
        xv[u] = x[fsw(src, n)];
      }
#pragma unroll
      for (int u = 0; u < 4; u += 2) {
        acc = cmacc(acc, xv[u], lv[u]);
        acc2 = cmacc(acc2, xv[u + 1], lv[u + 1]);
      }
    }
    for (; q < kb; ++q) {
      int src = p + selB[q];
      if (src >= n) src -= n;
      acc = cmacc(acc, x[fsw(src, n)], __ldg(LB + (size_t)q * n + src));
    }
    y[fsw(p, n)] = cadd(acc, acc2);
  }
  __syncthreads();
  fft_block(y, scratch, n, roots, true);
  for (int c = threadIdx.x; c < n; c += blockDim.x) {
    const double2 v = cconj(y[fsw(c, n)]);
    double2* pm = M + (size_t)r * n + c;
    *pm = cadd(*pm, v);
  }
}

// out[r][c] = sum_q Ssel[q][(r-c)%n] * w^{sel[q] c}   (circulant_materialize, :116-127)
__global__ void circ_materialize_kernel(const double2* __restrict__ Ssel, const int* __restrict__ sel, int k, int n,
                                        const double2* __restrict__ roots, double2* __restrict__ out) {
  const size_t total = (size_t)n * n;
  for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < total; e += (size_t)gridDim.x * blockDim.x) {
    const int r = (int)(e / n), c = (int)(e % n);
    int d = r - c;
    if (d < 0) d += n;
    double2 acc = make_double2(0.0, 0.0);
    for (int q = 0; q < k; ++q) acc = cadd(acc, cmul(Ssel[(size_t)q * n + d], cconj(roots[mulmod_n(sel[q], c, n)])));
    out[e] = acc;
  }
}

// circulant_component (:94-108): col[j] = (1/n) sum_i A[(i+j)%n][i] w^{-k i}
template <typename T>
__global__ void circ_component_kernel(const T* __restrict__ A, int n, int kk, const double2* __restrict__ roots,
                                      double2* __restrict__ out) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  double2 acc = make_double2(0.0, 0.0);
  int idx = 0;
  for (int i = 0; i < n; ++i) {
    int r = i + j;
    if (r >= n) r -= n;
    acc = cadd(acc, cmul(ld_c<T>(A, (size_t)r * n + i), __ldg(roots + idx)));
    idx += kk;
    if (idx >= n) idx -= n;
  }
  out[j] = cscale(acc, 1.0 / n);
}

// unitary DFT of `batch` vectors of length n: element i of vector b at in[b*dist + i*stride]
__global__ void __launch_bounds__(512) dft_batch_kernel(const double2* __restrict__ in, int64_t stride, int64_t dist,
                                                        int n, int inverse, double scale,
                                                        const double2* __restrict__ roots, double2* __restrict__ out) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double2* x = reinterpret_cast<double2*>(smem_raw);
  double2* scratch = x + n;
  const int64_t b = blockIdx.x;
  for (int i = threadIdx.x; i < n; i += blockDim.x) x[fsw(i, n)] = in[b * dist + (int64_t)i * stride];
  __syncthreads();
  fft_block(x, scratch, n, roots, inverse != 0);
  for (int i = threadIdx.x; i < n; i += blockDim.x) out[b * dist + (int64_t)i * stride] = cscale(x[fsw(i, n)], scale);
}

// cycle layouts (core.py:106-137) and cycle powers (:140-154), element size es (8 or 16 bytes)
template <typename E>
__global__ void cycle_layout_kernel(const E* __restrict__ in, int n, int mode, E* __restrict__ out) {
  const size_t total = (size_t)n * n;
  for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < total; e += (size_t)gridDim.x * blockDim.x) {
    const int i = (int)(e / n), j = (int)(e % n);
    size_t src;
    switch (mode) {
      case 0: src = (size_t)((i + j) % n) * n + i; break;        // reorder right: A[(i+j)%n, i]
      case 1: src = (size_t)i * n + (i - j + n) % n; break;      // reorder left:  A[i, (i-j)%n]
      case 2: src = (size_t)j * n + (i - j + n) % n; break;      // inverse right: At[c, (r-c)%n]
      default: src = (size_t)i * n + (i - j + n) % n; break;     // inverse left:  At[r, (r-c)%n]
    }
    out[e] = in[src];
  }
}

template <typename E>
__global__ void cycle_power_kernel(const E* __restrict__ in, int rows, int cols, int k, int side, E* __restrict__ out) {
  const size_t total = (size_t)rows * cols;
  for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < total; e += (size_t)gridDim.x * blockDim.x) {
    const int i = (int)(e / cols), j = (int)(e % cols);
    size_t src = side == 0 ? (size_t)((i - k + rows) % rows) * cols + j   // C^k M: rows down by k
                           : (size_t)i * cols + (j + k) % cols;           // M C^k: cols left by k
    out[e] = in[src];
  }
}

// ---------------------------------------------------------------------------------------------
// Transforms longer than one CTA's shared memory (power-of-two n >= 8192 for the products, whose
// fused kernels above keep two length-n buffers in shared memory). Four-step FFT, n = n1 * n2,
// element i = i1 * n2 + i2 of a row, output k = k1 + n1 * k2:
//   pass 1: for every i2, the length-n1 DFT over i1, times the twiddle w_n^{i2 k1}  (in place)
//   pass 2: for every k1, the length-n2 DFT over i2, stored at k1 + n1 k2            (to `out`)
// Each CTA keeps a tile of TC columns (pass 1) or TR rows (pass 2) of one sequence in shared
// memory, so every global access is a run of TC (TR) consecutive complex values. The products
// then run unfused: skew / transpose -> batched FFT -> gather in frequency space -> inverse FFT.
// ---------------------------------------------------------------------------------------------

// `count` independent power-of-two transforms of length len, transform t at x + t * stride (each
// XOR-swizzled by fsw), all threads of the CTA cooperating; same butterflies as fft_block.
__device__ inline void fft_multi(double2* x, int count, int len, int stride, const double2* __restrict__ roots,
                                 bool inverse) {
  const int tid = threadIdx.x, nt = blockDim.x;
  if (len == 1) return;
  const int logn = ilog2(len);
  for (int e = tid; e < count * len; e += nt) {
    const int t = e >> logn, i = bitrev_order(e & (len - 1), logn);
    const int j = (int)(__brev((unsigned)i) >> (32 - logn));
    if (i < j) {
      double2* b = x + (size_t)t * stride;
      const double2 v = b[fsw(i, len)];
      b[fsw(i, len)] = b[fsw(j, len)];
      b[fsw(j, len)] = v;
    }
  }
  __syncthreads();
  int s = 1;
  const int lg8 = logn - 3;
  for (; s + 2 <= logn; s += 3) {
    const int h = 1 << (s - 1);
    for (int gg = tid; gg < (count << lg8); gg += nt) {
      const int t = gg >> lg8, g = gg & ((1 << lg8) - 1);
      double2* b = x + (size_t)t * stride;
      const int pos = g & (h - 1);
      const int base = (g >> (s - 1)) << (s + 2);
      double2 v[8];
#pragma unroll
      for (int m = 0; m < 8; ++m) v[m] = b[fsw(base + pos + m * h, len)];
      radix8_apply(v, radix8_twiddles(roots, pos << (logn - s - 2), inverse));
#pragma unroll
      for (int m = 0; m < 8; ++m) b[fsw(base + pos + m * h, len)] = v[m];
    }
    __syncthreads();
  }
  const int lg2 = logn - 1;
  for (; s <= logn; ++s) {
    const int half = 1 << (s - 1);
    for (int gg = tid; gg < (count << lg2); gg += nt) {
      const int t = gg >> lg2, bb = gg & ((1 << lg2) - 1);
      double2* b = x + (size_t)t * stride;
      const int pos = bb & (half - 1);
      const int i = ((bb >> (s - 1)) << s) + pos;
      const int j = i + half;
      double2 w = __ldg(roots + (pos << (logn - s)));
      if (inverse) w.y = -w.y;
      const double2 tt = cmul(w, b[fsw(j, len)]);
      const double2 u = b[fsw(i, len)];
      b[fsw(i, len)] = cadd(u, tt);
      b[fsw(j, len)] = csub(u, tt);
    }
    __syncthreads();
  }
}

// Tiles of kBigTile sequences per CTA; tile t sits at x + t * (len + 1) in shared memory: the pad
// puts element i of the kBigTile sequences in different 16-byte bank groups, so the transposing
// tile loads / stores (consecutive threads = consecutive sequences) are conflict-free.
constexpr int kBigTile = 16;  // columns (pass 1) / rows (pass 2) per CTA: 256-byte global runs
constexpr int kBigThreads = 512;
constexpr int kBigMaxE = 16;  // tile elements per thread (kBigTile * len / kBigThreads, len <= 512)
constexpr int kBigRound = 8;  // loads in flight per thread (two CTAs per SM: <= 64 registers)

// pass 1 of the four-step transform of `rows` sequences of length n = n1 * n2: in (TI) -> data
// (complex; may alias `in` when TI is complex). grid (n2 / kBigTile, rows).
template <typename TI>
__global__ void __launch_bounds__(kBigThreads, 2) fft4_pass1_kernel(const TI* in, int n1, int n2, int inverse,
                                                                 const double2* __restrict__ roots_n,
                                                                 const double2* __restrict__ roots_n1, double2* data) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double2* x = reinterpret_cast<double2*>(smem_raw);
  const int P = n1 + 1;
  const size_t n = (size_t)n1 * n2;
  const size_t row = blockIdx.y;
  const int i20 = blockIdx.x * kBigTile;
  const int c = threadIdx.x & (kBigTile - 1), e0 = threadIdx.x / kBigTile;  // column, first i1 / k1
  constexpr int kStep = kBigThreads / kBigTile;                              // i1 / k1 step per element
  // the tile's loads in rounds of kBigRound, all of a round in flight before its stores
  const TI* src = in + row * n + i20 + c;
#pragma unroll
  for (int j0 = 0; j0 < kBigMaxE; j0 += kBigRound) {
    double2 v[kBigRound];
#pragma unroll
    for (int j = 0; j < kBigRound; ++j) {
      const int i1 = e0 + kStep * (j0 + j);
      if (i1 < n1) v[j] = ld_c<TI>(src, (size_t)i1 * n2);
    }
#pragma unroll
    for (int j = 0; j < kBigRound; ++j) {
      const int i1 = e0 + kStep * (j0 + j);
      if (i1 < n1) x[c * P + fsw(i1, n1)] = v[j];
    }
  }
  __syncthreads();
  fft_multi(x, kBigTile, n1, P, roots_n1, inverse != 0);
  // twiddle w_n^{i2 k1} for k1 = e0 + kStep j: the first from the table, the rest by repeated
  // multiplication with w_n^{i2 kStep} (<= 15 products: a few ulp)
  const size_t i2 = (size_t)(i20 + c);
  double2 w = __ldg(roots_n + ((i2 * e0) & (n - 1)));
  double2 stp = __ldg(roots_n + ((i2 * kStep) & (n - 1)));
  if (inverse) {
    w.y = -w.y;
    stp.y = -stp.y;
  }
  double2* dst = data + row * n + i2;
#pragma unroll
  for (int j = 0; j < kBigMaxE; ++j) {
    const int k1 = e0 + kStep * j;
    if (k1 < n1) {
      dst[(size_t)k1 * n2] = cmul(x[c * P + fsw(k1, n1)], w);
      w = cmul(w, stp);
    }
  }
}

// pass 2: data -> out (must not alias). grid (n1 / kBigTile, rows).
__global__ void __launch_bounds__(kBigThreads, 2) fft4_pass2_kernel(const double2* __restrict__ data, int n1, int n2,
                                                                 int inverse, const double2* __restrict__ roots_n2,
                                                                 double scale, double2* __restrict__ out) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double2* x = reinterpret_cast<double2*>(smem_raw);
  const int P = n2 + 1;
  const size_t n = (size_t)n1 * n2;
  const size_t row = blockIdx.y;
  const int k10 = blockIdx.x * kBigTile;
  // rows k10 .. k10 + kBigTile of the n1 x n2 matrix are one contiguous run of the sequence
  const double2* src = data + row * n + (size_t)k10 * n2;
  const int tot = kBigTile * n2;
#pragma unroll
  for (int j0 = 0; j0 < kBigMaxE; j0 += kBigRound) {
    double2 v[kBigRound];
#pragma unroll
    for (int j = 0; j < kBigRound; ++j) {
      const int e = threadIdx.x + kBigThreads * (j0 + j);
      if (e < tot) v[j] = __ldg(src + e);
    }
#pragma unroll
    for (int j = 0; j < kBigRound; ++j) {
      const int e = threadIdx.x + kBigThreads * (j0 + j);
      if (e < tot) {
        const int r = e / n2, i2 = e - r * n2;
        x[r * P + fsw(i2, n2)] = v[j];
      }
    }
  }
  __syncthreads();
  fft_multi(x, kBigTile, n2, P, roots_n2, inverse != 0);
  const int r = threadIdx.x & (kBigTile - 1), e0 = threadIdx.x / kBigTile;
  constexpr int kStep = kBigThreads / kBigTile;
  double2* dst = out + row * n + k10 + r;
#pragma unroll
  for (int j = 0; j < kBigMaxE; ++j) {
    const int k2 = e0 + kStep * j;
    if (k2 < n2) dst[(size_t)n1 * k2] = cscale(x[r * P + fsw(k2, n2)], scale);
  }
}

// Register-resident four-step passes for the lengths n1, n2 in {128, 256} (C5c: n = 32768 =
// 128 x 256, the n = 16384 / 65536 transforms, Bluestein lengths up to 2^16). A length
// N = R * 16 (R = 8 or 16) transform of each of the CTA's 16 sequences runs as
//   i = j + 16 m (j < 16, m < R),  k = ka + R kb:
//   A: thread (seq, j): DFT_R over m of x[j + 16 m] -> ka, times w_N^{j ka}, E[seq][ka][j]
//   B: thread (seq, ka): DFT16 over j of E[seq][ka][j] -> kb: X[ka + R kb]
// with E at seq * (16 R + 1) + ka * 16 + j (pitch = 1 mod 8 complex: every warp access hits each
// 16-byte bank group four times, the minimum). One shared exchange per pass against log2 N
// rounds of fft_multi's radix-2 tile passes; the global loads and stores keep the 256-byte runs of
// the generic kernels. 256 threads; phase B uses the first 16 R.
template <int R, bool INV>
__device__ __forceinline__ void dft_r(double2 (&v)[R]) {
  if constexpr (R == 8) dft8<INV>(v);
  else dft16<INV>(v);
}

template <typename TI, int R, bool INV>
__global__ void __launch_bounds__(256, 2) fft4_pass1_r16_kernel(const TI* in, int n2, const double2* __restrict__ roots_n,
                                                                const double2* __restrict__ roots_n1, double2* data) {
  constexpr int N1 = 16 * R, P = N1 + 1;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double2* E = reinterpret_cast<double2*>(smem_raw);  // 16 P complex
  const size_t n = (size_t)N1 * n2;
  const size_t row = blockIdx.y;
  const int i20 = blockIdx.x * 16;
  const int t = threadIdx.x;
  {
    const int c = t & 15, j = t >> 4;
    const TI* src = in + row * n + i20 + c;
    double2 v[R];
#pragma unroll
    for (int m = 0; m < R; ++m) v[m] = ld_c<TI>(src, (size_t)(j + 16 * m) * n2);
    dft_r<R, INV>(v);
    twiddle_powers<INV, R>(v, roots_n1, j);  // w_N1^{j ka}
#pragma unroll
    for (int ka = 0; ka < R; ++ka) E[c * P + ka * 16 + j] = v[ka];
  }
  __syncthreads();  // every load of the tile is done before any store (in-place when TI is complex)
  if (t < 16 * R) {
    const int c = t & 15, ka = t >> 4;
    double2 v[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) v[j] = E[c * P + ka * 16 + j];
    dft16<INV>(v);
    // X[k1] for k1 = ka + R kb, times w_n^{i2 k1}: the first from the table, then steps w_n^{i2 R}
    const size_t i2 = (size_t)(i20 + c);
    double2 w = __ldg(roots_n + ((i2 * ka) & (n - 1)));
    double2 stp = __ldg(roots_n + ((i2 * R) & (n - 1)));
    if (INV) {
      w.y = -w.y;
      stp.y = -stp.y;
    }
    double2* dst = data + row * n + i2;
#pragma unroll
    for (int kb = 0; kb < 16; ++kb) {
      dst[(size_t)(ka + R * kb) * n2] = cmul(v[kb], w);
      w = cmul(w, stp);
    }
  }
}

template <int R, bool INV>
__global__ void __launch_bounds__(256, 2) fft4_pass2_r16_kernel(const double2* __restrict__ data, int n1,
                                                                const double2* __restrict__ roots_n2, double scale,
                                                                double2* __restrict__ out) {
  constexpr int N2 = 16 * R, P = N2 + 1;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double2* E = reinterpret_cast<double2*>(smem_raw);  // 16 P complex
  const size_t n = (size_t)n1 * N2;
  const size_t row = blockIdx.y;
  const int k10 = blockIdx.x * 16;
  const int t = threadIdx.x;
  {
    const int s = t >> 4, j = t & 15;
    const double2* src = data + row * n + (size_t)(k10 + s) * N2 + j;
    double2 v[R];
#pragma unroll
    for (int m = 0; m < R; ++m) v[m] = __ldg(src + 16 * m);
    dft_r<R, INV>(v);
    twiddle_powers<INV, R>(v, roots_n2, j);  // w_N2^{j ka}
#pragma unroll
    for (int ka = 0; ka < R; ++ka) E[s * P + ka * 16 + j] = v[ka];
  }
  __syncthreads();
  if (t < 16 * R) {
    const int s = t & 15, ka = t >> 4;
    double2 v[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) v[j] = E[s * P + ka * 16 + j];
    dft16<INV>(v);
    double2* dst = out + row * n + k10 + s;
#pragma unroll
    for (int kb = 0; kb < 16; ++kb) dst[(size_t)n1 * (ka + R * kb)] = cscale(v[kb], scale);
  }
}

// big-path helpers (all grid-stride over n x n, or tiled where a transpose is involved)
// out[c][p] = in[p][c] (real or complex in, complex out), 32 x 32 tiles
template <typename TI>
__global__ void __launch_bounds__(256) transpose_to_c_kernel(const TI* __restrict__ in, int n, double2* __restrict__ out) {
  __shared__ double2 tile[32][33];
  const int c0 = blockIdx.x * 32, p0 = blockIdx.y * 32;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int r = w; r < 32; r += 8)
    if (p0 + r < n && c0 + lane < n) tile[r][lane] = ld_c<TI>(in, (size_t)(p0 + r) * n + c0 + lane);
  __syncthreads();
  for (int r = w; r < 32; r += 8)
    if (c0 + r < n && p0 + lane < n) out[(size_t)(c0 + r) * n + p0 + lane] = tile[lane][r];
}

// M[p][c] = scale * Y[c][p]
__global__ void __launch_bounds__(256) transpose_scale_c_kernel(const double2* __restrict__ Y, int n, double scale,
                                                                double2* __restrict__ M) {
  __shared__ double2 tile[32][33];
  const int p0 = blockIdx.x * 32, c0 = blockIdx.y * 32;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int r = w; r < 32; r += 8)
    if (c0 + r < n && p0 + lane < n) tile[r][lane] = Y[(size_t)(c0 + r) * n + p0 + lane];
  __syncthreads();
  for (int r = w; r < 32; r += 8)
    if (p0 + r < n && c0 + lane < n) M[(size_t)(p0 + r) * n + c0 + lane] = cscale(tile[lane][r], scale);
}

// magnitudes: partial[g][t] = sum over rows j of chunk g of |St[j][t]|^2 * s2; then mag[t] = sqrt(sum_g)
__global__ void __launch_bounds__(256) colsum_abs2_kernel(const double2* __restrict__ St, int n, int rpc, double s2,
                                                          double* __restrict__ partial) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  const int j0 = blockIdx.y * rpc, j1 = min(n, j0 + rpc);
  if (t >= n) return;
  double a = 0.0;
  for (int j = j0; j < j1; ++j) {
    const double2 v = __ldg(St + (size_t)j * n + t);
    a = fma(v.x, v.x, fma(v.y, v.y, a));
  }
  partial[(size_t)blockIdx.y * n + t] = a * s2;
}

// Ssel[q][i] = scale * St[i][sel[q]]
__global__ void __launch_bounds__(256) gather_cols_kernel(const double2* __restrict__ St, int n, const int* __restrict__ sel,
                                                          double scale, double2* __restrict__ Ssel) {
  const int q = blockIdx.y;
  const int t = sel[q];
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    Ssel[(size_t)q * n + i] = cscale(__ldg(St + (size_t)i * n + t), scale);
}

// Frequency-space gathers of the unfused path, kGatherRows rows per thread: the coefficient of
// a term (L_q[p], or conj(L_q[src]) on the right) does not depend on the row, so one load of it
// serves all the thread's rows (the rows' X reads are the only per-row traffic; a whole row is
// 16n bytes, beyond shared memory at these n, so they stream from L2).
constexpr int kGatherRows = 4;

// term1: Y[c][p] = sum_q L_q[p] * rs * FB[c][(p - t_q) % n]
__global__ void __launch_bounds__(256) big_left_gather_kernel(const double2* __restrict__ FB, int n,
                                                              const double2* __restrict__ L, const int* __restrict__ sel,
                                                              int k, double rs, double2* __restrict__ Y) {
  __shared__ int s_buf[512];
  for (int q = threadIdx.x; q < k && q < 512; q += blockDim.x) s_buf[q] = sel[q];
  __syncthreads();
  const int* s_sel = k <= 512 ? s_buf : sel;
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  const size_t c0 = (size_t)blockIdx.y * kGatherRows;
  if (p >= n) return;
  double2 a[kGatherRows];
#pragma unroll
  for (int rr = 0; rr < kGatherRows; ++rr) a[rr] = make_double2(0.0, 0.0);
  for (int q = 0; q < k; ++q) {
    int src = p - s_sel[q];
    if (src < 0) src += n;
    const double2 l = __ldg(L + (size_t)q * n + p);
    double2 x[kGatherRows];
#pragma unroll
    for (int rr = 0; rr < kGatherRows; ++rr)
      x[rr] = c0 + rr < (size_t)n ? __ldg(FB + (c0 + rr) * n + src) : make_double2(0.0, 0.0);
#pragma unroll
    for (int rr = 0; rr < kGatherRows; ++rr) a[rr] = cadd(a[rr], cmul(l, x[rr]));
  }
#pragma unroll
  for (int rr = 0; rr < kGatherRows; ++rr)
    if (c0 + rr < (size_t)n) Y[(c0 + rr) * n + p] = cscale(a[rr], rs);
}

// X[r][c] = conj(A[r][c] - Ahat[r][c]), Ahat[r][c] = sum_q Ssel[q][(r - c) % n] exp(+2 pi i t_q c / n).
// Thread = column c of a block of kDaRows rows: the twiddle of (q, c) -- a scattered table load --
// is shared by the block's rows, and for a fixed row the lanes read consecutive S_q entries.
constexpr int kDaRows = 16;
template <typename T>
// [row_base, row_end): the rows to form (sharded product); X holds them from row row_base on.
__global__ void __launch_bounds__(256, 2) big_dA_kernel(const T* __restrict__ A, int n, const double2* __restrict__ Ssel,
                                                     const int* __restrict__ sel, int k,
                                                     const double2* __restrict__ roots, double2* __restrict__ X,
                                                     int row_base = 0, int row_end = -1) {
  if (row_end < 0) row_end = n;
  __shared__ int s_buf[512];
  for (int q = threadIdx.x; q < k && q < 512; q += blockDim.x) s_buf[q] = sel[q];
  __syncthreads();
  const int* s_sel = k <= 512 ? s_buf : sel;
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  const int r0 = row_base + blockIdx.y * kDaRows;
  if (c >= n) return;
  double2 ah[kDaRows];
#pragma unroll
  for (int rr = 0; rr < kDaRows; ++rr) ah[rr] = make_double2(0.0, 0.0);
  int d0 = r0 - c;
  if (d0 < 0) d0 += n;
  for (int q = 0; q < k; ++q) {
    const double2 w = cconj(__ldg(roots + mulmod_n(s_sel[q], c, n)));
    const double2* Sq = Ssel + (size_t)q * n;
#pragma unroll
    for (int rr = 0; rr < kDaRows; ++rr) {
      int d = d0 + rr;
      if (d >= n) d -= n;
      ah[rr] = cmac(ah[rr], __ldg(Sq + d), w);
    }
  }
#pragma unroll
  for (int rr = 0; rr < kDaRows; ++rr) {
    const size_t r = (size_t)r0 + rr;
    if (r < (size_t)row_end) X[(r - row_base) * n + c] = cconj(csub(ld_c<T>(A, r * n + c), ah[rr]));
  }
}

// Same result as big_dA_kernel with the S_q reads staged through shared memory: for the CTA's
// 256 columns x kDaRows rows, d = r - c spans one window of 256 + kDaRows - 1 consecutive
// (cyclic) indices per term, so the k windows (k x 271 x 16 B = 69 KB at k = 16) are loaded once,
// coalesced, and every thread's 16 reads per term are conflict-free LDS.128 (the lanes' d are
// consecutive) instead of L2 loads (big_dA_kernel: 74% of its stalls waited on them). The
// twiddle of (q, c) is loaded one term ahead. k <= kDaWinMaxK (smem).
constexpr int kDaWinMaxK = 48;
template <typename T, int ROWS>
__global__ void __launch_bounds__(256, 2) big_dA_win_kernel(const T* __restrict__ A, int n,
                                                         const double2* __restrict__ Ssel,
                                                         const int* __restrict__ sel, int k,
                                                         const double2* __restrict__ roots,
                                                         double2* __restrict__ X, int row_base, int row_end) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  constexpr int W = 256 + ROWS - 1;
  double2* win = reinterpret_cast<double2*>(smem_raw);  // k x W
  // twiddles w_q(c0 + l) = conj(roots[t_q (c0 + l) mod n]), factored as base_q * hi_q[l >> 4] *
  // lo_q[l & 15]: 33 table loads per term per CTA instead of one scattered load per (term, thread)
  __shared__ double2 tw_base[kDaWinMaxK], tw_lo[kDaWinMaxK][16], tw_hi[kDaWinMaxK][16];
  const int tid = threadIdx.x;
  const int c0 = blockIdx.x * 256;
  for (int e = tid; e < k * 33; e += blockDim.x) {
    const int q = e / 33, j = e - q * 33;
    const int t = sel[q];
    if (j == 32) tw_base[q] = cconj(__ldg(roots + mulmod_n(t, c0 % n, n)));
    else if (j < 16) tw_lo[q][j] = cconj(__ldg(roots + mulmod_n(t, j % n, n)));
    else tw_hi[q][j - 16] = cconj(__ldg(roots + mulmod_n(t, (16 * (j - 16)) % n, n)));
  }
  const int r0 = row_base + blockIdx.y * ROWS;
  // the epilogue reads this CTA's ROWS x 256 tile of A (DRAM-resident): pull it into L2 now, one bulk
  // prefetch per row, so the final loads (the kernel's largest stall) hit L2
  if (tid < ROWS && r0 + tid < row_end && c0 < n) {
    const T* rowp = A + (size_t)(r0 + tid) * n + c0;
    const unsigned bytes = (unsigned)(min(256, n - c0) * sizeof(T)) & ~15u;
    if (((uintptr_t)rowp & 15) == 0 && bytes > 0)
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(rowp), "r"(bytes) : "memory");
  }
  // window j of term q holds S_q[(r0 - c0 - 255 + j) mod n]; thread tid, row rr reads j = 255 - tid + rr
  int dbase = (r0 - c0 - 255) % n;
  if (dbase < 0) dbase += n;
  for (int e = tid; e < k * W; e += blockDim.x) {
    const int q = e / W, j = e - q * W;
    int d = dbase + j;
    if (d >= n) d -= n;
    win[e] = __ldg(Ssel + (size_t)q * n + d);
  }
  __syncthreads();
  const int c = c0 + tid;
  if (c >= n) return;
  double2 ah[ROWS];
#pragma unroll
  for (int rr = 0; rr < ROWS; ++rr) ah[rr] = make_double2(0.0, 0.0);
  for (int q = 0; q < k; ++q) {
    const double2 w = cmul(cmul(tw_base[q], tw_hi[q][tid >> 4]), tw_lo[q][tid & 15]);
    const double2* wq = win + (size_t)q * W + (255 - tid);
    APX_DCHECK(255 - tid + ROWS - 1 < W);
#pragma unroll
    for (int rr = 0; rr < ROWS; ++rr) ah[rr] = cmac(ah[rr], wq[rr], w);
  }
#pragma unroll
  for (int rr = 0; rr < ROWS; ++rr) {
    const size_t r = (size_t)r0 + rr;
    if (r < (size_t)row_end) X[(r - row_base) * n + c] = cconj(csub(ld_c<T>(A, r * n + c), ah[rr]));
  }
}

// Same result as big_dA_win_kernel by register blocks: a thread forms an 8-row x 4-column tile
// (rows r0 + 8 rg + a, columns c0 + 4 cg + b) and the CTA a 32 x 4 kCG tile. Over the thread's tile
// d = r - c takes only 11 distinct values (a - b in [-3, 7]), so one term costs 11 window loads and
// 2 twiddle loads (LDS.128) for 32 complex MACs -- the per-column kernel spends 16 + 3 on 16 -- and
// the column twiddles w_q(c + b) come from w_q(c) by the recurrence w *= w_q(1). The window of term
// q (W = 32 + 4 kCG - 1 consecutive cyclic indices of S_q) is stored split by j mod 4 at position
// j >> 2: for a fixed m the lanes' reads j = 4 (2 rg - cg + kCG - 1) + m are consecutive positions of
// one class, i.e. conflict-free. Terms are staged kKC at a time into two buffers by cp.async (the
// next chunk lands while this one is multiplied), so any k runs. NW warps per CTA: 4 row groups x
// NW/4 column halves of 32 column groups; the default NW = 4 (128 x 32 tile, 194 registers) keeps
// two CTAs per SM so one CTA's staging and epilogue overlap the other's multiplies.
template <int NW>
struct DaBlk {
  static constexpr int kThreads = 32 * NW, kR = 32, kCG = 8 * NW, kC = 4 * kCG, kKC = 8;
  static constexpr int kW = kR + kC - 1, kP = (kW + 3) / 4;
  static constexpr size_t kWinBytes = sizeof(double2) * kKC * 4 * kP;
  static constexpr size_t kTwBytes = sizeof(double2) * kKC * (kCG + 1);
  static constexpr size_t kSmem = 2 * (kWinBytes + kTwBytes);
  static constexpr size_t kATile = sizeof(double) * kR * kC;  // real operands: A's tile for the epilogue
};
__device__ __forceinline__ void da_cp16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"((unsigned)__cvta_generic_to_shared(dst)),
               "l"(src)
               : "memory");
}
template <typename T, int NW>
__global__ void __launch_bounds__(32 * NW, 8 / NW) big_dA_blk_kernel(const T* __restrict__ A, int n,
                                                                  const double2* __restrict__ Ssel,
                                                                  const int* __restrict__ sel, int k,
                                                                  const double2* __restrict__ roots,
                                                                  double2* __restrict__ X, int row_base,
                                                                  int row_end) {
  using G = DaBlk<NW>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  using Win = double2[G::kKC][4][G::kP];
  using Tw = double2[G::kKC][G::kCG + 1];  // [q][column group g] = w_q(c0 + 4 g); [q][kCG] = w_q(1)
  Win* win = reinterpret_cast<Win*>(smem_raw);
  Tw* tw = reinterpret_cast<Tw*>(smem_raw + 2 * G::kWinBytes);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int cg = (warp >> 2) * 32 + lane, rg = warp & 3;
  const int c0 = blockIdx.x * G::kC, r0 = row_base + blockIdx.y * G::kR;
  // window entry j of every term is S_q[(r0 - c0 - (kC - 1) + j) mod n]
  int dbase = (int)(((long long)r0 - c0 - (G::kC - 1)) % n);
  if (dbase < 0) dbase += n;
  // the epilogue reads the CTA's tile of A: real operands stage it into shared memory by cp.async
  // with the first chunk (it lands under the multiplies), complex ones pull it into L2
  constexpr bool kStageA = std::is_same<T, double>::value;
  double* As = reinterpret_cast<double*>(smem_raw + G::kSmem);  // [kR][kC] when kStageA
  if constexpr (kStageA) {
    const int cols = min(G::kC, n - c0);
    if ((n & 1) == 0) {
      for (int e = tid; e < G::kR * (G::kC / 2); e += G::kThreads) {
        const int rr = e / (G::kC / 2), cc = 2 * (e - rr * (G::kC / 2));
        if (r0 + rr < row_end && cc < cols) da_cp16(As + rr * G::kC + cc, A + (size_t)(r0 + rr) * n + c0 + cc);
      }
    } else {
      for (int e = tid; e < G::kR * G::kC; e += G::kThreads) {
        const int rr = e / G::kC, cc = e - rr * G::kC;
        if (r0 + rr < row_end && cc < cols)
          asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(
                           (unsigned)__cvta_generic_to_shared(As + rr * G::kC + cc)),
                       "l"(A + (size_t)(r0 + rr) * n + c0 + cc)
                       : "memory");
      }
    }
  } else if (tid < G::kR && r0 + tid < row_end) {
    const T* rowp = A + (size_t)(r0 + tid) * n + c0;
    const unsigned bytes = (unsigned)(min(G::kC, n - c0) * sizeof(T)) & ~15u;
    if (((uintptr_t)rowp & 15) == 0 && bytes > 0)
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(rowp), "r"(bytes) : "memory");
  }
  // the staging is all cp.async (windows and twiddle-table entries; conj applied at use), indices
  // wrapped by one conditional subtract when n >= W (a 64-bit modulo per entry was 11% of the stalls)
  auto stage = [&](int q0, int buf) {
    const int kc = min(G::kKC, k - q0);
    if (n >= G::kW) {
      for (int q = 0; q < kc; ++q) {
        const double2* Sq = Ssel + (size_t)(q0 + q) * n;
        for (int j = tid; j < G::kW; j += G::kThreads) {
          const int d = dbase + j;
          da_cp16(&win[buf][q][j & 3][j >> 2], Sq + (d >= n ? d - n : d));
        }
      }
    } else {
      for (int e = tid; e < kc * G::kW; e += G::kThreads) {
        const int q = e / G::kW, j = e - q * G::kW;
        da_cp16(&win[buf][q][j & 3][j >> 2], Ssel + (size_t)(q0 + q) * n + (dbase + j) % n);
      }
    }
    for (int e = tid; e < kc * (G::kCG + 1); e += G::kThreads) {
      const int q = e / (G::kCG + 1), g = e - q * (G::kCG + 1);
      int c = g < G::kCG ? c0 + 4 * g : 1;
      if (c >= n) c %= n;
      da_cp16(&tw[buf][q][g], roots + mulmod_n(__ldg(sel + q0 + q), c, n));  // conj: exp(+2 pi i t c / n)
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  };
  double2 ah[8][4];
#pragma unroll
  for (int a = 0; a < 8; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) ah[a][b] = make_double2(0.0, 0.0);
  // j(a, b) = 8 rg + a - 4 cg - b + kC - 1 = 4 pbase + (a - b + 3)
  const int pbase = 2 * rg + G::kCG - 1 - cg;
  if (k > 0) stage(0, 0);
  for (int q0 = 0, it = 0; q0 < k; q0 += G::kKC, ++it) {
    const int buf = it & 1;
    if (q0 + G::kKC < k) {
      stage(q0 + G::kKC, buf ^ 1);
      asm volatile("cp.async.wait_group 1;\n" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    }
    __syncthreads();
    const int kc = min(G::kKC, k - q0);
    for (int q = 0; q < kc; ++q) {
      double2 v[11];
#pragma unroll
      for (int m = 0; m < 11; ++m) v[m] = win[buf][q][m & 3][pbase + (m >> 2)];
      double2 w[4];
      w[0] = cconj(tw[buf][q][cg]);
      const double2 w1 = cconj(tw[buf][q][G::kCG]);
#pragma unroll
      for (int b = 1; b < 4; ++b) w[b] = cmul(w[b - 1], w1);
#pragma unroll
      for (int a = 0; a < 8; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) ah[a][b] = cmac(ah[a][b], v[a - b + 3], w[b]);
    }
    __syncthreads();  // buffer buf is restaged two chunks on
  }
  if (k <= 0) {  // nothing staged a window: the A tile's copies still need their wait
    asm volatile("cp.async.commit_group;\n" ::: "memory");
    asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    __syncthreads();
  }
  // epilogue: all of the tile's A loads first (the stores' asm would otherwise order each row's
  // loads behind the previous row's stores), then conj(A - Ahat) out as 32-byte stores
  const int cb = c0 + 4 * cg;
#pragma unroll
  for (int a = 0; a < 8; ++a) {
    const int r = r0 + 8 * rg + a;
#pragma unroll
    for (int b = 0; b < 4; ++b)
      if (r < row_end && cb + b < n) {
        double2 x;
        if constexpr (kStageA) x = make_double2(As[(8 * rg + a) * G::kC + 4 * cg + b], 0.0);
        else x = ld_c<T>(A, (size_t)r * n + cb + b);
        ah[a][b] = cconj(csub(x, ah[a][b]));
      }
  }
#pragma unroll
  for (int a = 0; a < 8; ++a) {
    const int r = r0 + 8 * rg + a;
    if (r >= row_end) continue;
    double2* dst = X + (size_t)(r - row_base) * n + cb;
    if (cb + 3 < n && (((uintptr_t)dst) & 31) == 0) {
#pragma unroll
      for (int h = 0; h < 2; ++h)
        asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(dst + 2 * h), "d"(ah[a][2 * h].x),
                     "d"(ah[a][2 * h].y), "d"(ah[a][2 * h + 1].x), "d"(ah[a][2 * h + 1].y)
                     : "memory");
    } else {
#pragma unroll
      for (int b = 0; b < 4; ++b)
        if (cb + b < n) dst[b] = ah[a][b];
    }
  }
}

// conj(dA) rows [row_base, row_end) into X (rows from row_base on): the register-blocked kernel
// (any k); APX_DA_KERNEL=win|l2 selects the earlier per-column kernels for A/B timing
template <typename T>
static int launch_big_dA(const T* A, int n, const double2* Ssel, const int* sel, int k, const double2* roots,
                         double2* X, int row_base, int row_end, cudaStream_t st) {
  const dim3 grid((unsigned)ceil_div(n, 256), (unsigned)ceil_div(row_end - row_base, kDaRows));
  // rows per CTA of the windowed kernel (APX_DA_ROWS=16|32, tuning knob)
  static const int da_rows = [] {
    const char* e = getenv("APX_DA_ROWS");
    return (e && atoi(e) == 32) ? 32 : 16;
  }();
  static const int da_kind = [] {
    const char* e = getenv("APX_DA_KERNEL");
    if (getenv("APX_DA_L2")) return 2;
    return !e ? 0 : (strcmp(e, "win") == 0 ? 1 : strcmp(e, "l2") == 0 ? 2 : 0);
  }();
  if (da_kind == 0) {
    auto go = [&](auto kern, auto geom) -> int {
      using G = decltype(geom);
      const size_t smem = G::kSmem + (std::is_same<T, double>::value ? G::kATile : 0);
      APX_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      const dim3 g((unsigned)ceil_div(n, G::kC), (unsigned)ceil_div(row_end - row_base, G::kR));
      kern<<<g, G::kThreads, smem, st>>>(A, n, Ssel, sel, k, roots, X, row_base, row_end);
      return OK;
    };
    static const bool wide = getenv("APX_DA_WIDE") != nullptr;  // 256-thread CTAs (one per SM)
    if (wide) APX_TRY(go(big_dA_blk_kernel<T, 8>, DaBlk<8>{}));
    else APX_TRY(go(big_dA_blk_kernel<T, 4>, DaBlk<4>{}));
  } else if (da_kind == 1 && k <= kDaWinMaxK && n >= 256) {
    auto go = [&](auto kern, int rows) -> int {
      const size_t smem = (size_t)std::max(k, 1) * (256 + rows - 1) * sizeof(double2);
      APX_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      const dim3 g((unsigned)ceil_div(n, 256), (unsigned)ceil_div(row_end - row_base, rows));
      kern<<<g, 256, smem, st>>>(A, n, Ssel, sel, k, roots, X, row_base, row_end);
      return OK;
    };
    if (da_rows == 32) APX_TRY(go(big_dA_win_kernel<T, 32>, 32));
    else APX_TRY(go(big_dA_win_kernel<T, 16>, 16));
  } else {
    big_dA_kernel<T><<<grid, 256, 0, st>>>(A, n, Ssel, sel, k, roots, X, row_base, row_end);
  }
  APX_LAUNCH_CHECK();
  return OK;
}

// term2: Y[r][p] = sum_q (rs * X[r][(p + s_q) % n]) * conj(L_q[(p + s_q) % n])
__global__ void __launch_bounds__(256) big_right_gather_kernel(const double2* __restrict__ X, int n,
                                                               const double2* __restrict__ L, const int* __restrict__ sel,
                                                               int k, double rs, double2* __restrict__ Y) {
  __shared__ int s_buf[512];
  for (int q = threadIdx.x; q < k && q < 512; q += blockDim.x) s_buf[q] = sel[q];
  __syncthreads();
  const int* s_sel = k <= 512 ? s_buf : sel;
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  const size_t r0 = (size_t)blockIdx.y * kGatherRows;
  if (p >= n) return;
  double2 a[kGatherRows];
#pragma unroll
  for (int rr = 0; rr < kGatherRows; ++rr) a[rr] = make_double2(0.0, 0.0);
  for (int q = 0; q < k; ++q) {
    int src = p + s_sel[q];
    if (src >= n) src -= n;
    const double2 l = __ldg(L + (size_t)q * n + src);
    double2 x[kGatherRows];
#pragma unroll
    for (int rr = 0; rr < kGatherRows; ++rr)
      x[rr] = r0 + rr < (size_t)n ? __ldg(X + (r0 + rr) * n + src) : make_double2(0.0, 0.0);
#pragma unroll
    for (int rr = 0; rr < kGatherRows; ++rr) a[rr] = cadd(a[rr], cmulc(x[rr], l));
  }
#pragma unroll
  for (int rr = 0; rr < kGatherRows; ++rr)
    if (r0 + rr < (size_t)n) Y[(r0 + rr) * n + p] = cscale(a[rr], rs);
}

// M += conj(rs * Y)
__global__ void __launch_bounds__(256) acc_conj_kernel(const double2* __restrict__ Y, size_t count, double rs,
                                                       double2* __restrict__ M) {
  for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < count; e += (size_t)gridDim.x * blockDim.x)
    M[e] = cadd(M[e], cconj(cscale(Y[e], rs)));
}

// ---------------------------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------------------------
struct CircPlan {
  double2 *roots, *S_a, *S_b, *Ssel_a, *L_a, *Ssel_b, *L_b;
  double *part, *mag_a, *mag_b, *red;
  double *red2, *msq;  // side-stream ||A||^2 / ||B||^2 partials; per-CTA ||M||^2 of term2's epilogue
  int cpc, parts;
};

static void plan_circ(Workspace& ws, CircPlan& p, int n, int k, bool need_sa_full) {
  p.cpc = std::max(1, (int)ceil_div(n, 2 * kNumSMs));
  p.parts = (int)ceil_div(n, p.cpc);
  p.roots = ws.take<double2>(n);
  p.S_a = ws.take<double2>((size_t)n * n);
  p.S_b = need_sa_full ? ws.take<double2>((size_t)n * n) : p.S_a;
  p.Ssel_a = ws.take<double2>((size_t)std::max(k, 1) * n);
  p.L_a = ws.take<double2>((size_t)std::max(k, 1) * n);
  p.Ssel_b = ws.take<double2>((size_t)std::max(k, 1) * n);
  p.L_b = ws.take<double2>((size_t)std::max(k, 1) * n);
  p.part = ws.take<double>((size_t)p.parts * n);
  p.mag_a = ws.take<double>(n);
  p.mag_b = ws.take<double>(n);
  p.red = ws.take<double>(4 * kNumSMs + 64);
  p.red2 = ws.take<double>(4 * kNumSMs + 64);
  p.msq = ws.take<double>((size_t)ceil_div(n, 2) + 1);
}

// term1's L rows staged in shared memory by bulk async copies (circ_left2_kernel stage_l; n = 4096:
// kPP positions of 512 threads, halves = the threads' first / second kPP/2 positions). Measured
// neutral to slightly slower at C3 (0.704 vs 0.684 ms: the gather is not waiting on L2 for L), so
// it is off by default; APX_L2_STAGE=1 turns it on (A/B).
static int left2_stage_l(int n, int k) {
  static const bool on = getenv("APX_L2_STAGE") != nullptr;
  return on && n == kPP * 512 && k > 0;
}
static size_t left2_stage_bytes(int n) { return 128 + (size_t)n * sizeof(double2) + 2 * sizeof(uint64_t); }

// term2's forward transforms in plain order (APX_R2_SWIZZLED=1: the XOR-swizzled order, A/B)
static int right2_linear() {
  static const int v = getenv("APX_R2_SWIZZLED") == nullptr ? 1 : 0;
  return v;
}

// real operands whose transform runs in the packed-pair branch read the diagonals directly
template <typename T>
static int decompose_direct(int n) {
  static const bool off = getenv("APX_CIRC_SKEW") != nullptr;  // A/B switch: the skewed-copy path
  return std::is_same<T, double>::value && n <= 8 * 512 && !off;
}

// S^T (St[j][t] = S[t][j]) and the magnitudes; `skew` is n x n scratch of T
template <typename T>
static int circ_decompose_run(const T* A, int n, const CircPlan& p, double2* St, double* mag, T* skew,
                              cudaStream_t st) {
  const size_t smem = fft_smem_bytes(n, 1) + (size_t)n * sizeof(double);
  const int direct = decompose_direct<T>(n);
  if (!direct) {
    circ_skew_kernel<T><<<dim3((unsigned)ceil_div(n, 32), (unsigned)ceil_div(n, 32)), 256, 0, st>>>(A, n, skew);
    APX_LAUNCH_CHECK();
  }
  (void)smem;
  APX_TRY(launch_decompose_rows<T>(direct ? A : skew, n, p.cpc, p.roots, St, p.part, p.parts, 0, 0, direct, st));
  mag_finalize_kernel<<<(unsigned)ceil_div(n, 32), 256, 0, st>>>(p.part, p.parts, n, mag);
  APX_LAUNCH_CHECK();
  return OK;
}

static int circ_spectra_run(const double2* S, int n, const int* sel, int k, const double2* roots, double2* Ssel,
                            double2* L, cudaStream_t st) {
  if (k <= 0) return OK;
  const size_t smem = fft_smem_bytes(n, 1);
  APX_CUDA(cudaFuncSetAttribute(circ_spectra_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  // L carries both unitary factors of the fused products (rs for the forward and rs for the
  // inverse transform, an exact power-of-two scale for power-of-two n): the gathers and the
  // outputs need no scaling of their own
  circ_spectra_kernel<<<k, 512, smem, st>>>(S, n, sel, roots, Ssel, L, 0, 1.0 / n);
  APX_LAUNCH_CHECK();
  return OK;
}

template <typename T>
static int run_circulant(const T* A, const T* B, int n, int k, int order, const int* fa, const int* fb, double2* M,
                         int* sa, int* sb, double* scal, const CircPlan& p, cudaStream_t st) {
  stage_mark(0, st);
  APX_CUDA(cudaMemsetAsync(scal, 0, APX_NSCALARS * sizeof(double), st));
  // ||A||^2 and ||B||^2 on the side stream: HBM passes under the L1-pipe-bound transform kernels
  cudaStream_t side = st;
  APX_TRY(side_fork(st, &side));
  {
    int sp = 0;
    const size_t nel = (size_t)n * n * (sizeof(T) / sizeof(double));
    APX_TRY(launch_sumsq<double>(reinterpret_cast<const double*>(A), nel, p.red2, &sp, side));
    APX_TRY(launch_sum_vector(p.red2, sp, scal + APX_S_FRO2_A, side));
    APX_TRY(launch_sumsq<double>(reinterpret_cast<const double*>(B), nel, p.red2, &sp, side));
    APX_TRY(launch_sum_vector(p.red2, sp, scal + APX_S_FRO2_B, side));
  }
  launch_roots(p.roots, n, st);
  APX_LAUNCH_CHECK();
  T* skew = reinterpret_cast<T*>(M);  // M (n x n complex) is scratch until the left product
  APX_TRY(circ_decompose_run<T>(A, n, p, p.S_a, p.mag_a, skew, st));
  if (fa) { if (k) APX_CUDA(cudaMemcpyAsync(sa, fa, k * sizeof(int), cudaMemcpyDeviceToDevice, st)); }
  else APX_TRY(launch_topk(p.mag_a, n, k, sa, st));
  APX_TRY(launch_kept_energy(p.mag_a, sa, k, (double)n, scal + APX_S_KEPT_A, st));
  APX_TRY(circ_spectra_run(p.S_a, n, sa, k, p.roots, p.Ssel_a, p.L_a, st));
  // B's spectrum reuses S_a's storage (A's selected rows are already copied out)
  APX_TRY(circ_decompose_run<T>(B, n, p, p.S_b, p.mag_b, skew, st));
  if (fb) { if (k) APX_CUDA(cudaMemcpyAsync(sb, fb, k * sizeof(int), cudaMemcpyDeviceToDevice, st)); }
  else APX_TRY(launch_topk(p.mag_b, n, k, sb, st));
  APX_TRY(launch_kept_energy(p.mag_b, sb, k, (double)n, scal + APX_S_KEPT_B, st));
  APX_TRY(circ_spectra_run(p.S_b, n, sb, k, p.roots, p.Ssel_b, p.L_b, st));
  stage_mark(1, st);
  const size_t smem = fft_smem_bytes(n, 2) + (size_t)2 * k * sizeof(int);  // + staged selections
  const bool pairs = n >= 2 && n <= kPP * 512;  // two columns / rows per CTA (same smem footprint)
  static const bool r16_off = getenv("APX_CIRC_R16") != nullptr && atoi(getenv("APX_CIRC_R16")) == 0;
  if (std::is_same<T, double>::value && n == 4096 && !r16_off) {
    const size_t smem2r = (size_t)2 * kFFT16Buf * sizeof(double2) + (size_t)k * sizeof(int);
    APX_CUDA(cudaFuncSetAttribute(circ_left2_r16_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem2r));
    circ_left2_r16_kernel<<<n / 2, 512, smem2r, st>>>(reinterpret_cast<const double*>(B), p.L_a, sa, k, p.roots, M,
                                                       0, n, (int64_t)n);
    APX_LAUNCH_CHECK();
  } else if (pairs) {
    auto fn = circ_left2_kernel<T>;
    const int stage_l = left2_stage_l(n, k);
    const size_t smem_l = smem + (stage_l ? left2_stage_bytes(n) : 0);
    APX_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_l));
    fn<<<(unsigned)ceil_div(n, 2), 512, smem_l, st>>>(B, n, p.L_a, sa, k, p.roots, M, 0, (int)n, (int64_t)n,
                                                      stage_l);
    APX_LAUNCH_CHECK();
  } else {
    auto fn = circ_left_kernel<T>;
    APX_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    fn<<<n, 512, smem, st>>>(B, n, p.L_a, sa, k, p.roots, M);
    APX_LAUNCH_CHECK();
  }
  stage_mark(2, st);
  if (order == 1) {
    if (pairs) {
      auto fn = circ_right2_kernel<T>;
      APX_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      // conj(dA) = conj(A - Ahat) into S_a's storage (free once both spectra are copied out)
      const double2* Xpre = nullptr;
      static const bool inline_da = [] {
        const char* e = getenv("APX_CIRC_DA_INLINE");  // A/B switch: Ahat formed inside the row kernel
        return e != nullptr && atoi(e) != 0;
      }();
      if (!inline_da && n >= kDaRows) {  // (big_dA_kernel wraps d0 + rr < 2n once)
        APX_TRY(launch_big_dA<T>(A, n, p.Ssel_a, sa, k, p.roots, p.S_a, 0, n, st));
        Xpre = p.S_a;
      }
      if (Xpre != nullptr && n == 4096 && !r16_off) {
        const size_t smem2r = (size_t)2 * kFFT16Buf * sizeof(double2) + (size_t)k * sizeof(int);
        APX_CUDA(cudaFuncSetAttribute(circ_right2_r16_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem2r));
        circ_right2_r16_kernel<<<n / 2, 512, smem2r, st>>>(Xpre, p.L_b, sb, k, p.roots, M, p.msq, 0, n);
      } else {
        fn<<<(unsigned)ceil_div(n, 2), 512, smem, st>>>(A, n, p.Ssel_a, sa, k, p.L_b, sb, k, p.roots, M, Xpre, 0,
                                                        (int)n, right2_linear(), p.msq);
      }
    } else {
      auto fn = circ_right_kernel<T>;
      APX_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      fn<<<n, 512, smem, st>>>(A, n, p.Ssel_a, sa, k, p.L_b, sb, k, p.roots, M);
    }
    APX_LAUNCH_CHECK();
  }
  stage_mark(3, st);
  if (order == 1 && pairs) {  // term2's epilogue left one ||M||^2 partial per CTA
    APX_TRY(launch_sum_vector(p.msq, (int)ceil_div(n, 2), scal + APX_S_FRO2_M, st));
  } else {
    int parts = 0;
    APX_TRY(launch_sumsq<double>(reinterpret_cast<const double*>(M), (size_t)2 * n * n, p.red, &parts, st));
    APX_TRY(launch_sum_vector(p.red, parts, scal + APX_S_FRO2_M, st));
  }
  APX_TRY(side_join(st, side));
  stage_mark(4, st);
  return OK;
}


// ---- big path: transforms whose buffers exceed shared memory ---------------------------------------
// Powers of two run the four-step transform directly; other lengths go through Bluestein's
// identity jk = (j^2 + k^2 - (k-j)^2) / 2: X[k] = w[k] sum_j (x[j] w[j]) conj(w[k-j]),
// w[m] = exp(-pi i m^2 / n), a cyclic convolution of length L = 2^ceil(log2(2n-1)) evaluated with
// two four-step transforms of length L and the precomputed transform of the conjugate chirp.
static int next_pow2(int64_t v) {
  int64_t p = 1;
  while (p < v) p <<= 1;
  return (int)p;
}
static int big_len(int64_t n) { return is_pow2((int)n) ? (int)n : next_pow2(2 * n - 1); }
static bool big_fft_ok(int64_t n) { return n >= 256 && n <= 46340 * 2 && big_len(n) <= (1 << 18); }
// APX_FFT_BIG=1 routes every eligible length through this path (tests compare it with the fused one)
static bool force_big(int64_t n) {
  static const bool on = [] {
    const char* e = getenv("APX_FFT_BIG");
    return e && atoi(e) != 0;
  }();
  return on && big_fft_ok(n);
}
static bool circ_fused_fits(int n, int k) {
  return !force_big(n) && fft_smem_bytes(n, 2) + (size_t)2 * std::max(k, 0) * sizeof(int) <= 227 * 1024;
}

struct BigFFT {
  int n, L, n1, n2;  // transform length; four-step length L = n1 * n2 (n itself for powers of two)
  bool blue;
  int chunk;         // Bluestein: rows per pass through t1 / t2
  double2 *roots, *roots1, *roots2, *chirp, *bf, *t1, *t2;
};

static void plan_big_fft(Workspace& ws, BigFFT& f, int n, int max_rows) {
  f.n = n;
  f.blue = !is_pow2(n);
  f.L = big_len(n);
  const int l = ilog2(f.L);
  f.n1 = 1 << (l / 2);
  f.n2 = 1 << (l - l / 2);
  f.roots = ws.take<double2>(f.L);
  f.roots1 = ws.take<double2>(f.n1);
  f.roots2 = ws.take<double2>(f.n2);
  f.chunk = 0;
  f.chirp = f.bf = f.t1 = f.t2 = nullptr;
  if (f.blue) {
    f.chunk = (int)std::max<int64_t>(1, std::min<int64_t>(std::max(max_rows, 1), (int64_t)(1 << 26) / f.L));
    f.chirp = ws.take<double2>(n);
    f.bf = ws.take<double2>(f.L);
    f.t1 = ws.take<double2>((size_t)f.chunk * f.L);
    f.t2 = ws.take<double2>((size_t)f.chunk * f.L);
  }
}

__global__ void chirp_kernel(double2* w, int n) {
  for (int m = blockIdx.x * blockDim.x + threadIdx.x; m < n; m += gridDim.x * blockDim.x) {
    const long long q = ((long long)m * m) % (2LL * n);  // exact: the angle pi m^2 / n mod 2 pi
    double sn, cs;
    sincospi((double)q / (double)n, &sn, &cs);
    w[m] = make_double2(cs, -sn);  // exp(-pi i m^2 / n)
  }
}

// b[m] = conj(w[|m|]) on the cyclic index set of length L (zero between n and L - n)
__global__ void chirp_conv_kernel(const double2* __restrict__ w, int n, int L, double2* __restrict__ b) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < L; i += gridDim.x * blockDim.x) {
    double2 v = make_double2(0.0, 0.0);
    if (i < n) v = cconj(w[i]);
    else if (i > L - n) v = cconj(w[L - i]);
    b[i] = v;
  }
}

// a[r][j] = (conj if inverse)(x[r][j]) * w[j] for j < n, 0 up to L
template <typename TI>
__global__ void chirp_pre_kernel(const TI* __restrict__ x, int n, int L, int rows, const double2* __restrict__ w,
                                 int inverse, double2* __restrict__ a) {
  const size_t total = (size_t)rows * L;
  for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < total; e += (size_t)gridDim.x * blockDim.x) {
    const size_t r = e / L;
    const int j = (int)(e - r * L);
    double2 v = make_double2(0.0, 0.0);
    if (j < n) {
      double2 xv = ld_c<TI>(x, r * n + j);
      if (inverse) xv = cconj(xv);
      v = cmul(xv, w[j]);
    }
    a[e] = v;
  }
}

__global__ void rows_mul_kernel(double2* __restrict__ a, int L, int rows, const double2* __restrict__ bf) {
  const size_t total = (size_t)rows * L;
  for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < total; e += (size_t)gridDim.x * blockDim.x)
    a[e] = cmul(a[e], __ldg(bf + (e % L)));
}

// out[r][k] = scale * (conj if inverse)(w[k] * c[r][k]), k < n
__global__ void chirp_post_kernel(const double2* __restrict__ c, int n, int L, int rows,
                                  const double2* __restrict__ w, int inverse, double scale,
                                  double2* __restrict__ out) {
  const size_t total = (size_t)rows * n;
  for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < total; e += (size_t)gridDim.x * blockDim.x) {
    const size_t r = e / n;
    const int k = (int)(e - r * n);
    double2 v = cmul(w[k], c[r * L + k]);
    if (inverse) v = cconj(v);
    out[e] = cscale(v, scale);
  }
}

// the four-step transform of `rows` power-of-two sequences of length f.L
static bool r16_len(int len) { return len == 128 || len == 256; }
static bool big_r16_enabled() {
  static const bool on = [] {
    const char* e = getenv("APX_BIG_R16");
    return !(e && e[0] == '0');
  }();
  return on;
}

template <typename K>
static size_t r16_smem(K kern, int len) {
  const size_t bytes = (size_t)16 * (len + 1) * sizeof(double2);
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  return bytes;
}

template <typename TI, bool INV>
static void four_step_r16_launch(const BigFFT& f, const TI* in, double2* data, double2* out, int rr, double scale,
                                 cudaStream_t st) {
  const dim3 g1((unsigned)(f.n2 / 16), (unsigned)rr), g2((unsigned)(f.n1 / 16), (unsigned)rr);
  if (f.n1 == 128) {
    auto k = fft4_pass1_r16_kernel<TI, 8, INV>;
    k<<<g1, 256, r16_smem(k, 128), st>>>(in, f.n2, f.roots, f.roots1, data);
  } else {
    auto k = fft4_pass1_r16_kernel<TI, 16, INV>;
    k<<<g1, 256, r16_smem(k, 256), st>>>(in, f.n2, f.roots, f.roots1, data);
  }
  if (f.n2 == 128) {
    auto k = fft4_pass2_r16_kernel<8, INV>;
    k<<<g2, 256, r16_smem(k, 128), st>>>(data, f.n1, f.roots2, scale, out);
  } else {
    auto k = fft4_pass2_r16_kernel<16, INV>;
    k<<<g2, 256, r16_smem(k, 256), st>>>(data, f.n1, f.roots2, scale, out);
  }
}

template <typename TI>
static int four_step_rows(const BigFFT& f, const TI* in, double2* data, double2* out, int rows, bool inverse,
                          double scale, cudaStream_t st) {
  if (r16_len(f.n1) && r16_len(f.n2) && big_r16_enabled()) {
    const size_t L = (size_t)f.L;
    for (int r0 = 0; r0 < rows; r0 += 65535) {
      const int rr = std::min(65535, rows - r0);
      if (inverse) four_step_r16_launch<TI, true>(f, in + r0 * L, data + r0 * L, out + r0 * L, rr, scale, st);
      else four_step_r16_launch<TI, false>(f, in + r0 * L, data + r0 * L, out + r0 * L, rr, scale, st);
      APX_LAUNCH_CHECK();
    }
    return OK;
  }
  const size_t s1 = (size_t)kBigTile * (f.n1 + 1) * sizeof(double2), s2 = (size_t)kBigTile * (f.n2 + 1) * sizeof(double2);
  APX_CUDA(cudaFuncSetAttribute(fft4_pass1_kernel<TI>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)s1));
  APX_CUDA(cudaFuncSetAttribute(fft4_pass2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)s2));
  const size_t L = (size_t)f.L;
  for (int r0 = 0; r0 < rows; r0 += 65535) {
    const int rr = std::min(65535, rows - r0);
    fft4_pass1_kernel<TI><<<dim3((unsigned)(f.n2 / kBigTile), (unsigned)rr), kBigThreads, s1, st>>>(
        in + r0 * L, f.n1, f.n2, inverse ? 1 : 0, f.roots, f.roots1, data + r0 * L);
    APX_LAUNCH_CHECK();
    fft4_pass2_kernel<<<dim3((unsigned)(f.n1 / kBigTile), (unsigned)rr), kBigThreads, s2, st>>>(
        data + r0 * L, f.n1, f.n2, inverse ? 1 : 0, f.roots2, scale, out + r0 * L);
    APX_LAUNCH_CHECK();
  }
  return OK;
}

static int big_fft_init(const BigFFT& f, cudaStream_t st) {
  launch_roots(f.roots, f.L, st);
  launch_roots(f.roots1, f.n1, st);
  launch_roots(f.roots2, f.n2, st);
  APX_LAUNCH_CHECK();
  if (f.blue) {
    const unsigned g = (unsigned)std::min<int64_t>(ceil_div(f.L, 256), 1024);
    chirp_kernel<<<g, 256, 0, st>>>(f.chirp, f.n);
    APX_LAUNCH_CHECK();
    chirp_conv_kernel<<<g, 256, 0, st>>>(f.chirp, f.n, f.L, f.t1);
    APX_LAUNCH_CHECK();
    APX_TRY(four_step_rows<double2>(f, f.t1, f.t1, f.bf, 1, false, 1.0, st));
  }
  return OK;
}

// rows x n: in (TI) -> out (complex) via `data` (complex, may alias `in` but not `out`); scale
// multiplies the result
template <typename TI>
static int big_fft_rows(const BigFFT& f, const TI* in, double2* data, double2* out, int rows, bool inverse,
                        double scale, cudaStream_t st) {
  if (rows <= 0) return OK;
  if (!f.blue) return four_step_rows<TI>(f, in, data, out, rows, inverse, scale, st);
  const size_t n = (size_t)f.n;
  for (int r0 = 0; r0 < rows; r0 += f.chunk) {
    const int rr = std::min(f.chunk, rows - r0);
    const unsigned g = (unsigned)std::min<int64_t>(ceil_div((int64_t)rr * f.L, 256), kNumSMs * 16);
    chirp_pre_kernel<TI><<<g, 256, 0, st>>>(in + r0 * n, f.n, f.L, rr, f.chirp, inverse ? 1 : 0, f.t1);
    APX_LAUNCH_CHECK();
    APX_TRY(four_step_rows<double2>(f, f.t1, f.t1, f.t2, rr, false, 1.0, st));
    rows_mul_kernel<<<g, 256, 0, st>>>(f.t2, f.L, rr, f.bf);
    APX_LAUNCH_CHECK();
    APX_TRY(four_step_rows<double2>(f, f.t2, f.t2, f.t1, rr, true, 1.0 / f.L, st));
    chirp_post_kernel<<<g, 256, 0, st>>>(f.t1, f.n, f.L, rr, f.chirp, inverse ? 1 : 0, scale, out + r0 * n);
    APX_LAUNCH_CHECK();
  }
  return OK;
}

struct BigCircPlan {
  BigFFT f;
  double2* rootsn;  // exp(-2 pi i k / n): the on-the-fly Ahat (f.roots is for the length-L transforms)
  double2 *W1, *W2, *Ssel_a, *L_a, *Ssel_b, *L_b;
  double *part, *mag_a, *mag_b, *red;
  int groups;
};

static void plan_circ_big(Workspace& ws, BigCircPlan& p, int n, int k) {
  plan_big_fft(ws, p.f, n, n);
  p.rootsn = ws.take<double2>(n);
  p.W1 = ws.take<double2>((size_t)n * n);
  p.W2 = ws.take<double2>((size_t)n * n);
  const size_t kn = (size_t)std::max(k, 1) * n;
  p.Ssel_a = ws.take<double2>(kn);
  p.L_a = ws.take<double2>(kn);
  p.Ssel_b = ws.take<double2>(kn);
  p.L_b = ws.take<double2>(kn);
  p.groups = 64;
  p.part = ws.take<double>((size_t)p.groups * n);
  p.mag_a = ws.take<double>(n);
  p.mag_b = ws.take<double>(n);
  p.red = ws.take<double>(4 * kNumSMs + 64);
}

// S^T (unnormalised, in W2) and the magnitudes of X's circulant spectrum
template <typename T>
static int big_decompose(const T* X, int n, const BigCircPlan& p, double* mag, cudaStream_t st) {
  // the skewed copy: in W2 for the four-step path (pass 1 consumes it before pass 2 writes W2);
  // in W1 for Bluestein, which writes its output rows chunk by chunk while later rows are unread
  T* skew = reinterpret_cast<T*>(p.f.blue ? p.W1 : p.W2);
  circ_skew_kernel<T><<<dim3((unsigned)ceil_div(n, 32), (unsigned)ceil_div(n, 32)), 256, 0, st>>>(X, n, skew);
  APX_LAUNCH_CHECK();
  APX_TRY(big_fft_rows<T>(p.f, skew, p.W1, p.W2, n, false, 1.0, st));
  const int rpc = (int)ceil_div(n, p.groups);
  colsum_abs2_kernel<<<dim3((unsigned)ceil_div(n, 256), (unsigned)ceil_div(n, rpc)), 256, 0, st>>>(
      p.W2, n, rpc, 1.0 / ((double)n * n), p.part);
  APX_LAUNCH_CHECK();
  mag_finalize_kernel<<<(unsigned)ceil_div(n, 32), 256, 0, st>>>(p.part, (int)ceil_div(n, rpc), n, mag);
  APX_LAUNCH_CHECK();
  return OK;
}

// Ssel = selected rows of S (= columns of S^T / n), L = fft(Ssel)
static int big_spectra(int n, const BigCircPlan& p, const int* sel, int k, double2* Ssel, double2* L, cudaStream_t st) {
  if (k <= 0) return OK;
  gather_cols_kernel<<<dim3((unsigned)std::min<int64_t>(ceil_div(n, 256), 64), (unsigned)k), 256, 0, st>>>(
      p.W2, n, sel, 1.0 / n, Ssel);
  APX_LAUNCH_CHECK();
  return big_fft_rows<double2>(p.f, Ssel, p.W1, L, k, false, 1.0, st);
}

template <typename T>
static int run_circulant_big(const T* A, const T* B, int n, int k, int order, const int* fa, const int* fb, double2* M,
                             int* sa, int* sb, double* scal, const BigCircPlan& p, cudaStream_t st) {
  stage_mark(0, st);
  APX_CUDA(cudaMemsetAsync(scal, 0, APX_NSCALARS * sizeof(double), st));
  APX_TRY(big_fft_init(p.f, st));
  launch_roots(p.rootsn, n, st);
  APX_LAUNCH_CHECK();
  const double rs = 1.0 / sqrt((double)n);
  const dim3 gather_grid((unsigned)ceil_div(n, 256), (unsigned)ceil_div(n, kGatherRows));
  APX_TRY(big_decompose<T>(A, n, p, p.mag_a, st));
  if (fa) { if (k) APX_CUDA(cudaMemcpyAsync(sa, fa, k * sizeof(int), cudaMemcpyDeviceToDevice, st)); }
  else APX_TRY(launch_topk(p.mag_a, n, k, sa, st));
  APX_TRY(launch_kept_energy(p.mag_a, sa, k, (double)n, scal + APX_S_KEPT_A, st));
  APX_TRY(big_spectra(n, p, sa, k, p.Ssel_a, p.L_a, st));
  APX_TRY(big_decompose<T>(B, n, p, p.mag_b, st));
  if (fb) { if (k) APX_CUDA(cudaMemcpyAsync(sb, fb, k * sizeof(int), cudaMemcpyDeviceToDevice, st)); }
  else APX_TRY(launch_topk(p.mag_b, n, k, sb, st));
  APX_TRY(launch_kept_energy(p.mag_b, sb, k, (double)n, scal + APX_S_KEPT_B, st));
  APX_TRY(big_spectra(n, p, sb, k, p.Ssel_b, p.L_b, st));
  stage_mark(1, st);
  // term1 = Ahat . B, column-local: columns of B as rows of W1, FFT, gather with L_A, inverse FFT
  const dim3 tgrid((unsigned)ceil_div(n, 32), (unsigned)ceil_div(n, 32));
  transpose_to_c_kernel<T><<<tgrid, 256, 0, st>>>(B, n, p.W1);
  APX_LAUNCH_CHECK();
  APX_TRY(big_fft_rows<double2>(p.f, p.W1, p.W1, p.W2, n, false, 1.0, st));
  big_left_gather_kernel<<<gather_grid, 256, 0, st>>>(p.W2, n, p.L_a, sa, k, rs, p.W1);
  APX_LAUNCH_CHECK();
  APX_TRY(big_fft_rows<double2>(p.f, p.W1, p.W1, p.W2, n, true, 1.0, st));
  transpose_scale_c_kernel<<<tgrid, 256, 0, st>>>(p.W2, n, rs, M);
  APX_LAUNCH_CHECK();
  stage_mark(2, st);
  if (order == 1) {
    // term2 = dA . Bhat, row-local: conj(dA) rows, FFT, gather with conj(L_B), inverse FFT, conj
    APX_TRY(launch_big_dA<T>(A, n, p.Ssel_a, sa, k, p.rootsn, p.W1, 0, n, st));
    APX_TRY(big_fft_rows<double2>(p.f, p.W1, p.W1, p.W2, n, false, 1.0, st));
    big_right_gather_kernel<<<gather_grid, 256, 0, st>>>(p.W2, n, p.L_b, sb, k, rs, p.W1);
    APX_LAUNCH_CHECK();
    APX_TRY(big_fft_rows<double2>(p.f, p.W1, p.W1, p.W2, n, true, 1.0, st));
    acc_conj_kernel<<<kNumSMs * 8, 256, 0, st>>>(p.W2, (size_t)n * n, rs, M);
    APX_LAUNCH_CHECK();
  }
  stage_mark(3, st);
  int parts = 0;
  APX_TRY(launch_sumsq<double>(reinterpret_cast<const double*>(M), (size_t)2 * n * n, p.red, &parts, st));
  APX_TRY(launch_sum_vector(p.red, parts, scal + APX_S_FRO2_M, st));
  const size_t nel = (size_t)n * n * (sizeof(T) / sizeof(double));
  APX_TRY(launch_sumsq<double>(reinterpret_cast<const double*>(A), nel, p.red, &parts, st));
  APX_TRY(launch_sum_vector(p.red, parts, scal + APX_S_FRO2_A, st));
  APX_TRY(launch_sumsq<double>(reinterpret_cast<const double*>(B), nel, p.red, &parts, st));
  APX_TRY(launch_sum_vector(p.red, parts, scal + APX_S_FRO2_B, st));
  stage_mark(4, st);
  return OK;
}

}  // namespace apx

using namespace apx;

// ---- the circulant product sharded by rows of M ------------------------------
// Rank g holds both operands (replicated) and produces the rows R_g = [row0, row0 + m) of M.
// term1 (circulant.py:136-147) is column-local and term2 (:150-161) row-local, so:
//   1  decompose only the cycle blocks [blk0, blk1) of the full decomposition grid (cycle rows of
//      the skewed operand): per-CTA magnitude partials into their full-grid slots (zero-padded),
//      for A and B                                                  out: 2 x parts x n fp64
//   2  (partials summed over ranks) magnitudes exactly as on one device -> identical selections;
//      the selected spectrum rows from this rank's cycles (zero-padded)  out: 2 x k x n complex
//   3  (spectra summed = gathered) L = fft(S_t); term1 for the columns [col0, col0 + w) into the
//      n x w block T1, which the caller redistributes by rows (all-to-all) into M's rows
//   4  term2 for the rows R_g (dA rows from A's spectra), accumulated onto M's rows;
//                                                                   out: [||M_g||^2]
// Every per-column / per-row computation is the single-device kernel on the same inputs, so the
// rows of M are bitwise the single-device product's.
__global__ void circ_sel_extract_kernel(const double2* __restrict__ St, int n, int j_lo, int j_hi,
                                        const int* __restrict__ sel, int k, double2* __restrict__ out) {
  const size_t total = (size_t)k * n;
  for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < total; e += (size_t)gridDim.x * blockDim.x) {
    const int q = (int)(e / n), j = (int)(e % n);
    APX_DCHECK(sel[q] >= 0 && sel[q] < n);
    out[e] = (j >= j_lo && j < j_hi) ? St[(size_t)(j - j_lo) * n + sel[q]] : make_double2(0.0, 0.0);
  }
}

struct CircRowsPlan {
  double2 *roots, *St_a, *St_b, *Ssel_a, *L_a, *Ssel_b, *L_b, *Xpre;
  double *mag_a, *mag_b, *red;
  void* skew;
  int cpc, parts, j_lo, j_hi;
};

static void circ_grid(int n, int* cpc, int* parts) {
  *cpc = std::max(1, (int)ceil_div(n, 2 * kNumSMs));
  *parts = (int)ceil_div(n, *cpc);
}

static void plan_circ_rows(Workspace& ws, CircRowsPlan& p, int elem, int n, int k, int m, int blk0, int blk1) {
  circ_grid(n, &p.cpc, &p.parts);
  p.j_lo = std::min(n, blk0 * p.cpc);
  p.j_hi = std::min(n, blk1 * p.cpc);
  const size_t jr = (size_t)std::max(1, p.j_hi - p.j_lo);
  p.roots = ws.take<double2>(n);
  p.St_a = ws.take<double2>(jr * n);
  p.St_b = ws.take<double2>(jr * n);
  p.skew = ws.take<char>(jr * n * elem);
  p.Ssel_a = ws.take<double2>((size_t)std::max(k, 1) * n);
  p.L_a = ws.take<double2>((size_t)std::max(k, 1) * n);
  p.Ssel_b = ws.take<double2>((size_t)std::max(k, 1) * n);
  p.L_b = ws.take<double2>((size_t)std::max(k, 1) * n);
  p.Xpre = ws.take<double2>((size_t)std::max(m, 1) * n);
  p.mag_a = ws.take<double>(n);
  p.mag_b = ws.take<double>(n);
  p.red = ws.take<double>(4 * kNumSMs + 64);
}

template <typename T>
static int run_circ_rows_phase(int phase, const T* A, const T* B, int n, int k, int order, int row0, int m, int col0,
                               int w, int blk0, int blk1, double2* M_rows, double2* T1, int* sa, int* sb,
                               const double* red_in, double* red_out, double* scal, const CircRowsPlan& p,
                               cudaStream_t st) {
  const size_t smem2 = fft_smem_bytes(n, 2) + (size_t)2 * k * sizeof(int);
  if (phase == 1) {
    APX_CUDA(cudaMemsetAsync(scal, 0, APX_NSCALARS * sizeof(double), st));
    launch_roots(p.roots, n, st);
    APX_LAUNCH_CHECK();
    APX_CUDA(cudaMemsetAsync(red_out, 0, (size_t)2 * p.parts * n * sizeof(double), st));
    const T* ops[2] = {A, B};
    double2* Sts[2] = {p.St_a, p.St_b};
    const size_t smem = fft_smem_bytes(n, 1) + (size_t)n * sizeof(double);
    auto fn = circ_decompose_rows_kernel<T>;
    APX_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    for (int o = 0; o < 2; ++o) {
      if (p.j_hi > p.j_lo) {
        const int direct = decompose_direct<T>(n);
        if (!direct) {
          circ_skew_kernel<T><<<dim3((unsigned)ceil_div(n, 32), (unsigned)ceil_div(p.j_hi - p.j_lo, 32)), 256, 0,
                                st>>>(ops[o], n, (T*)p.skew, p.j_lo, p.j_hi);
          APX_LAUNCH_CHECK();
        }
        APX_TRY(launch_decompose_rows<T>(direct ? ops[o] : (const T*)p.skew, n, p.cpc, p.roots, Sts[o],
                                         red_out + (size_t)o * p.parts * n, blk1 - blk0, blk0, p.j_lo, direct, st));
      }
    }
    int parts = 0;
    const size_t nel = (size_t)n * n * (sizeof(T) / sizeof(double));
    APX_TRY(launch_sumsq<double>(reinterpret_cast<const double*>(A), nel, p.red, &parts, st));
    APX_TRY(launch_sum_vector(p.red, parts, scal + APX_S_FRO2_A, st));
    APX_TRY(launch_sumsq<double>(reinterpret_cast<const double*>(B), nel, p.red, &parts, st));
    APX_TRY(launch_sum_vector(p.red, parts, scal + APX_S_FRO2_B, st));
    return OK;
  }
  if (phase == 2) {
    double* mags[2] = {p.mag_a, p.mag_b};
    int* sels[2] = {sa, sb};
    double2* Sts[2] = {p.St_a, p.St_b};
    double2* out = reinterpret_cast<double2*>(red_out);
    for (int o = 0; o < 2; ++o) {
      mag_finalize_kernel<<<(unsigned)ceil_div(n, 32), 256, 0, st>>>(red_in + (size_t)o * p.parts * n, p.parts, n,
                                                                      mags[o]);
      APX_LAUNCH_CHECK();
      APX_TRY(launch_topk(mags[o], n, k, sels[o], st));
      APX_TRY(launch_kept_energy(mags[o], sels[o], k, (double)n, scal + (o ? APX_S_KEPT_B : APX_S_KEPT_A), st));
      if (k > 0) {
        circ_sel_extract_kernel<<<(unsigned)std::min<int64_t>(ceil_div((int64_t)k * n, 256), kNumSMs * 8), 256, 0,
                                  st>>>(Sts[o], n, p.j_lo, p.j_hi, sels[o], k, out + (size_t)o * k * n);
        APX_LAUNCH_CHECK();
      }
    }
    return OK;
  }
  if (phase == 3) {
    const double2* in = reinterpret_cast<const double2*>(red_in);
    if (k > 0) {
      APX_CUDA(cudaMemcpyAsync(p.Ssel_a, in, (size_t)k * n * sizeof(double2), cudaMemcpyDeviceToDevice, st));
      APX_CUDA(cudaMemcpyAsync(p.Ssel_b, in + (size_t)k * n, (size_t)k * n * sizeof(double2), cudaMemcpyDeviceToDevice,
                               st));
      const size_t smem = fft_smem_bytes(n, 1);
      APX_CUDA(cudaFuncSetAttribute(circ_spectra_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      circ_spectra_kernel<<<k, 512, smem, st>>>(p.Ssel_a, n, sa, p.roots, nullptr, p.L_a, 1, 1.0 / n);
      APX_LAUNCH_CHECK();
      circ_spectra_kernel<<<k, 512, smem, st>>>(p.Ssel_b, n, sb, p.roots, nullptr, p.L_b, 1, 1.0 / n);
      APX_LAUNCH_CHECK();
    }
    if (w > 0) {
      static const bool r16_off = getenv("APX_CIRC_R16") != nullptr && atoi(getenv("APX_CIRC_R16")) == 0;
      if (std::is_same<T, double>::value && n == 4096 && !r16_off) {  // the single-device kernel
        const size_t smem2r = (size_t)2 * kFFT16Buf * sizeof(double2) + (size_t)k * sizeof(int);
        APX_CUDA(cudaFuncSetAttribute(circ_left2_r16_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem2r));
        circ_left2_r16_kernel<<<(unsigned)ceil_div(w, 2), 512, smem2r, st>>>(reinterpret_cast<const double*>(B), p.L_a,
                                                                             sa, k, p.roots, T1, col0, col0 + w,
                                                                             (int64_t)w);
        APX_LAUNCH_CHECK();
        return OK;
      }
      auto fn = circ_left2_kernel<T>;
      APX_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem2));
      const int stage_l = left2_stage_l(n, k);
      const size_t smem_l = smem2 + (stage_l ? left2_stage_bytes(n) : 0);
      APX_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_l));
      fn<<<(unsigned)ceil_div(w, 2), 512, smem_l, st>>>(B, n, p.L_a, sa, k, p.roots, T1, col0, col0 + w, (int64_t)w,
                                                        stage_l);
      APX_LAUNCH_CHECK();
    }
    return OK;
  }
  // phase 4: term2 on this rank's rows (M_rows holds term1's rows, assembled by the caller)
  if (order == 1 && m > 0) {
    APX_TRY(launch_big_dA<T>(A, n, p.Ssel_a, sa, k, p.roots, p.Xpre, row0, row0 + m, st));
    static const bool r16_off = getenv("APX_CIRC_R16") != nullptr && atoi(getenv("APX_CIRC_R16")) == 0;
    if (p.Xpre != nullptr && n == 4096 && !r16_off) {  // the single-device kernel
      const size_t smem2r = (size_t)2 * kFFT16Buf * sizeof(double2) + (size_t)k * sizeof(int);
      APX_CUDA(cudaFuncSetAttribute(circ_right2_r16_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem2r));
      circ_right2_r16_kernel<<<(unsigned)ceil_div(m, 2), 512, smem2r, st>>>(p.Xpre, p.L_b, sb, k, p.roots, M_rows,
                                                                            (double*)nullptr, row0, row0 + m);
    } else {
      auto fn = circ_right2_kernel<T>;
      APX_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem2));
      fn<<<(unsigned)ceil_div(m, 2), 512, smem2, st>>>(A, n, p.Ssel_a, sa, k, p.L_b, sb, k, p.roots, M_rows, p.Xpre,
                                                       row0, row0 + m, right2_linear(), (double*)nullptr);
    }
    APX_LAUNCH_CHECK();
  }
  int parts = 0;
  APX_TRY(launch_sumsq<double>(reinterpret_cast<const double*>(M_rows), (size_t)2 * m * n, p.red, &parts, st));
  APX_TRY(launch_sum_vector(p.red, parts, red_out, st));
  return OK;
}

extern "C" {

// The decomposition grid the sharded product partitions ([blk0, blk1) per rank): parts CTA blocks
// of cpc cycles each (the single-device grid).
int apx_circulant_rows_grid(int64_t n, int64_t* parts, int64_t* cpc) {
  APX_REQUIRE(n >= 1, "n must be >= 1");
  int c = 0, q = 0;
  circ_grid((int)n, &c, &q);
  *parts = q;
  *cpc = c;
  return OK;
}

size_t apx_circulant_rows_workspace(int dtype, int64_t n, int k, int64_t m_rows, int64_t blk0, int64_t blk1) {
  Workspace ws(nullptr, 0, true);
  CircRowsPlan p;
  plan_circ_rows(ws, p, dtype == C128 ? 16 : 8, (int)n, k, (int)m_rows, (int)blk0, (int)blk1);
  return ws.off;
}

int apx_circulant_rows_phase(int phase, int dtype, const void* A, const void* B, int64_t n, int k, int order,
                             int64_t row0, int64_t m_rows, int64_t col0, int64_t w_cols, int64_t blk0, int64_t blk1,
                             void* M_rows, void* T1, int32_t* sel_a, int32_t* sel_b, const double* red_in,
                             double* red_out, double* scalars, void* wsp, size_t ws_bytes, void* stream) {
  APX_NVTX("apx_circulant_rows_phase");
  APX_REQUIRE(phase >= 1 && phase <= 4, "phase must be 1..4");
  APX_REQUIRE(dtype == F64 || dtype == C128, "circulant product: fp64 or complex128 inputs");
  APX_REQUIRE(k >= 0 && k <= n, "k=%d out of range [0, %lld]", k, (long long)n);
  APX_REQUIRE(order == 0 || order == 1, "order must be 0 or 1");
  APX_REQUIRE(n >= kDaRows && n <= kPP * 512 && circ_fused_fits((int)n, k),
              "sharded circulant product: n=%lld outside the fused shared-memory range [%d, %d]", (long long)n,
              kDaRows, kPP * 512);
  APX_REQUIRE(row0 >= 0 && m_rows >= 0 && row0 + m_rows <= n && (row0 % 2) == 0, "row block [%lld, %lld) invalid",
              (long long)row0, (long long)(row0 + m_rows));
  APX_REQUIRE(col0 >= 0 && w_cols >= 0 && col0 + w_cols <= n && (col0 % 2) == 0, "column block invalid");
  int cpc = 0, parts = 0;
  circ_grid((int)n, &cpc, &parts);
  APX_REQUIRE(blk0 >= 0 && blk0 <= blk1 && blk1 <= parts, "cycle blocks [%lld, %lld) outside [0, %d)",
              (long long)blk0, (long long)blk1, parts);
  APX_REQUIRE(phase == 1 || red_in != nullptr || phase == 4, "phase %d needs the summed exchange", phase);
  Workspace ws(wsp, ws_bytes);
  CircRowsPlan p;
  plan_circ_rows(ws, p, dtype == C128 ? 16 : 8, (int)n, k, (int)m_rows, (int)blk0, (int)blk1);
  APX_WS_CHECK(ws);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (dtype == F64)
    return run_circ_rows_phase<double>(phase, (const double*)A, (const double*)B, (int)n, k, order, (int)row0,
                                       (int)m_rows, (int)col0, (int)w_cols, (int)blk0, (int)blk1, (double2*)M_rows,
                                       (double2*)T1, sel_a, sel_b, red_in, red_out, scalars, p, st);
  return run_circ_rows_phase<double2>(phase, (const double2*)A, (const double2*)B, (int)n, k, order, (int)row0,
                                      (int)m_rows, (int)col0, (int)w_cols, (int)blk0, (int)blk1, (double2*)M_rows,
                                      (double2*)T1, sel_a, sel_b, red_in, red_out, scalars, p, st);
}

size_t apx_circulant_first_order_workspace(int dtype, int64_t n, int k, int order) {
  (void)dtype;
  (void)order;
  Workspace ws(nullptr, 0, true);
  if (!circ_fused_fits((int)n, k) && big_fft_ok(n)) {
    BigCircPlan b;
    plan_circ_big(ws, b, (int)n, k);
    return ws.off;
  }
  CircPlan p;
  plan_circ(ws, p, (int)n, k, false);
  return ws.off;
}

int apx_circulant_first_order(int dtype, const void* A, const void* B, int64_t n, int k, int order,
                              const int32_t* force_sel_a, const int32_t* force_sel_b, void* M, int32_t* sel_a,
                              int32_t* sel_b, double* scalars, void* wsp, size_t ws_bytes, void* stream) {
  APX_NVTX("apx_circulant_first_order");
  APX_REQUIRE(dtype == F64 || dtype == C128, "circulant product: fp64 or complex128 inputs");
  APX_REQUIRE(k >= 0 && k <= n, "k=%d out of range [0, %lld]", k, (long long)n);
  APX_REQUIRE(order == 0 || order == 1, "order must be 0 or 1");
  APX_REQUIRE(n >= 1 && (circ_fused_fits((int)n, k) || big_fft_ok(n)),
              "n=%lld: beyond the shared-memory transforms only powers of two up to 2^18 are supported",
              (long long)n);
  Workspace ws(wsp, ws_bytes);
  if (!circ_fused_fits((int)n, k)) {
    BigCircPlan b;
    plan_circ_big(ws, b, (int)n, k);
    APX_WS_CHECK(ws);
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    if (dtype == F64)
      return run_circulant_big<double>((const double*)A, (const double*)B, (int)n, k, order, force_sel_a, force_sel_b,
                                       (double2*)M, sel_a, sel_b, scalars, b, st);
    return run_circulant_big<double2>((const double2*)A, (const double2*)B, (int)n, k, order, force_sel_a,
                                      force_sel_b, (double2*)M, sel_a, sel_b, scalars, b, st);
  }
  CircPlan p;
  plan_circ(ws, p, (int)n, k, false);
  APX_WS_CHECK(ws);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (dtype == F64)
    return run_circulant<double>((const double*)A, (const double*)B, (int)n, k, order, force_sel_a, force_sel_b,
                                 (double2*)M, sel_a, sel_b, scalars, p, st);
  return run_circulant<double2>((const double2*)A, (const double2*)B, (int)n, k, order, force_sel_a, force_sel_b,
                                (double2*)M, sel_a, sel_b, scalars, p, st);
}

static bool decompose_fits(int64_t n) {
  return !force_big(n) && fft_smem_bytes((int)n, 1) + (size_t)n * 8 <= 227 * 1024;
}

size_t apx_circulant_decompose_workspace(int dtype, int64_t n) {
  Workspace ws(nullptr, 0, true);
  if (!decompose_fits(n) && big_fft_ok(n)) {
    BigCircPlan b;
    plan_circ_big(ws, b, (int)n, 0);
    return ws.off;
  }
  ws.take<double2>(n);
  ws.take<double>((size_t)ceil_div(n, std::max(1, (int)ceil_div(n, 2 * kNumSMs))) * n);
  ws.take<double2>((size_t)n * n);                                  // S^T
  ws.take<char>((size_t)n * n * (dtype == C128 ? 16 : 8));           // skewed copy of A
  return ws.off;
}

int apx_circulant_decompose(int dtype, const void* A, int64_t n, void* columns, double* magnitudes, void* wsp,
                            size_t ws_bytes, void* stream) {
  APX_NVTX("apx_circulant_decompose");
  APX_REQUIRE(dtype == F64 || dtype == C128, "circulant_decompose: fp64 or complex128 input");
  APX_REQUIRE(n >= 1 && (decompose_fits(n) || big_fft_ok(n)),
              "n=%lld: beyond the shared-memory transforms only powers of two up to 2^18 are supported",
              (long long)n);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  Workspace ws(wsp, ws_bytes);
  if (!decompose_fits(n)) {
    BigCircPlan b;
    plan_circ_big(ws, b, (int)n, 0);
    APX_WS_CHECK(ws);
    APX_TRY(big_fft_init(b.f, st));
    if (dtype == F64) APX_TRY(big_decompose<double>((const double*)A, (int)n, b, magnitudes, st));
    else APX_TRY(big_decompose<double2>((const double2*)A, (int)n, b, magnitudes, st));
    transpose_scale_c_kernel<<<dim3((unsigned)ceil_div(n, 32), (unsigned)ceil_div(n, 32)), 256, 0, st>>>(b.W2, (int)n, 1.0 / n,
                                                                                           (double2*)columns);
    APX_LAUNCH_CHECK();
    return OK;
  }
  CircPlan p{};
  p.cpc = std::max(1, (int)ceil_div(n, 2 * kNumSMs));
  p.parts = (int)ceil_div(n, p.cpc);
  p.roots = ws.take<double2>(n);
  p.part = ws.take<double>((size_t)p.parts * n);
  double2* St = ws.take<double2>((size_t)n * n);
  void* skew = ws.take<char>((size_t)n * n * (dtype == C128 ? 16 : 8));
  APX_WS_CHECK(ws);
  launch_roots(p.roots, (int)n, st);
  APX_LAUNCH_CHECK();
  if (dtype == F64)
    APX_TRY(circ_decompose_run<double>((const double*)A, (int)n, p, St, magnitudes, (double*)skew, st));
  else
    APX_TRY(circ_decompose_run<double2>((const double2*)A, (int)n, p, St, magnitudes, (double2*)skew, st));
  return launch_transpose_c128(St, n, (int)n, (int)n, (double2*)columns, n, st);
}

size_t apx_circulant_materialize_workspace(int64_t n) {
  Workspace ws(nullptr, 0, true);
  ws.take<double2>(n);
  return ws.off;
}

// out (n x n complex) = sum_q R_{sel[q]} D^{sel[q]} from the selected first columns Ssel (k x n)
int apx_circulant_materialize(const void* Ssel, const int32_t* sel, int k, int64_t n, void* out, void* wsp,
                              size_t ws_bytes, void* stream) {
  APX_REQUIRE(n >= 1 && k >= 0 && k <= n, "bad materialize arguments");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  Workspace ws(wsp, ws_bytes);
  double2* roots = ws.take<double2>(n);
  APX_WS_CHECK(ws);
  launch_roots(roots, (int)n, st);
  APX_LAUNCH_CHECK();
  circ_materialize_kernel<<<kNumSMs * 4, 256, 0, st>>>((const double2*)Ssel, sel, k, (int)n, roots, (double2*)out);
  APX_LAUNCH_CHECK();
  return OK;
}

int apx_circulant_component(int dtype, const void* A, int64_t n, int kk, void* out, void* wsp, size_t ws_bytes,
                            void* stream) {
  APX_REQUIRE(dtype == F64 || dtype == C128, "circulant_component: fp64 or complex128 input");
  APX_REQUIRE(kk >= 0 && kk < n, "component index %d out of range [0, %lld)", kk, (long long)n);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  Workspace ws(wsp, ws_bytes);
  double2* roots = ws.take<double2>(n);
  APX_WS_CHECK(ws);
  launch_roots(roots, (int)n, st);
  APX_LAUNCH_CHECK();
  const unsigned blocks = (unsigned)ceil_div(n, 128);
  if (dtype == F64) circ_component_kernel<double><<<blocks, 128, 0, st>>>((const double*)A, (int)n, kk, roots, (double2*)out);
  else circ_component_kernel<double2><<<blocks, 128, 0, st>>>((const double2*)A, (int)n, kk, roots, (double2*)out);
  APX_LAUNCH_CHECK();
  return OK;
}

static bool dft_fits(int64_t n) { return !force_big(n) && fft_smem_bytes((int)n, 1) <= 227 * 1024; }

__global__ void strided_to_rows_kernel(const double2* __restrict__ x, int64_t stride, int64_t dist, int n,
                                       size_t count, double2* __restrict__ rows) {
  for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < count; e += (size_t)gridDim.x * blockDim.x) {
    const size_t b = e / n, i = e - b * n;
    rows[e] = x[b * dist + i * stride];
  }
}
__global__ void rows_to_strided_kernel(const double2* __restrict__ rows, int64_t stride, int64_t dist, int n,
                                       size_t count, double2* __restrict__ y) {
  for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < count; e += (size_t)gridDim.x * blockDim.x) {
    const size_t b = e / n, i = e - b * n;
    y[b * dist + i * stride] = rows[e];
  }
}

size_t apx_unitary_dft_workspace(int64_t n, int64_t batch) {
  Workspace ws(nullptr, 0, true);
  if (!dft_fits(n) && big_fft_ok(n)) {
    BigFFT f;
    plan_big_fft(ws, f, (int)n, (int)std::min<int64_t>(batch, 1 << 30));
    ws.take<double2>((size_t)std::max<int64_t>(batch, 1) * n);
    ws.take<double2>((size_t)std::max<int64_t>(batch, 1) * n);
    return ws.off;
  }
  ws.take<double2>(n);
  return ws.off;
}

// unitary_dft (core.py:82-97): `batch` complex128 vectors of length n, element i of vector b at
// x[b*dist + i*stride]; forward applies W (e^{-2 pi i pq/n}/sqrt(n)), inverse W*.
int apx_unitary_dft(const void* x, void* y, int64_t n, int64_t batch, int64_t stride, int64_t dist, int inverse,
                    void* wsp, size_t ws_bytes, void* stream) {
  APX_NVTX("apx_unitary_dft");
  APX_REQUIRE(n >= 1, "transform length must be >= 1");
  APX_REQUIRE(dft_fits(n) || big_fft_ok(n),
              "transform length %lld: beyond shared memory only powers of two up to 2^18 are supported",
              (long long)n);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  Workspace ws(wsp, ws_bytes);
  if (!dft_fits(n)) {
    BigFFT f;
    plan_big_fft(ws, f, (int)n, (int)std::min<int64_t>(batch, 1 << 30));
    double2* t1 = ws.take<double2>((size_t)std::max<int64_t>(batch, 1) * n);
    double2* t2 = ws.take<double2>((size_t)std::max<int64_t>(batch, 1) * n);
    APX_WS_CHECK(ws);
    if (batch == 0) return OK;
    APX_TRY(big_fft_init(f, st));
    const size_t count = (size_t)batch * n;
    const unsigned blocks = (unsigned)std::min<int64_t>(ceil_div((int64_t)count, 256), kNumSMs * 16);
    const double2* src = (const double2*)x;
    const bool contiguous = stride == 1 && dist == n;
    if (!contiguous) {
      strided_to_rows_kernel<<<blocks, 256, 0, st>>>(src, stride, dist, (int)n, count, t2);
      APX_LAUNCH_CHECK();
      src = t2;
    }
    for (int64_t b0 = 0; b0 < batch; b0 += 65535) {
      const int rows = (int)std::min<int64_t>(65535, batch - b0);
      double2* outp = contiguous ? (double2*)y + b0 * n : t2 + b0 * n;
      APX_TRY(big_fft_rows<double2>(f, src + b0 * n, t1 + b0 * n, outp, rows, inverse != 0, 1.0 / sqrt((double)n),
                                    st));
    }
    if (!contiguous) {
      rows_to_strided_kernel<<<blocks, 256, 0, st>>>(t2, stride, dist, (int)n, count, (double2*)y);
      APX_LAUNCH_CHECK();
    }
    return OK;
  }
  double2* roots = ws.take<double2>(n);
  APX_WS_CHECK(ws);
  if (batch == 0) return OK;
  launch_roots(roots, (int)n, st);
  APX_LAUNCH_CHECK();
  const size_t smem = fft_smem_bytes((int)n, 1);
  APX_CUDA(cudaFuncSetAttribute(dft_batch_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  dft_batch_kernel<<<(unsigned)batch, 512, smem, st>>>((const double2*)x, stride, dist, (int)n, inverse,
                                                       1.0 / sqrt((double)n), roots, (double2*)y);
  APX_LAUNCH_CHECK();
  return OK;
}

// cycle_reorder / cycle_reorder_inverse (core.py:106-137). mode: 0 reorder right, 1 reorder left,
// 2 inverse right, 3 inverse left. elem_bytes 8 (fp64) or 16 (complex128).
int apx_cycle_layout(int elem_bytes, const void* in, int64_t n, int mode, void* out, void* stream) {
  APX_REQUIRE(n >= 1 && mode >= 0 && mode <= 3, "bad cycle layout arguments");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const unsigned blocks = (unsigned)std::min<int64_t>(ceil_div(n * n, 256), kNumSMs * 8);
  if (elem_bytes == 8) cycle_layout_kernel<double><<<blocks, 256, 0, st>>>((const double*)in, (int)n, mode, (double*)out);
  else cycle_layout_kernel<double2><<<blocks, 256, 0, st>>>((const double2*)in, (int)n, mode, (double2*)out);
  APX_LAUNCH_CHECK();
  return OK;
}

// apply_cycle_power (core.py:140-154): side 0 = C^k M (rows down by k), 1 = M C^k (cols left by k)
int apx_apply_cycle_power(int elem_bytes, const void* in, int64_t rows, int64_t cols, int64_t k, int side, void* out,
                          void* stream) {
  const int64_t lim = side == 0 ? rows : cols;
  APX_REQUIRE(k >= 0 && k < lim, "k=%lld out of range [0, %lld)", (long long)k, (long long)lim);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const unsigned blocks = (unsigned)std::min<int64_t>(ceil_div(rows * cols, 256), kNumSMs * 8);
  if (elem_bytes == 8)
    cycle_power_kernel<double><<<blocks, 256, 0, st>>>((const double*)in, (int)rows, (int)cols, (int)k, side, (double*)out);
  else
    cycle_power_kernel<double2><<<blocks, 256, 0, st>>>((const double2*)in, (int)rows, (int)cols, (int)k, side,
                                                        (double2*)out);
  APX_LAUNCH_CHECK();
  return OK;
}

}  // extern "C"
