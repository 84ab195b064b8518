// Thin QR of the n x l sketch (K13; reference qr_decompose svd.py:63-69 -> LAPACK geqrf/orgqr).
//
// Fast path: CholeskyQR2 in fp64 -- Gram G = Y^T Y (row-chunk partials + fixed-order reduce),
// one-CTA Cholesky + triangular inverse, Q = Y R^{-1}, all twice. Any pivot below
// 4*l*eps*max(diag G) raises a device flag; the Householder kernel (one CTA, fp64, same
// reflector convention as LAPACK dlarfg: x -> -sign(x0)||x|| e1, H = I for a zero tail) then
// recomputes Q from Y, so rank-deficient sketches (zero / rank-1 test matrices,
// test_svd.py:56-77) still yield an orthonormal Q. Everything is asynchronous: the flag is
// read on the device, never by the host.
//
// Inputs and outputs take explicit (row, col) strides, so Z^T views (power iterations,
// Q^T outputs) need no transposition pass.
#include "common.cuh"
#include "kernels.cuh"

namespace apx {

// Q output: plain conversion, or (tf32) rounded to the nearest TF32-representable fp32 value --
// the TF32 tensor-core paths then read Q exactly (the tensor core itself would truncate it).
template <typename TO>
__device__ __forceinline__ TO qout(double v, int tf32) {
  if constexpr (std::is_same<TO, float>::value) {
    float f = (float)v;
    if (tf32) f = __uint_as_float((__float_as_uint(f) + 0x1000u) & 0xffffe000u);
    return f;
  } else {
    return (TO)v;
  }
}

constexpr int kMaxL = 128;               // CholeskyQR2 fast path
constexpr int kMaxHouseholderL = 12288;  // Householder: s_dot / s_tau in dynamic shared memory

// ---- 64-row tile of a strided n x l matrix (l <= 64) into shared memory as fp64 -------------
// Each of the 256 threads owns 16 elements; all 16 loads are issued before the first store, so a
// CTA waits for one memory latency instead of sixteen. Elements past m rows / l columns are 0.
// The element order follows the contiguous dimension (cs == 1: columns, else rows) so the loads
// coalesce; T_[i][r] (TRANSPOSED) or T_[r][i] layout, row pitch 66 (16-byte aligned rows).
constexpr int kTP = 66;
constexpr size_t kApplySmem = 2 * 64 * kTP * sizeof(double);
template <bool TRANSPOSED, typename T>
__device__ __forceinline__ void load_tile64(const T* __restrict__ Y, int64_t rs, int64_t cs, int m, int l, int r0,
                                            double (*Ts)[kTP]) {
  const int tid = threadIdx.x;
  const bool col_fast = cs == 1;
  T v[16];
#pragma unroll
  for (int u = 0; u < 16; ++u) {
    const int e = tid + 256 * u;
    const int r = col_fast ? (e >> 6) : (e & 63), i = col_fast ? (e & 63) : (e >> 6);
    v[u] = (r0 + r < m && i < l) ? Y[(size_t)(r0 + r) * rs + (size_t)i * cs] : T(0);
  }
#pragma unroll
  for (int u = 0; u < 16; ++u) {
    const int e = tid + 256 * u;
    const int r = col_fast ? (e >> 6) : (e & 63), i = col_fast ? (e & 63) : (e >> 6);
    if (TRANSPOSED)
      Ts[i][r] = (double)v[u];
    else
      Ts[r][i] = (double)v[u];
  }
}

// ---- Gram partials: G_p = Y[rows_p]^T Y[rows_p] over 64-row tiles (fp64) ---------------------
// 256 threads on a 16 x 16 grid of 4 x 4 blocks of the (padded) 64 x 64 Gram matrix; each row
// of the tile costs two 16-byte loads per operand and 16 FMAs. The full l x l block is written.
template <typename T>
__global__ void __launch_bounds__(256) gram_partial_kernel(const T* __restrict__ Y, int64_t rs, int64_t cs, int m,
                                                           int l, const int* __restrict__ skip,
                                                           double* __restrict__ part) {
  pdl_trigger();  // programmatic dependent launch: the next QR stage may start launching
  pdl_wait();
  if (skip && *skip) return;
  __shared__ __align__(16) double Ys[64][kTP];  // [r][i]
  load_tile64<false>(Y, rs, cs, m, l, blockIdx.x * 64, Ys);
  __syncthreads();
  const int bi = (threadIdx.x >> 4) * 4, bj = (threadIdx.x & 15) * 4;
  double acc[4][4];
#pragma unroll
  for (int x = 0; x < 4; ++x)
#pragma unroll
    for (int y = 0; y < 4; ++y) acc[x][y] = 0.0;
#pragma unroll 8
  for (int r = 0; r < 64; ++r) {
    const double2 a01 = *reinterpret_cast<const double2*>(&Ys[r][bi]);
    const double2 a23 = *reinterpret_cast<const double2*>(&Ys[r][bi + 2]);
    const double2 b01 = *reinterpret_cast<const double2*>(&Ys[r][bj]);
    const double2 b23 = *reinterpret_cast<const double2*>(&Ys[r][bj + 2]);
    const double av[4] = {a01.x, a01.y, a23.x, a23.y}, bv[4] = {b01.x, b01.y, b23.x, b23.y};
#pragma unroll
    for (int x = 0; x < 4; ++x)
#pragma unroll
      for (int y = 0; y < 4; ++y) acc[x][y] = fma(av[x], bv[y], acc[x][y]);
  }
  double* out = part + (size_t)blockIdx.x * l * l;
#pragma unroll
  for (int x = 0; x < 4; ++x)
#pragma unroll
    for (int y = 0; y < 4; ++y) {
      const int i = bi + x, j = bj + y;
      if (i < l && j < l) out[i * l + j] = acc[x][y];
    }
}

// ---- Gram partials for 64 < l <= 128: G_p = Y[rows_p]^T Y[rows_p] ----------------------------
// 64 rows per CTA staged as fp64 in shared memory; thread t owns a 4x4 block (bi, bj) of G
// (upper block triangle only), so each pair of 4-wide row loads feeds 16 FMAs.
template <typename T>
__global__ void __launch_bounds__(256) gram_partial_wide_kernel(const T* __restrict__ Y, int64_t rs, int64_t cs, int m,
                                                           int l, int rows_per, const int* __restrict__ skip,
                                                           double* __restrict__ part) {
  pdl_trigger();  // programmatic dependent launch: the next QR stage may start launching
  pdl_wait();
  if (skip && *skip) return;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* Ys = reinterpret_cast<double*>(smem_raw);  // rows_per x LP
  const int LP = (int)ceil_div(l, 4) * 4 + 4;          // padded row (multiple of 4 plus skew)
  const int r0 = blockIdx.x * rows_per;
  const int rows = min(rows_per, m - r0);
  for (int e = threadIdx.x; e < rows_per * LP; e += blockDim.x) {
    const int r = e / LP, c = e - r * LP;
    Ys[e] = (r < rows && c < l) ? (double)Y[(size_t)(r0 + r) * rs + (size_t)c * cs] : 0.0;
  }
  __syncthreads();
  double* out = part + (size_t)blockIdx.x * l * l;
  const int nb = (int)ceil_div(l, 4);
  for (int blk = threadIdx.x; blk < nb * nb; blk += blockDim.x) {
    const int bi = blk / nb, bj = blk - bi * nb;
    double acc[4][4];
#pragma unroll
    for (int x = 0; x < 4; ++x)
#pragma unroll
      for (int y = 0; y < 4; ++y) acc[x][y] = 0.0;
    if (bi <= bj) {
      for (int r = 0; r < rows; ++r) {
        const double* yr = Ys + r * LP;
        const double2 a01 = *reinterpret_cast<const double2*>(yr + 4 * bi);
        const double2 a23 = *reinterpret_cast<const double2*>(yr + 4 * bi + 2);
        const double2 b01 = *reinterpret_cast<const double2*>(yr + 4 * bj);
        const double2 b23 = *reinterpret_cast<const double2*>(yr + 4 * bj + 2);
        const double av[4] = {a01.x, a01.y, a23.x, a23.y}, bv[4] = {b01.x, b01.y, b23.x, b23.y};
#pragma unroll
        for (int x = 0; x < 4; ++x)
#pragma unroll
          for (int y = 0; y < 4; ++y) acc[x][y] = fma(av[x], bv[y], acc[x][y]);
      }
    }
#pragma unroll
    for (int x = 0; x < 4; ++x)
#pragma unroll
      for (int y = 0; y < 4; ++y) {
        const int i = 4 * bi + x, j = 4 * bj + y;
        if (i < l && j < l) out[i * l + j] = (j >= i) ? acc[x][y] : 0.0;
      }
  }
}

// G[e] = sum_p part[p][e]: a CTA covers 32 entries with 8 thread groups striding over the
// partials; the 8 group sums are combined in a fixed order (deterministic).
__global__ void __launch_bounds__(256) gram_reduce_kernel(const double* __restrict__ part, int parts, int l,
                                                          const int* __restrict__ skip, double* __restrict__ G) {
  pdl_trigger();  // programmatic dependent launch: the next QR stage may start launching
  pdl_wait();
  if (skip && *skip) return;
  __shared__ double red[8][33];
  const int lane = threadIdx.x & 31, grp = threadIdx.x >> 5;
  const int e = blockIdx.x * 32 + lane;
  const int ll = l * l;
  double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
  if (e < ll) {
    int p = grp;
    for (; p + 24 < parts; p += 32) {
      s0 += part[(size_t)p * ll + e];
      s1 += part[(size_t)(p + 8) * ll + e];
      s2 += part[(size_t)(p + 16) * ll + e];
      s3 += part[(size_t)(p + 24) * ll + e];
    }
    for (; p < parts; p += 8) s0 += part[(size_t)p * ll + e];
  }
  red[grp][lane] = (s0 + s1) + (s2 + s3);
  __syncthreads();
  if (grp == 0 && e < ll) {
    double t = 0.0;
#pragma unroll
    for (int g = 0; g < 8; ++g) t += red[g][lane];
    G[e] = t;
  }
}

// ---- Cholesky G = R^T R (R upper) by one warp, written with the reciprocal diagonal ---------
// Lanes own columns c = lane + 32q of the upper triangle (shared memory); each step needs only
// __syncwarp, so the 64 dependent pivots cost tens of cycles each instead of CTA barriers.
// A pivot below 4*l*eps*max(diag G) raises the breakdown flag. No triangular inverse: the apply
// kernel solves q R = y row by row.
__global__ void __launch_bounds__(32) chol_kernel(const double* __restrict__ Gin, int l, double* __restrict__ Rout,
                                                  double* __restrict__ rdiag, int* __restrict__ flag) {
  pdl_trigger();  // programmatic dependent launch: the next QR stage may start launching
  pdl_wait();
  if (*flag) return;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* Gs = reinterpret_cast<double*>(smem_raw);  // column-major copy: Gs[c * l + r] = G[r][c]
  const int lane = threadIdx.x;
  for (int e = lane; e < l * l; e += 32) {
    const int r = e / l, c = e - r * l;
    if (r <= c) Gs[c * l + r] = Gin[e];
  }
  __syncwarp();
  double md = 0.0;
  for (int i = lane; i < l; i += 32) md = fmax(md, Gs[i * l + i]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) md = fmax(md, __shfl_xor_sync(0xffffffffu, md, o));
  const double tol = 4.0 * l * 2.220446049250313e-16 * md;
  int bad = 0;
  for (int j = 0; j < l; ++j) {
    const double d2 = Gs[j * l + j];
    if (!(d2 > tol)) { bad = 1; break; }
    const double inv = rsqrt(d2);
    // row j of R for my columns c > j, then update my columns' entries r in (j, c]
    for (int c = lane; c < l; c += 32) {
      if (c <= j) continue;
      const double rjc = Gs[c * l + j] * inv;
      Gs[c * l + j] = rjc;
    }
    __syncwarp();
    for (int c = lane; c < l; c += 32) {
      if (c <= j) continue;
      const double rjc = Gs[c * l + j];
      double* col = Gs + c * l;
      for (int r = j + 1; r <= c; ++r) col[r] = fma(-Gs[r * l + j], rjc, col[r]);
    }
    if (lane == 0) {
      Gs[j * l + j] = d2 * inv;
      rdiag[j] = inv;
    }
    __syncwarp();
  }
  if (bad) {
    if (lane == 0) *flag = 1;
    return;
  }
  for (int e = lane; e < l * l; e += 32) {
    const int r = e / l, c = e - r * l;
    Rout[e] = r <= c ? Gs[c * l + r] : 0.0;
  }
}

// ---- register Cholesky for l <= 64: thread c keeps column c of G in registers ---------------
// Step j: thread j publishes 1/sqrt(pivot); every thread c > j scales its row-j entry into
// R[j][c] and publishes it; then thread c folds R[j][r] R[j][c] into its column (fully unrolled,
// predicated on j < r <= c). 64 steps x ~70 predicated FMAs + one 64-thread barrier each.
__global__ void __launch_bounds__(64) chol64_kernel(const double* __restrict__ Gin, int l, double* __restrict__ Rout,
                                                    double* __restrict__ rdiag, int* __restrict__ flag) {
  pdl_trigger();  // programmatic dependent launch: the next QR stage may start launching
  pdl_wait();
  if (*flag) return;
  __shared__ double rowj[64];
  __shared__ double s_inv;
  __shared__ int s_bad;
  const int c = threadIdx.x;
  double g[64];
#pragma unroll
  for (int r = 0; r < 64; ++r) g[r] = (c < l && r <= c) ? Gin[r * l + c] : 0.0;
  // max diagonal for the breakdown tolerance
  double dmax = (c < l) ? g[0] : 0.0;
#pragma unroll
  for (int r = 0; r < 64; ++r)
    if (r == c) dmax = g[r];
  rowj[c] = dmax;
  if (c == 0) s_bad = 0;
  __syncthreads();
  double md = 0.0;
  for (int i = 0; i < l; ++i) md = fmax(md, rowj[i]);
  const double tol = 4.0 * l * 2.220446049250313e-16 * md;
  __syncthreads();
#pragma unroll 1
  for (int j = 0; j < l; ++j) {
    if (c == j) {
      double d2 = 0.0;
#pragma unroll
      for (int r = 0; r < 64; ++r)
        if (r == j) d2 = g[r];
      if (!(d2 > tol)) s_bad = 1;
      const double inv = rsqrt(fmax(d2, 1e-300));
      s_inv = inv;
      rdiag[j] = inv;
    }
    __syncthreads();
    if (s_bad) break;
    const double inv = s_inv;
    double rjc = 0.0;
    if (c >= j) {
#pragma unroll
      for (int r = 0; r < 64; ++r)
        if (r == j) { g[r] *= inv; rjc = g[r]; }  // c == j: R[j][j] = d2 * inv = sqrt(d2)
    }
    rowj[c] = (c > j) ? rjc : 0.0;
    __syncthreads();
    if (c > j) {
#pragma unroll
      for (int r = 0; r < 64; ++r)
        if (r > j && r <= c) g[r] = fma(-rowj[r], rjc, g[r]);
    }
    __syncthreads();
  }
  if (s_bad) {
    if (c == 0) *flag = 1;
    return;
  }
  if (c < l) {
#pragma unroll
    for (int r = 0; r < 64; ++r)
      if (r < l) Rout[r * l + c] = (r <= c) ? g[r] : 0.0;
  }
}

// ---- fast path (l <= 64): Cholesky + triangular inverse + conditioning test, one CTA --------
// Elimination on the augmented pair [G | I] (rows/columns l..63 padded with the identity): the
// row operations of the Cholesky factorisation turn G into R and I into R^{-T}, so X = R^{-1} is
// read off transposed -- no separate back substitution. 256 threads; thread t owns row t % 64,
// columns [16 (t / 64), +16) of both blocks in registers (the lanes of a warp share their
// columns, so the row-j reads are shared-memory broadcasts). Step j: the four owners of row j
// publish it (double-buffered), one barrier, then every row r > j subtracts (A[j][r] / p) * row j
// and row j scales itself by 1 / sqrt(p). The two blocks are kept apart, so the update needs no
// per-entry masks (a combined 64 x 64 work matrix with R^{-T} in its lower triangle needed ~4x
// the instructions per step), and a warp skips a block whose 16 columns cannot change at step j
// (left: all columns < j; right: all columns > j -- row j's right part is zero there). Only the
// l real pivots run. The loop over j is not unrolled (the instruction cache; measured).
// kappa_F = ||R||_F ||X||_F >= cond_2(Y) decides whether CholeskyQR's second pass can be
// skipped: with fp32 outputs one fp64 pass already leaves ||Q^T Q - I|| <~ u64 * kappa^2, so
// kappa_F <= skip_kappa skips pass 2 (skip_out = 1). A pivot below 4*l*eps*max(diag G) raises
// the breakdown flag (Householder fallback).
// fp64 reciprocal and reciprocal square root for positive normal x: the MUFU seeds refined by two
// Newton steps (full double precision), without the library routines' special-case branches
__device__ __forceinline__ double fast_rcp(double x) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  double e = fma(-x, y, 1.0);
  y = fma(y, e, y);
  e = fma(-x, y, 1.0);
  return fma(y, e, y);
}
__device__ __forceinline__ double fast_rsqrt(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double h = 0.5 * x;
  double e = fma(-h * y, y, 0.5);
  y = fma(y, e, y);
  e = fma(-h * y, y, 0.5);
  return fma(y, e, y);
}

__global__ void __launch_bounds__(256) cholinv64_kernel(const double* __restrict__ Gin, int l, double* __restrict__ Xout,
                                                        const int* __restrict__ gate, int* __restrict__ breakdown,
                                                        int* __restrict__ skip_out, double skip_kappa) {
  pdl_trigger();  // programmatic dependent launch: the next QR stage may start launching
  pdl_wait();
  if (*gate) return;
  __shared__ __align__(16) double rowL[2][64];
  __shared__ __align__(16) double rowR[2][64];
  __shared__ double red[8][2];
  const int t = threadIdx.x, r = t & 63, c0 = (t >> 6) * 16;
  const int lane = t & 31, warp = t >> 5;
  double wl[16], wr[16];
#pragma unroll
  for (int u = 0; u < 16; ++u) {
    const int c = c0 + u;
    wl[u] = (r < l && c < l) ? (c >= r ? Gin[r * l + c] : 0.0) : (c == r ? 1.0 : 0.0);
    wr[u] = c == r ? 1.0 : 0.0;
  }
  double md = (t < 64 && r < l) ? Gin[r * l + r] : 0.0;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) md = fmax(md, __shfl_xor_sync(0xffffffffu, md, o));
  if (lane == 0) red[warp][0] = md;
  __syncthreads();
#pragma unroll
  for (int i = 0; i < 8; ++i) md = fmax(md, red[i][0]);
  const double tol = 4.0 * l * 2.220446049250313e-16 * md;
  bool bad = false;
#pragma unroll 1
  for (int j = 0; j < l; ++j) {
    double* bl = rowL[j & 1];
    double* br = rowR[j & 1];
    if (r == j) {
#pragma unroll
      for (int u = 0; u < 16; u += 2) {
        *reinterpret_cast<double2*>(&bl[c0 + u]) = make_double2(wl[u], wl[u + 1]);
        *reinterpret_cast<double2*>(&br[c0 + u]) = make_double2(wr[u], wr[u + 1]);
      }
    }
    __syncthreads();
    double p = bl[j];
    if (!(p > tol)) bad = true;  // uniform: every thread reads the same pivot
    if (!(p > 1e-300)) p = 1.0;  // keep the (discarded) arithmetic finite after a breakdown
    if (r > j) {
      const double f = bl[r] * fast_rcp(p);  // A[r][j] / p, with A[r][j] = A[j][r]
      if (c0 + 15 > j) {
#pragma unroll
        for (int u = 0; u < 16; u += 2) {
          const double2 bv = *reinterpret_cast<const double2*>(&bl[c0 + u]);
          wl[u] = fma(-f, bv.x, wl[u]);
          wl[u + 1] = fma(-f, bv.y, wl[u + 1]);
        }
      }
      if (c0 <= j) {
#pragma unroll
        for (int u = 0; u < 16; u += 2) {
          const double2 bv = *reinterpret_cast<const double2*>(&br[c0 + u]);
          wr[u] = fma(-f, bv.x, wr[u]);
          wr[u + 1] = fma(-f, bv.y, wr[u + 1]);
        }
      }
    } else if (r == j) {
      const double rsq = fast_rsqrt(p);
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        wl[u] *= rsq;
        wr[u] *= rsq;
      }
    }
  }
  if (bad) {
    if (t == 0) {
      *breakdown = 1;
      if (skip_out) *skip_out = 1;
    }
    return;
  }
  double r2 = 0.0, x2 = 0.0;
  if (r < l) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      const int c = c0 + u;
      if (c >= l) continue;
      if (c >= r) r2 = fma(wl[u], wl[u], r2);  // R[r][c]
      const double xv = c <= r ? wr[u] : 0.0;  // (R^{-T})[r][c] = X[c][r]
      x2 = fma(xv, xv, x2);
      Xout[c * l + r] = xv;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    r2 += __shfl_xor_sync(0xffffffffu, r2, o);
    x2 += __shfl_xor_sync(0xffffffffu, x2, o);
  }
  __syncthreads();  // red[] is reused
  if (lane == 0) {
    red[warp][0] = r2;
    red[warp][1] = x2;
  }
  __syncthreads();
  if (t == 0 && skip_out) {
    double sr = 0.0, sx = 0.0;
    for (int i = 0; i < 8; ++i) {
      sr += red[i][0];
      sx += red[i][1];
    }
    *skip_out = (sqrt(sr) * sqrt(sx) <= skip_kappa) ? 1 : 0;
  }
}

// The same elimination without a CTA barrier per pivot: every pivot row gets its own shared slot
// (64 rows x (64 + 64) doubles = 64 KB, never reused, so no write-after-read hazard) and its own
// mbarrier, on which the four owners of row j arrive after publishing it (release) and every thread
// waits before reading it (acquire). A thread that is still finishing step j's update no longer
// holds up the publication of row j + 1: the per-step chain is the owner's own update, publish and
// arrive, instead of the slowest warp plus a barrier.
__global__ void __launch_bounds__(256) cholinv64f_kernel(const double* __restrict__ Gin, int l,
                                                         double* __restrict__ Xout, const int* __restrict__ gate,
                                                         int* __restrict__ breakdown, int* __restrict__ skip_out,
                                                         double skip_kappa) {
  pdl_trigger();
  pdl_wait();
  if (*gate) return;
  extern __shared__ __align__(16) double rows[];  // [64][128]: left block, then right block
  __shared__ __align__(8) uint64_t rbar[64];
  __shared__ double red[8][2];
  const int t = threadIdx.x, r = t & 63, c0 = (t >> 6) * 16;
  const int lane = t & 31, warp = t >> 5;
  if (t < 64) asm volatile("mbarrier.init.shared::cta.b64 [%0], 4;" ::"r"((uint32_t)__cvta_generic_to_shared(&rbar[t])));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  double wl[16], wr[16];
#pragma unroll
  for (int u = 0; u < 16; ++u) {
    const int c = c0 + u;
    wl[u] = (r < l && c < l) ? (c >= r ? Gin[r * l + c] : 0.0) : (c == r ? 1.0 : 0.0);
    wr[u] = c == r ? 1.0 : 0.0;
  }
  double md = (t < 64 && r < l) ? Gin[r * l + r] : 0.0;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) md = fmax(md, __shfl_xor_sync(0xffffffffu, md, o));
  if (lane == 0) red[warp][0] = md;
  __syncthreads();
#pragma unroll
  for (int i = 0; i < 8; ++i) md = fmax(md, red[i][0]);
  const double tol = 4.0 * l * 2.220446049250313e-16 * md;
  bool bad = false;
  double rs_row = 1.0;  // rows l..63 (identity padding) stay unscaled
#pragma unroll 1
  for (int j = 0; j < l; ++j) {
    double* bl = rows + (size_t)j * 128;
    double* br = bl + 64;
    const uint32_t bar = (uint32_t)__cvta_generic_to_shared(&rbar[j]);
    if (r == j) {
#pragma unroll
      for (int u = 0; u < 16; u += 2) {
        *reinterpret_cast<double2*>(&bl[c0 + u]) = make_double2(wl[u], wl[u + 1]);
        *reinterpret_cast<double2*>(&br[c0 + u]) = make_double2(wr[u], wr[u + 1]);
      }
      asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
    }
    asm volatile(
        "{\n.reg .pred p;\nCW_%=:\n"
        "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%0], 0;\n"
        "@!p bra CW_%=;\n}\n" ::"r"(bar)
        : "memory");
    double p = bl[j];
    if (!(p > tol)) bad = true;  // uniform: every thread reads the same pivot
    if (!(p > 1e-300)) p = 1.0;  // keep the (discarded) arithmetic finite after a breakdown
    if (r > j) {
      const double f = bl[r] * fast_rcp(p);  // A[r][j] / p, with A[r][j] = A[j][r]
      if (c0 + 15 > j) {
#pragma unroll
        for (int u = 0; u < 16; u += 2) {
          const double2 bv = *reinterpret_cast<const double2*>(&bl[c0 + u]);
          wl[u] = fma(-f, bv.x, wl[u]);
          wl[u + 1] = fma(-f, bv.y, wl[u + 1]);
        }
      }
      if (c0 <= j) {
#pragma unroll
        for (int u = 0; u < 16; u += 2) {
          const double2 bv = *reinterpret_cast<const double2*>(&br[c0 + u]);
          wr[u] = fma(-f, bv.x, wr[u]);
          wr[u + 1] = fma(-f, bv.y, wr[u + 1]);
        }
      }
    }
    // row j keeps its unscaled values (the published copy is what the later rows need); its
    // 1 / sqrt(p) scaling is applied once after the loop, off the per-pivot chain
    if (r == j) rs_row = fast_rsqrt(p);
  }
  __syncthreads();
#pragma unroll
  for (int u = 0; u < 16; ++u) {
    wl[u] *= rs_row;
    wr[u] *= rs_row;
  }
  if (bad) {
    if (t == 0) {
      *breakdown = 1;
      if (skip_out) *skip_out = 1;
    }
    return;
  }
  double r2 = 0.0, x2 = 0.0;
  if (r < l) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      const int c = c0 + u;
      if (c >= l) continue;
      if (c >= r) r2 = fma(wl[u], wl[u], r2);  // R[r][c]
      const double xv = c <= r ? wr[u] : 0.0;  // (R^{-T})[r][c] = X[c][r]
      x2 = fma(xv, xv, x2);
      Xout[c * l + r] = xv;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    r2 += __shfl_xor_sync(0xffffffffu, r2, o);
    x2 += __shfl_xor_sync(0xffffffffu, x2, o);
  }
  if (lane == 0) {
    red[warp][0] = r2;
    red[warp][1] = x2;
  }
  __syncthreads();
  if (t == 0 && skip_out) {
    double sr = 0.0, sx = 0.0;
    for (int i = 0; i < 8; ++i) {
      sr += red[i][0];
      sx += red[i][1];
    }
    *skip_out = (sqrt(sr) * sqrt(sx) <= skip_kappa) ? 1 : 0;
  }
}

// ---- blocked Cholesky inverse (l <= 64): 64 pivots on one warp, the bulk on the whole CTA -------
// Gauss-Jordan on [G | I] by 16-column blocks. Step k (kb = 16 k):
//   (a) warp 0 eliminates the 16 x 16 diagonal block A_kk in registers: lane i (< 16) holds row i
//       of A_kk, lane i + 16 row i of the identity beside it; each pivot row is published in its own
//       shared slot behind one __syncwarp, and every later row folds it in (its multiplier is
//       a_j[i] / a_j[j]: the trailing block is symmetric, so both halves of a row read it from the
//       published row). Rows scaled by 1 / sqrt(pivot) give Li = L_kk^{-1} (A_kk = L_kk L_kk^T).
//   (b) the CTA: T = Li [A_k | B_k] (block row k normalised; only the left columns past the block
//       and the right columns up to it are non-trivial: 64 columns), Mb = A_ik Li^T for the rows
//       below, then [A_i | B_i] -= Mb T (4 x 4 register blocks) and block row k's right part := T.
// At the end the right half is L^{-1}, X = R^{-1} = L^{-T}. The serial chain is the 64 pivots at a
// warp's latency (one shared round trip, a reciprocal and 16 FMAs each) instead of a CTA-wide
// publish/acquire per pivot (cholinv64f_kernel: ~1000 cycles per pivot); the O(l^3) work runs in
// three CTA-wide phases per block. Same breakdown rule (pivot <= 4 l eps max diag G) and kappa
// estimate: ||R||_F^2 = trace(G), so kappa_F = sqrt(trace G) ||X||_F.
struct CholBlkSmem {
  double S[64][130];  // [G | I] -> [.. | L^{-1}]; pitch 130 doubles
  double T[16][66];
  double Mb[48][17];
  double Li[16][17];
  double rowbuf[16][32];
  double red[8][2];
  double tol, trace;
  int bad;
  // scratch for the fused QR's Gram reduction (S is free between Cholesky runs)
  __device__ double (*red_wide())[33] { return reinterpret_cast<double(*)[33]>(&S[0][0]); }
};

#ifndef APX_CHOL_STAMP
#define APX_CHOL_STAMP(i)  // tools/chol_blk_probe.cu: per-phase clock stamps
#endif
#ifndef APX_CQR_STAMP
#define APX_CQR_STAMP(i)  // tools/chol_blk_probe.cu: per-phase timer stamps of the fused QR (CTA 0)
#endif

__device__ __forceinline__ int cholblk_col(int q, int kb, int nr) { return q < nr ? kb + 16 + q : 64 + q - nr; }

// All 256 threads. G: l x l (global or shared). Writes X = R^{-1} (zero-padded to 64 x 64) to Xs
// (row pitch xp) and returns breakdown; *skip = (kappa_F <= skip_kappa). Ends with a CTA barrier.
__device__ bool cholinv_blk(const double* __restrict__ G, int l, CholBlkSmem& sm, double* Xs, int xp,
                            double skip_kappa, bool* skip) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int e = tid; e < 64 * 64; e += 256) {
    const int r = e >> 6, c = e & 63;
    sm.S[r][c] = (r < l && c < l) ? G[r * l + c] : (r == c ? 1.0 : 0.0);
    sm.S[r][64 + c] = r == c ? 1.0 : 0.0;
  }
  if (warp == 0) {
    double d0 = lane < l ? G[lane * l + lane] : 0.0, d1 = lane + 32 < l ? G[(lane + 32) * l + lane + 32] : 0.0;
    double md = fmax(d0, d1), tr = d0 + d1;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      md = fmax(md, __shfl_xor_sync(0xffffffffu, md, o));
      tr += __shfl_xor_sync(0xffffffffu, tr, o);
    }
    if (lane == 0) {
      sm.tol = 4.0 * l * 2.220446049250313e-16 * md;
      sm.trace = tr;
      sm.bad = 0;
    }
  }
  __syncthreads();
  APX_CHOL_STAMP(0);
  const double tol = sm.tol;
  const int nblk = (l + 15) >> 4;  // blocks past l are identity: nothing to eliminate
#pragma unroll 1
  for (int k = 0; k < nblk; ++k) {
    const int kb = 16 * k, nr = 48 - kb;
    // (a) the diagonal block on warp 0 by 2 x 2 block pivots: rows j, j + 1 are published together
    //     and every later row eliminates both at once with the pivot block's inverse (one shared
    //     round trip and one reciprocal per two pivots: tools/warp_chol_probe.cu, ~320 cycles per
    //     single pivot); the identity half of each pivot pair is then normalised by the inverse of
    //     the pair's 2 x 2 Cholesky factor (L^{-1} = C^{-1} E for A = (E^{-1} C)(E^{-1} C)^T).
    if (warp == 0) {
      const int li = lane & 15, half = lane >> 4;
      double v[16];
#pragma unroll
      for (int c = 0; c < 16; ++c) v[c] = half == 0 ? sm.S[kb + li][kb + c] : (c == li ? 1.0 : 0.0);
      bool wbad = false;
#pragma unroll
      for (int j = 0; j < 16; j += 2) {
        if ((li >> 1) == (j >> 1)) {
#pragma unroll
          for (int c = 0; c < 16; c += 2)
            *reinterpret_cast<double2*>(&sm.rowbuf[li][half * 16 + c]) = make_double2(v[c], v[c + 1]);
        }
        __syncwarp();
        double a = sm.rowbuf[j][j], b = sm.rowbuf[j][j + 1], d = sm.rowbuf[j + 1][j + 1];
        double det = fma(a, d, -b * b);
        if (!(a > tol) || !(det > tol * a)) {  // pivots a and det / a (the sequential elimination's)
          wbad = true;
          a = 1.0;
          b = 0.0;
          d = 1.0;
          det = 1.0;
        }
        const double idet = fast_rcp(det);
        const double i00 = d * idet, i01 = -b * idet, i11 = a * idet;
        if (li > j + 1) {
          const double x0 = sm.rowbuf[j][li], x1 = sm.rowbuf[j + 1][li];  // a_ij, a_i,j+1 (symmetric)
          const double f0 = fma(x1, i01, x0 * i00), f1 = fma(x1, i11, x0 * i01);
          const double* p0 = &sm.rowbuf[j][half * 16];
          const double* p1 = &sm.rowbuf[j + 1][half * 16];
#pragma unroll
          for (int c = 0; c < 16; c += 2) {
            const double2 w0 = *reinterpret_cast<const double2*>(p0 + c);
            const double2 w1 = *reinterpret_cast<const double2*>(p1 + c);
            v[c] = fma(-f1, w1.x, fma(-f0, w0.x, v[c]));
            v[c + 1] = fma(-f1, w1.y, fma(-f0, w0.y, v[c + 1]));
          }
        }
      }
      if (half == 1) {
        // C = chol([[a, b], [b, d]]) = [[c00, 0], [c10, c11]]: rows j, j + 1 of Li = C^{-1} [b_j; b_j+1]
        const int j = li & ~1;
        const double a = sm.rowbuf[j][j], b = sm.rowbuf[j][j + 1], d = sm.rowbuf[j + 1][j + 1];
        const double r00 = fast_rsqrt(fmax(a, 1e-300)), c10 = b * r00;
        const double r11 = fast_rsqrt(fmax(fma(-c10, c10, d), 1e-300));
        const double* bj = &sm.rowbuf[j][16];
        const double* bj1 = &sm.rowbuf[j + 1][16];
        if (li == j) {
#pragma unroll
          for (int c = 0; c < 16; ++c) sm.Li[li][c] = bj[c] * r00;
        } else {
          const double t = c10 * r00;
#pragma unroll
          for (int c = 0; c < 16; ++c) sm.Li[li][c] = fma(-t, bj[c], bj1[c]) * r11;
        }
      }
      if (lane == 0 && wbad) sm.bad = 1;
    }
    __syncthreads();
    APX_CHOL_STAMP(1 + 3 * k);
    // (b1) T = Li [A_k | B_k] (64 columns), Mb = A_ik Li^T
    {
      const int mrow = tid >> 4, q0 = tid & 15;
      double acc[4] = {0.0, 0.0, 0.0, 0.0};
      int cols[4];
#pragma unroll
      for (int x = 0; x < 4; ++x) cols[x] = cholblk_col(q0 + 16 * x, kb, nr);
#pragma unroll
      for (int s = 0; s < 16; ++s) {
        const double w = sm.Li[mrow][s];  // zero above the diagonal
#pragma unroll
        for (int x = 0; x < 4; ++x) acc[x] = fma(w, sm.S[kb + s][cols[x]], acc[x]);
      }
#pragma unroll
      for (int x = 0; x < 4; ++x) sm.T[mrow][q0 + 16 * x] = acc[x];
    }
    {
      // up to three independent rows per thread (nr <= 48)
      const int sc = tid & 15, ip0 = tid >> 4;
      double a[3] = {0.0, 0.0, 0.0};
#pragma unroll
      for (int s2 = 0; s2 < 16; ++s2) {
        const double li_v = sm.Li[sc][s2];
#pragma unroll
        for (int x = 0; x < 3; ++x)
          if (ip0 + 16 * x < nr) a[x] = fma(sm.S[kb + 16 + ip0 + 16 * x][kb + s2], li_v, a[x]);
      }
#pragma unroll
      for (int x = 0; x < 3; ++x)
        if (ip0 + 16 * x < nr) sm.Mb[ip0 + 16 * x][sc] = a[x];
    }
    __syncthreads();
    APX_CHOL_STAMP(2 + 3 * k);
    // (b2) the trailing update in 4 x 4 register blocks, and block row k's right part
    if (tid < (nr / 4) * 16) {
      const int rb = (tid >> 4) * 4, q0 = tid & 15;
      double acc[4][4];
      int cols[4];
#pragma unroll
      for (int x = 0; x < 4; ++x) cols[x] = cholblk_col(q0 + 16 * x, kb, nr);
#pragma unroll
      for (int y = 0; y < 4; ++y)
#pragma unroll
        for (int x = 0; x < 4; ++x) acc[y][x] = sm.S[kb + 16 + rb + y][cols[x]];
#pragma unroll 4
      for (int s = 0; s < 16; ++s) {
        double mv[4], tv[4];
#pragma unroll
        for (int y = 0; y < 4; ++y) mv[y] = sm.Mb[rb + y][s];
#pragma unroll
        for (int x = 0; x < 4; ++x) tv[x] = sm.T[s][q0 + 16 * x];
#pragma unroll
        for (int y = 0; y < 4; ++y)
#pragma unroll
          for (int x = 0; x < 4; ++x) acc[y][x] = fma(-mv[y], tv[x], acc[y][x]);
      }
#pragma unroll
      for (int y = 0; y < 4; ++y)
#pragma unroll
        for (int x = 0; x < 4; ++x) sm.S[kb + 16 + rb + y][cols[x]] = acc[y][x];
    }
    for (int e = tid; e < 16 * 64; e += 256) {
      const int mrow = e >> 6, c = e & 63;
      if (c <= kb + 15) sm.S[kb + mrow][64 + c] = sm.T[mrow][nr + c];
    }
    __syncthreads();
    APX_CHOL_STAMP(3 + 3 * k);
  }
  double x2 = 0.0;
  for (int e = tid; e < 64 * 64; e += 256) {
    const int i = e >> 6, c = e & 63;
    const double xv = (i < l && c < l && i <= c) ? sm.S[c][64 + i] : 0.0;  // X[i][c] = L^{-1}[c][i]
    Xs[i * xp + c] = xv;
    x2 = fma(xv, xv, x2);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x2 += __shfl_xor_sync(0xffffffffu, x2, o);
  if (lane == 0) sm.red[warp][0] = x2;
  __syncthreads();
  double sx = 0.0;
#pragma unroll
  for (int i = 0; i < 8; ++i) sx += sm.red[i][0];
  *skip = sqrt(sm.trace) * sqrt(sx) <= skip_kappa;
  const bool bad = sm.bad != 0;
  __syncthreads();  // sm may be reused by the caller
  return bad;
}

// standalone launch of cholinv_blk: same contract as cholinv64f_kernel
__global__ void __launch_bounds__(256, 1) cholinv_blk_kernel(const double* __restrict__ Gin, int l,
                                                             double* __restrict__ Xout, const int* __restrict__ gate,
                                                             int* __restrict__ breakdown, int* __restrict__ skip_out,
                                                             double skip_kappa) {
  pdl_trigger();
  pdl_wait();
  if (*gate) return;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  CholBlkSmem& sm = *reinterpret_cast<CholBlkSmem*>(smem_raw);
  double* Xs = reinterpret_cast<double*>(smem_raw + sizeof(CholBlkSmem));  // 64 x 64
  bool skip = false;
  const bool bad = cholinv_blk(Gin, l, sm, Xs, 64, skip_kappa, &skip);
  if (bad) {
    if (threadIdx.x == 0) {
      *breakdown = 1;
      if (skip_out) *skip_out = 1;
    }
    return;
  }
  for (int e = threadIdx.x; e < l * l; e += 256) {
    const int i = e / l, c = e - i * l;
    Xout[e] = Xs[i * 64 + c];
  }
  if (threadIdx.x == 0 && skip_out) *skip_out = skip ? 1 : 0;
}
constexpr size_t kCholBlkSmem = sizeof(CholBlkSmem) + 64 * 64 * sizeof(double);

// Cholesky-inverse launch for l <= 64. (Measured alternative: the same elimination on 1024 threads,
// 4 + 4 columns per thread, was slower -- 65 vs 55 us in the C4 chain, C1 2.19 vs 2.11 ms. The
// step is bound by its owner warp: rows j and j+1 sit in one warp, so row j's scaling and row
// j+1's update serialise before row j+1 can be published; tools/chol_probe2.cu, fp64_issue_probe.cu.)
static cudaError_t launch_cholinv64(const double* G, int l, double* X, const int* gate, int* breakdown, int* skip_out,
                                   double skip_kappa, cudaStream_t st) {
  static const bool barrier = getenv("APX_CHOL_BARRIER") != nullptr;  // A/B: one CTA barrier per pivot
  static const bool flat = getenv("APX_CHOL_FLAT") != nullptr;        // A/B: unblocked, per-row mbarriers
  if (barrier)
    return launch_pdl(cholinv64_kernel, dim3(1), dim3(256), 0, st, G, l, X, gate, breakdown, skip_out, skip_kappa);
  if (!flat) {
    const cudaError_t a = cudaFuncSetAttribute(cholinv_blk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                               (int)kCholBlkSmem);
    if (a != cudaSuccess) return a;
    return launch_pdl(cholinv_blk_kernel, dim3(1), dim3(256), kCholBlkSmem, st, G, l, X, gate, breakdown, skip_out,
                      skip_kappa);
  }
  constexpr size_t smem = (size_t)64 * 128 * sizeof(double);
  const cudaError_t attr = cudaFuncSetAttribute(cholinv64f_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (attr != cudaSuccess) return attr;
  return launch_pdl(cholinv64f_kernel, dim3(1), dim3(256), smem, st, G, l, X, gate, breakdown, skip_out, skip_kappa);
}

// ---- Q = Y X (X = R^{-1} upper, l <= 64) over 64-row tiles ---------------------------------
// CTA = 64 rows x 64 columns of Q, 256 threads on a 16 x 16 grid of 4 x 4 blocks. The Y tile is
// staged transposed (Ys[i][r], fp64) with all loads in flight at once, X zero-padded to 64 x 64.
// Writes the fp64 copy Q1 (input of CholeskyQR's second pass, unless *q1_skip says it will not
// run) and/or the typed outputs Q, Q2.
template <typename TI, typename TO>
__global__ void __launch_bounds__(256) apply_x_kernel(const TI* __restrict__ Y, int64_t rs, int64_t cs, int m, int l,
                                                      const double* __restrict__ X, const int* __restrict__ skip,
                                                      const int* __restrict__ q1_skip, double* __restrict__ Q1,
                                                      TO* __restrict__ Q, int64_t qrs,
                                                      int64_t qcs, TO* __restrict__ Q2, int64_t q2rs, int64_t q2cs,
                                                      int tf32 = 0) {
  pdl_trigger();  // programmatic dependent launch: the next QR stage may start launching
  pdl_wait();
  if (*skip) return;
  if (q1_skip && *q1_skip) Q1 = nullptr;  // CholeskyQR's second pass will not run
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double(*Ys)[kTP] = reinterpret_cast<double(*)[kTP]>(smem_raw);  // [i][r]
  double(*Xs)[kTP] = Ys + 64;                                      // [i][c]
  const int tid = threadIdx.x;
  const int r0 = blockIdx.x * 64;
#pragma unroll 4
  for (int e = tid; e < 64 * 64; e += 256) {
    const int i = e >> 6, c = e & 63;
    Xs[i][c] = (i < l && c < l) ? X[i * l + c] : 0.0;
  }
  load_tile64<true>(Y, rs, cs, m, l, r0, Ys);
  __syncthreads();
  const int tr = (tid >> 4) * 4, tc = (tid & 15) * 4;
  double acc[4][4];
#pragma unroll
  for (int x = 0; x < 4; ++x)
#pragma unroll
    for (int y = 0; y < 4; ++y) acc[x][y] = 0.0;
#pragma unroll 8
  for (int i = 0; i < 64; ++i) {
    const double2 a01 = *reinterpret_cast<const double2*>(&Ys[i][tr]);
    const double2 a23 = *reinterpret_cast<const double2*>(&Ys[i][tr + 2]);
    const double2 b01 = *reinterpret_cast<const double2*>(&Xs[i][tc]);
    const double2 b23 = *reinterpret_cast<const double2*>(&Xs[i][tc + 2]);
    const double av[4] = {a01.x, a01.y, a23.x, a23.y}, bv[4] = {b01.x, b01.y, b23.x, b23.y};
#pragma unroll
    for (int x = 0; x < 4; ++x)
#pragma unroll
      for (int y = 0; y < 4; ++y) acc[x][y] = fma(av[x], bv[y], acc[x][y]);
  }
#pragma unroll
  for (int x = 0; x < 4; ++x) {
    const int r = r0 + tr + x;
    if (r >= m) continue;
#pragma unroll
    for (int y = 0; y < 4; ++y) {
      const int c = tc + y;
      if (c >= l) continue;
      if (Q1) Q1[(size_t)r * l + c] = acc[x][y];
      if (Q) Q[(size_t)r * qrs + (size_t)c * qcs] = qout<TO>(acc[x][y], tf32);
      if (Q2) Q2[(size_t)r * q2rs + (size_t)c * q2cs] = qout<TO>(acc[x][y], tf32);
    }
  }
}

// ---- fused CholeskyQR2 (l <= 64): one 64-row tile per CTA, every CTA resident at once --------------
// One launch instead of the chain gram -> reduce -> cholinv -> apply (-> the same again): each CTA
// keeps its tile of Y in shared memory (fp64) for the whole QR, writes its Gram partial, and after a
// grid barrier reduces a slice of the entries (each entry summed over the partials in a fixed order)
// ; after a second barrier EVERY CTA runs the same Cholesky inverse on the reduced G (cholinv_blk:
// bitwise the same X everywhere, no third barrier and no single-CTA stage), applies it to its tile,
// and -- when the conditioning asks for pass 2 -- repeats on the Q1 tile it still holds. Launched
// cooperatively (the runtime checks that the grid fits co-resident); the barriers are an atomic
// counter with a bounded wait: a barrier that does not complete within 50 ms (a co-tenant holding
// SMs) raises the breakdown flag instead, so the Householder kernel that follows recomputes Q.
// flag: [0] breakdown (-> Householder), [1] pass 2 skipped, [2] barrier counter (zeroed before).
// X = R^{-1} is written into the Cholesky buffer's left half (dead once the elimination is done),
// which keeps the CTA at ~121 KB of shared memory: a CTA of B's energy pass (96 KB) fits beside it on
// the same SM, so the QR and the energy pass that runs concurrently in the C4 plan do not exclude
// each other's CTAs
constexpr int kCqrXP = 130;  // = CholBlkSmem::S row pitch
template <int TPC>
struct CqrSmem {
  double Ys[TPC][64][kTP];  // the CTA's tiles [r][i]: Y, then Q1
  CholBlkSmem ch;           // ch.S[i][0..63] holds X[i][c] after each Cholesky inverse
  int abort;
};

__device__ __forceinline__ bool cqr_grid_sync(unsigned* ctr, unsigned target, volatile int* s_abort) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(ctr, 1u);
    unsigned long long t0, now;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    while (true) {
      unsigned v;
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory");
      if (v >= target) break;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
      if (now - t0 > 50000000ull) {
        *s_abort = 1;
        break;
      }
      __nanosleep(64);
    }
  }
  __syncthreads();
  return *s_abort == 0;
}

// partial Gram of the staged tiles -> part (l x l)
template <int TPC>
__device__ __forceinline__ void cqr_gram_tile(const double (*Yt)[64][kTP], int l, double* __restrict__ part) {
  const int bi = (threadIdx.x >> 4) * 4, bj = (threadIdx.x & 15) * 4;
  double acc[4][4];
#pragma unroll
  for (int x = 0; x < 4; ++x)
#pragma unroll
    for (int y = 0; y < 4; ++y) acc[x][y] = 0.0;
#pragma unroll 8
  for (int rr = 0; rr < 64 * TPC; ++rr) {
    const double(*Ys)[kTP] = Yt[rr >> 6];
    const int r = rr & 63;
    const double2 a01 = *reinterpret_cast<const double2*>(&Ys[r][bi]);
    const double2 a23 = *reinterpret_cast<const double2*>(&Ys[r][bi + 2]);
    const double2 b01 = *reinterpret_cast<const double2*>(&Ys[r][bj]);
    const double2 b23 = *reinterpret_cast<const double2*>(&Ys[r][bj + 2]);
    const double av[4] = {a01.x, a01.y, a23.x, a23.y}, bv[4] = {b01.x, b01.y, b23.x, b23.y};
#pragma unroll
    for (int x = 0; x < 4; ++x)
#pragma unroll
      for (int y = 0; y < 4; ++y) acc[x][y] = fma(av[x], bv[y], acc[x][y]);
  }
#pragma unroll
  for (int x = 0; x < 4; ++x)
#pragma unroll
    for (int y = 0; y < 4; ++y) {
      const int i = bi + x, j = bj + y;
      if (i < l && j < l) part[i * l + j] = acc[x][y];
    }
}

// this CTA's slice of G = sum_p part[p] (8 groups of 32 lanes stride the partials; fixed order)
__device__ __forceinline__ void cqr_reduce_slice(const double* __restrict__ part, int parts, int l,
                                                 double* __restrict__ G, double (*red)[33]) {
  const int ll = l * l, per = (int)ceil_div(ll, (int)gridDim.x);
  const int e0 = blockIdx.x * per, e1 = min(ll, e0 + per);
  const int lane = threadIdx.x & 31, grp = threadIdx.x >> 5;
  for (int eb = e0; eb < e1; eb += 32) {
    const int e = eb + lane;
    double s0 = 0.0, s1 = 0.0;
    if (e < e1) {
      int p = grp;
      for (; p + 8 < parts; p += 16) {
        s0 += __ldcg(part + (size_t)p * ll + e);
        s1 += __ldcg(part + (size_t)(p + 8) * ll + e);
      }
      for (; p < parts; p += 8) s0 += __ldcg(part + (size_t)p * ll + e);
    }
    red[grp][lane] = s0 + s1;
    __syncthreads();
    if (grp == 0 && e < e1) {
      double t = 0.0;
#pragma unroll
      for (int g = 0; g < 8; ++g) t += red[g][lane];
      G[e] = t;
    }
    __syncthreads();
  }
}

// acc = tile . X (4 x 4 per thread: rows tr.., columns tc..); X rows at pitch kCqrXP
__device__ __forceinline__ void cqr_apply_tile(const double (*Ys)[kTP], const double (*Xs)[kCqrXP], double (&acc)[4][4]) {
  const int tr = (threadIdx.x >> 4) * 4, tc = (threadIdx.x & 15) * 4;
#pragma unroll
  for (int x = 0; x < 4; ++x)
#pragma unroll
    for (int y = 0; y < 4; ++y) acc[x][y] = 0.0;
#pragma unroll 8
  for (int i = 0; i < 64; ++i) {
    const double2 b01 = *reinterpret_cast<const double2*>(&Xs[i][tc]);
    const double2 b23 = *reinterpret_cast<const double2*>(&Xs[i][tc + 2]);
    const double bv[4] = {b01.x, b01.y, b23.x, b23.y};
#pragma unroll
    for (int x = 0; x < 4; ++x) {
      const double a = Ys[tr + x][i];
#pragma unroll
      for (int y = 0; y < 4; ++y) acc[x][y] = fma(a, bv[y], acc[x][y]);
    }
  }
}

template <typename TI, typename TO, int TPC>
__global__ void __launch_bounds__(256, 1) cqr2_fused_kernel(const TI* __restrict__ Y, int64_t rs, int64_t cs, int m,
                                                            int l, double* __restrict__ part1,
                                                            double* __restrict__ part2, double* __restrict__ G1,
                                                            double* __restrict__ G2, int* __restrict__ flag,
                                                            TO* __restrict__ Q, int64_t qrs, int64_t qcs,
                                                            TO* __restrict__ Q2, int64_t q2rs, int64_t q2cs, int tf32,
                                                            double skip_kappa) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  CqrSmem<TPC>& sm = *reinterpret_cast<CqrSmem<TPC>*>(smem_raw);
  unsigned* ctr = reinterpret_cast<unsigned*>(flag + 2);
  const unsigned nb = gridDim.x;
  const int b = blockIdx.x;
  const int tr = (threadIdx.x >> 4) * 4, tc = (threadIdx.x & 15) * 4;
  APX_CQR_STAMP(0);
  if (threadIdx.x == 0) sm.abort = 0;
#pragma unroll
  for (int t = 0; t < TPC; ++t) load_tile64<false>(Y, rs, cs, m, l, (b * TPC + t) * 64, sm.Ys[t]);
  __syncthreads();
  APX_CQR_STAMP(1);
  cqr_gram_tile<TPC>(sm.Ys, l, part1 + (size_t)b * l * l);
  APX_CQR_STAMP(2);
  if (!cqr_grid_sync(ctr, nb, &sm.abort)) goto fail;
  APX_CQR_STAMP(3);
  cqr_reduce_slice(part1, nb, l, G1, sm.ch.red_wide());
  APX_CQR_STAMP(4);
  if (!cqr_grid_sync(ctr, 2 * nb, &sm.abort)) goto fail;
  APX_CQR_STAMP(5);
  {
    bool skip2 = false;
    if (cholinv_blk(G1, l, sm.ch, &sm.ch.S[0][0], kCqrXP, skip_kappa, &skip2)) goto fail;
    APX_CQR_STAMP(6);
    double acc[4][4];
    if (!skip2) {
      // Q1 = Y X, tile by tile, in place; then pass 2 on the Q1 tiles
#pragma unroll
      for (int t = 0; t < TPC; ++t) {
        cqr_apply_tile(sm.Ys[t], sm.ch.S, acc);
        __syncthreads();  // every read of the tile done
#pragma unroll
        for (int x = 0; x < 4; ++x)
#pragma unroll
          for (int y = 0; y < 4; ++y) sm.Ys[t][tr + x][tc + y] = (tc + y < l) ? acc[x][y] : 0.0;
      }
      __syncthreads();
      cqr_gram_tile<TPC>(sm.Ys, l, part2 + (size_t)b * l * l);
      if (!cqr_grid_sync(ctr, 3 * nb, &sm.abort)) goto fail;
      cqr_reduce_slice(part2, nb, l, G2, sm.ch.red_wide());
      if (!cqr_grid_sync(ctr, 4 * nb, &sm.abort)) goto fail;
      bool unused = false;
      if (cholinv_blk(G2, l, sm.ch, &sm.ch.S[0][0], kCqrXP, 0.0, &unused)) goto fail;
    }
    APX_CQR_STAMP(7);
    if (b == 0 && threadIdx.x == 0) flag[1] = skip2 ? 1 : 0;
#pragma unroll
    for (int t = 0; t < TPC; ++t) {
      cqr_apply_tile(sm.Ys[t], sm.ch.S, acc);
      const int r0 = (b * TPC + t) * 64;
#pragma unroll
      for (int x = 0; x < 4; ++x) {
        const int r = r0 + tr + x;
        if (r >= m) continue;
#pragma unroll
        for (int y = 0; y < 4; ++y) {
          const int c = tc + y;
          if (c >= l) continue;
          if (Q) Q[(size_t)r * qrs + (size_t)c * qcs] = qout<TO>(acc[x][y], tf32);
          if (Q2) Q2[(size_t)r * q2rs + (size_t)c * q2cs] = qout<TO>(acc[x][y], tf32);
        }
      }
    }
    return;
  }
fail:
  if (threadIdx.x == 0) atomicExch(flag, 1);  // breakdown or barrier timeout: the Householder kernel runs
}
// tiles per CTA: 2 when the sketch has many row tiles (C4: 64 CTAs instead of 128, so B's concurrent
// energy pass keeps the other SMs), else 1; APX_QR_TPC overrides
static int cqr_tpc(int tiles) {
  static const int env = getenv("APX_QR_TPC") ? atoi(getenv("APX_QR_TPC")) : 0;
  if (env == 1 || env == 2) return env;
  return tiles > 96 ? 2 : 1;
}

// ---- Q = Y R^{-1} by forward substitution q R = y, one warp per row ------------------------
// Lane c owns columns c, c+32, ...; at step j the owner finalises q_j = acc_j / R_jj and every
// lane folds q_j R[j][c] into its later columns. R (upper) is staged in shared memory.
template <typename TI, typename TO, int LW>
__global__ void __launch_bounds__(256) apply_rinv_kernel(const TI* __restrict__ Y, int64_t rs, int64_t cs, int m,
                                                         int l, const double* __restrict__ R,
                                                         const double* __restrict__ rdiag,
                                                         const int* __restrict__ flag, TO* __restrict__ Q,
                                                         int64_t qrs, int64_t qcs, TO* __restrict__ Q2, int64_t q2rs,
                                                         int64_t q2cs, int tf32) {
  pdl_trigger();  // programmatic dependent launch: the next QR stage may start launching
  pdl_wait();
  if (*flag) return;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* Rs = reinterpret_cast<double*>(smem_raw);
  double* rd = Rs + l * l;
  for (int e = threadIdx.x; e < l * l; e += blockDim.x) Rs[e] = R[e];
  for (int e = threadIdx.x; e < l; e += blockDim.x) rd[e] = rdiag[e];
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int warps = blockDim.x >> 5;
  for (int r = blockIdx.x * warps + (threadIdx.x >> 5); r < m; r += gridDim.x * warps) {
    double acc[LW];
#pragma unroll
    for (int q = 0; q < LW; ++q) {
      const int c = lane + 32 * q;
      acc[q] = c < l ? (double)Y[(size_t)r * rs + (size_t)c * cs] : 0.0;
    }
#pragma unroll
    for (int q = 0; q < LW; ++q) {
      for (int i = 0; i < 32; ++i) {
        const int j = 32 * q + i;
        if (j >= l) break;
        // owner lane i (register slot q) finalises q_j
        double qj = 0.0;
        if (lane == i) {
          acc[q] *= rd[j];
          qj = acc[q];
        }
        qj = __shfl_sync(0xffffffffu, qj, i);
#pragma unroll
        for (int p = 0; p < LW; ++p) {
          const int c = lane + 32 * p;
          if (c > j && c < l) acc[p] = fma(-qj, Rs[j * l + c], acc[p]);
        }
      }
    }
#pragma unroll
    for (int q = 0; q < LW; ++q) {
      const int c = lane + 32 * q;
      if (c < l) {
        Q[(size_t)r * qrs + (size_t)c * qcs] = qout<TO>(acc[q], tf32);
        if (Q2) Q2[(size_t)r * q2rs + (size_t)c * q2cs] = qout<TO>(acc[q], tf32);
      }
    }
  }
}

// ---- Householder QR fallback (one CTA, fp64, global working copy) ------------------------
template <typename TI, typename TO>
__global__ void __launch_bounds__(1024) householder_qr_kernel(const TI* __restrict__ Y, int64_t rs, int64_t cs, int m,
                                                              int l, const int* __restrict__ flag, int force,
                                                              double* __restrict__ W /*m x l*/,
                                                              double* __restrict__ V /*m x l*/, TO* __restrict__ Q,
                                                              int64_t qrs, int64_t qcs, TO* __restrict__ Q2,
                                                              int64_t q2rs, int64_t q2cs, int tf32) {
  pdl_trigger();  // programmatic dependent launch: the next QR stage may start launching
  pdl_wait();
  if (!force && !(*flag)) return;
  __shared__ double red[32];
  extern __shared__ double hh_smem[];  // s_dot[l], s_tau[l]
  double* s_dot = hh_smem;
  __shared__ double s_scal[2];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  for (size_t e = tid; e < (size_t)m * l; e += blockDim.x) {
    const size_t r = e / l, c = e % l;
    W[e] = (double)Y[r * rs + c * cs];
  }
  __syncthreads();
  // factor
  for (int j = 0; j < l; ++j) {
    // tail norm ||W[j+1:, j]||^2 and x0
    double s = 0.0;
    for (int r = j + 1 + tid; r < m; r += blockDim.x) {
      const double v = W[(size_t)r * l + j];
      s = fma(v, v, s);
    }
    s = block_sum(s, red);
    if (tid == 0) {
      const double x0 = W[(size_t)j * l + j];
      if (s == 0.0) {
        s_scal[0] = 0.0;  // H = I (LAPACK dlarfg: tau = 0)
        s_scal[1] = 0.0;
      } else {
        const double nrm = sqrt(x0 * x0 + s);
        const double beta = x0 >= 0.0 ? -nrm : nrm;
        // v = x - beta e1, normalised so that H = I - 2 v v^T / (v^T v)
        const double v0 = x0 - beta;
        s_scal[0] = v0;
        s_scal[1] = 2.0 / (v0 * v0 + s);  // 2 / (v^T v)
        W[(size_t)j * l + j] = beta;
      }
    }
    __syncthreads();
    const double v0 = s_scal[0], tau = s_scal[1];
    // store v in V[:, j] (rows >= j)
    for (int r = j + tid; r < m; r += blockDim.x) V[(size_t)r * l + j] = (r == j) ? v0 : W[(size_t)r * l + j];
    __syncthreads();
    if (tau != 0.0) {
      // dots for columns c > j: d_c = v^T W[j:, c]
      for (int c = j + 1 + warp; c < l; c += nw) {
        double d = 0.0;
        for (int r = j + lane; r < m; r += 32) d = fma(V[(size_t)r * l + j], (r == j) ? W[(size_t)j * l + c] : W[(size_t)r * l + c], d);
        d = warp_sum(d);
        if (lane == 0) s_dot[c] = d * tau;
      }
      __syncthreads();
      for (int c = j + 1 + warp; c < l; c += nw) {
        const double dc = s_dot[c];
        for (int r = j + lane; r < m; r += 32) W[(size_t)r * l + c] -= dc * V[(size_t)r * l + j];
      }
    }
    if (tid == 0) s_dot[j] = tau;  // remember tau_j (column j no longer needed in s_dot)
    __syncthreads();
    if (tid == 0) W[(size_t)j * l + j] = tau;  // stash tau_j on the diagonal slot of W
    __syncthreads();
  }
  // form Q = H_0 ... H_{l-1} [I; 0] in W; the taus sit on W's diagonal, copy them out first
  double* s_tau = hh_smem + l;
  for (int j = tid; j < l; j += blockDim.x) s_tau[j] = W[(size_t)j * l + j];
  __syncthreads();
  for (size_t e = tid; e < (size_t)m * l; e += blockDim.x) {
    const size_t r = e / l, c = e % l;
    W[e] = (r == c) ? 1.0 : 0.0;
  }
  __syncthreads();
  for (int j = l - 1; j >= 0; --j) {
    const double tau = s_tau[j];
    if (tau == 0.0) continue;
    for (int c = j + warp; c < l; c += nw) {
      double d = 0.0;
      for (int r = j + lane; r < m; r += 32) d = fma(V[(size_t)r * l + j], W[(size_t)r * l + c], d);
      d = warp_sum(d);
      if (lane == 0) s_dot[c] = d * tau;
    }
    __syncthreads();
    for (int c = j + warp; c < l; c += nw) {
      const double dc = s_dot[c];
      for (int r = j + lane; r < m; r += 32) W[(size_t)r * l + c] -= dc * V[(size_t)r * l + j];
    }
    __syncthreads();
  }
  for (size_t e = tid; e < (size_t)m * l; e += blockDim.x) {
    const size_t r = e / l, c = e % l;
    Q[r * qrs + c * qcs] = qout<TO>(W[e], tf32);
    if (Q2) Q2[r * q2rs + c * q2cs] = qout<TO>(W[e], tf32);
  }
}

// ---- fused CholeskyQR2 for sketches that fit one CTA's shared memory (C1: 512 x 40 fp64) ----------
// One CTA (512 threads) does both passes of CholeskyQR2 with Y resident in shared memory (row-major,
// pitch LP = 4 * ceil(l / 4) + 2 doubles: an odd number of 16-byte granules, so the lanes' rows
// spread over the bank groups):
//   Gram      4 x 4 register blocks of the upper block triangle, S row slices per block pair in S
//             consecutive lanes, reduced by a fixed xor-shuffle tree (16 FMAs per 4 LDS.128);
//   Cholesky  right-looking over all threads, two barriers per pivot; the trailing update walks a
//             pair table that lists the triangle from the last row up, so step p's entries are the
//             table's first (l-p-1)(l-p)/2 (one per thread);
//   R^{-1}    rows from the bottom, each row's entries in parallel (4 lanes per entry);
//   apply     Q = Y R^{-1} row-locally in place: thread = row, column chunks of 8 from the last
//             down (chunk c only reads Y columns <= its own, R^{-1} being upper triangular), 8
//             accumulators in registers, each Y value (LDS.64) against a broadcast row of R^{-1}.
// (A one-warp Cholesky and R^{-1} were a serial chain: 47% of the kernel's stalls sat at the barrier
// waiting for them.)
// The ten kernels of the unfused path (Gram partials and reduce, Cholesky-inverse, apply, twice, plus
// the flag reset) become one; the 4 l eps max(diag G) breakdown rule and the Householder fallback
// (the kernel launched after, gated by the flag) are those of cholinv64_kernel.
constexpr int kSmallQRThreads = 512;
constexpr int kSmallQRMaxL = 64;
static int small_lp(int l) { return 4 * (int)ceil_div(l, 4) + 2; }
size_t qr_small_smem(int m, int l) {
  return ((size_t)m * small_lp(l) + 2 * (size_t)l * l + l + 1) * sizeof(double) +
         (size_t)l * (l + 1) / 2 * sizeof(int);
}
bool qr_small_fits(int m, int l) {
  return l <= kSmallQRMaxL && m <= kSmallQRThreads && m > 2 * l && qr_small_smem(m, l) <= 220 * 1024;
}

template <typename TI, typename TO>
__global__ void __launch_bounds__(kSmallQRThreads) qr_small_kernel(const TI* __restrict__ Y, int64_t rs, int64_t cs,
                                                                   int m, int l, int* __restrict__ flag,
                                                                   TO* __restrict__ Q, int64_t qrs, int64_t qcs,
                                                                   TO* __restrict__ Q2, int64_t q2rs, int64_t q2cs,
                                                                   int tf32) {
  extern __shared__ __align__(16) double qs_smem[];
  const int LB = (int)ceil_div(l, 4), LP = 4 * LB + 2;
  double* Ys = qs_smem;                  // m x LP, row-major
  double* G = Ys + (size_t)m * LP;       // l x l: Gram, then R in the upper triangle
  double* X = G + (size_t)l * l;         // l x l: R^{-1} (upper triangle), row-major
  double* rdiag = X + (size_t)l * l;     // 1 / R[j][j] (+ the breakdown tolerance at [l])
  int* pairs = reinterpret_cast<int*>(rdiag + l + 1);
  __shared__ int s_bad;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int e = tid; e < m * LP; e += blockDim.x) {
    const int r = e / LP, i = e - r * LP;
    Ys[e] = i < l ? (double)Y[(size_t)r * rs + (size_t)i * cs] : 0.0;
  }
  for (int e = tid; e < l * (l + 1) / 2; e += blockDim.x) {
    int i = l - 1, rem = e;  // row l-1 has 1 entry, row l-2 has 2, ...
    while (rem >= l - i) { rem -= l - i; --i; }
    pairs[e] = (i << 8) | (i + rem);
  }
  if (tid == 0) s_bad = 0;
  // block pairs (I <= J) and row slices per pair (a power of two <= 32)
  const int npb = LB * (LB + 1) / 2;
  int S = 1;
  while (S < 32 && 2 * S * npb <= (int)blockDim.x) S *= 2;
  __syncthreads();
  for (int pass = 0; pass < 2; ++pass) {
    // ---- Gram (upper block triangle) ----
    const int pr = tid / S, sl = tid - pr * S;
    int I = 0, J = 0;
    if (pr < npb) {
      int rem = pr;
      while (rem >= LB - I) { rem -= LB - I; ++I; }
      J = I + rem;
    }
    double acc[4][4];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) acc[a][b] = 0.0;
    if (pr < npb) {
      for (int r = sl; r < m; r += S) {
        const double2* row = reinterpret_cast<const double2*>(Ys + (size_t)r * LP);
        const double2 a01 = row[2 * I], a23 = row[2 * I + 1], b01 = row[2 * J], b23 = row[2 * J + 1];
        const double av[4] = {a01.x, a01.y, a23.x, a23.y}, bv[4] = {b01.x, b01.y, b23.x, b23.y};
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int b = 0; b < 4; ++b) acc[a][b] = fma(av[a], bv[b], acc[a][b]);
      }
    }
    // the S lanes of a pair are consecutive and aligned: a fixed xor tree over them
    for (int o = 1; o < S; o <<= 1) {
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b] += __shfl_xor_sync(0xffffffffu, acc[a][b], o);
    }
    if (pr < npb && sl == 0) {
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          const int i = 4 * I + a, j = 4 * J + b;
          if (i <= j && j < l) G[i * l + j] = acc[a][b];
        }
    }
    __syncthreads();
    // ---- Cholesky (right-looking, all threads: two barriers per pivot) ----
    if (tid < 32) {
      double md = 0.0;
      for (int i = lane; i < l; i += 32) md = fmax(md, G[i * l + i]);
      for (int o = 16; o > 0; o >>= 1) md = fmax(md, __shfl_xor_sync(0xffffffffu, md, o));
      if (lane == 0) rdiag[l] = 4.0 * l * 2.220446049250313e-16 * md;  // breakdown tolerance
    }
    __syncthreads();
    const double tol = rdiag[l];
    for (int p = 0; p < l; ++p) {
      double piv = G[p * l + p];
      if (!(piv > tol)) {
        if (tid == 0) s_bad = 1;
        piv = 1.0;
      }
      const double rsq = rsqrt(piv);
      __syncthreads();  // every thread has read the pivot
      for (int j = p + 1 + tid; j < l; j += blockDim.x) G[p * l + j] *= rsq;
      if (tid == 0) {
        G[p * l + p] = piv * rsq;
        rdiag[p] = rsq;
      }
      __syncthreads();
      const int T = (l - p - 1) * (l - p) / 2;
      for (int e = tid; e < T; e += blockDim.x) {
        const int ij = pairs[e], i = ij >> 8, j = ij & 255;
        G[i * l + j] = fma(-G[p * l + i], G[p * l + j], G[i * l + j]);
      }
    }
    __syncthreads();
    if (s_bad) {
      if (tid == 0) *flag = 1;  // the Householder kernel recomputes Q
      return;
    }
    // ---- X = R^{-1} (upper), rows from the bottom: X[i][j] = -rdiag[i] sum_{q=i+1..j} R[i][q] X[q][j];
    // row i's entries are independent, each summed by 4 lanes (fixed xor tree) ----
    for (int i = l - 1; i >= 0; --i) {
      const int j = i + (tid >> 2), part = tid & 3;
      double t = 0.0;
      if (j < l && j > i)
        for (int q = i + 1 + part; q <= j; q += 4) t = fma(G[i * l + q], X[q * l + j], t);
      t += __shfl_xor_sync(0xffffffffu, t, 1);
      t += __shfl_xor_sync(0xffffffffu, t, 2);
      if (part == 0 && j < l) X[i * l + j] = j == i ? rdiag[i] : -t * rdiag[i];
      __syncthreads();
    }
    // ---- apply: row r of Q = row r of Y times R^{-1}, in place. The row is the thread's alone, and
    // the column chunks of 8 go from the last down: chunk c reads Y columns <= its own (X upper
    // triangular), all still unwritten ----
    if (tid < m) {
      double* yr = Ys + (size_t)tid * LP;
      for (int c0 = 8 * ((l - 1) >> 3); c0 >= 0; c0 -= 8) {
        double qv[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) qv[u] = 0.0;
        const int kend = min(l, c0 + 8);
        for (int k = 0; k < kend; ++k) {
          const double y = yr[k];
          const double* xk = X + k * l + c0;
#pragma unroll
          for (int u = 0; u < 8; ++u)
            if (c0 + u < l && c0 + u >= k) qv[u] = fma(y, xk[u], qv[u]);
        }
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (c0 + u < l) yr[c0 + u] = qv[u];
      }
    }
    __syncthreads();
  }
  for (int e = tid; e < m * l; e += blockDim.x) {
    const int r = e / l, i = e - r * l;
    const double v = Ys[(size_t)r * LP + i];
    Q[(size_t)r * qrs + (size_t)i * qcs] = qout<TO>(v, tf32);
    if (Q2) Q2[(size_t)r * q2rs + (size_t)i * q2cs] = qout<TO>(v, tf32);
  }
}

__global__ void reset_flag_kernel(int* flag, int v) {
  pdl_trigger();
  pdl_wait();
  flag[0] = v;
  flag[2] = 0;  // the fused QR's barrier counter
}
__global__ void flag_to_double_kernel(const int* flag, double* out) { *out = (double)*flag; }

int launch_flag_to_double(const int* flag, double* out, cudaStream_t st) {
  flag_to_double_kernel<<<1, 1, 0, st>>>(flag, out);
  APX_LAUNCH_CHECK();
  return OK;
}

// ------------------------------------------------------------------------------------------
size_t qr_ws_bytes(int m, int l) {
  Workspace ws(nullptr, 0, true);
  const int rows_per = 64;
  const int parts = (int)ceil_div(m, rows_per);
  ws.take<double>((size_t)parts * l * l);
  ws.take<double>((size_t)l * l);       // G
  ws.take<double>((size_t)l * l);       // R
  ws.take<double>((size_t)l);           // 1 / diag(R)
  ws.take<double>((size_t)m * l);       // Q1 (fp64)
  ws.take<double>((size_t)m * l);       // W (householder)
  ws.take<double>((size_t)m * l);       // V (householder)
  ws.take<int>(4);                      // flag
  return ws.off;
}

template <typename TI, typename TO>
static int launch_apply(const TI* Y, int64_t rs, int64_t cs, int m, int l, const double* Rinv, const double* rdiag,
                        const int* flag, TO* Q, int64_t qrs, int64_t qcs, TO* Q2, int64_t q2rs, int64_t q2cs,
                        cudaStream_t st, int tf32 = 0) {
  const size_t smem = (size_t)(l * l + l) * sizeof(double);
  const int blocks = (int)std::min<int64_t>(ceil_div(m, 8), kNumSMs);
  const int lw = (int)ceil_div(l, 32);
#define APX_APPLY(LWV)                                                                                     \
  {                                                                                                        \
    auto fn = apply_rinv_kernel<TI, TO, LWV>;                                                              \
    APX_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));            \
    APX_CUDA(launch_pdl(fn, dim3(blocks), dim3(256), smem, st, Y, rs, cs, m, l, Rinv, rdiag, flag, Q, qrs, qcs, Q2, \
                        q2rs, q2cs, tf32));                                                                \
  }
  if (lw == 1) APX_APPLY(1) else if (lw == 2) APX_APPLY(2) else if (lw == 3) APX_APPLY(3) else APX_APPLY(4)
#undef APX_APPLY
  APX_LAUNCH_CHECK();
  return OK;
}

template <typename TI>
static int launch_gram(const TI* Y, int64_t rs, int64_t cs, int m, int l, const int* skip, double* part, double* G,
                       cudaStream_t st) {
  const int parts = (int)ceil_div(m, 64);
  if (l <= 64) {
    APX_CUDA(launch_pdl(gram_partial_kernel<TI>, dim3(parts), dim3(256), 0, st, Y, rs, cs, m, l, skip, part));
    APX_LAUNCH_CHECK();
  } else {
    const size_t smem = (size_t)64 * (ceil_div(l, 4) * 4 + 4) * sizeof(double);
    auto fn = gram_partial_wide_kernel<TI>;
    APX_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    APX_CUDA(launch_pdl(fn, dim3(parts), dim3(256), smem, st, Y, rs, cs, m, l, 64, skip, part));
    APX_LAUNCH_CHECK();
  }
  APX_CUDA(launch_pdl(gram_reduce_kernel, dim3((unsigned)ceil_div(l * l, 32)), dim3(256), 0, st, (const double*)part,
                      parts, l, skip, G));
  APX_LAUNCH_CHECK();
  return OK;
}

static int launch_chol(const double* G, int l, double* R, double* rdiag, int* flag, cudaStream_t st) {
  if (l <= 64) {
    APX_CUDA(launch_pdl(chol64_kernel, dim3(1), dim3(64), 0, st, G, l, R, rdiag, flag));
    APX_LAUNCH_CHECK();
    return OK;
  }
  const size_t smem = (size_t)l * l * sizeof(double);
  APX_CUDA(cudaFuncSetAttribute(chol_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  APX_CUDA(launch_pdl(chol_kernel, dim3(1), dim3(32), smem, st, G, l, R, rdiag, flag));
  APX_LAUNCH_CHECK();
  return OK;
}

// Q (m x l, strides qrs/qcs) = orth(Y); optional second copy Q2 (e.g. Q^T). method: 0 auto,
// 1 force Householder. tf32: round the fp32 outputs to the nearest TF32 value (the TF32 tensor
// core operand paths; see qout).
// the fused CholeskyQR2 applies when its one-tile-per-CTA grid fits co-resident (one CTA per SM),
// outside graph capture (concurrent captured products would compete for co-residency);
// APX_QR_UNFUSED=1 selects the kernel chain (A/B)
static bool cqr_fused_ok(int m, cudaStream_t st) {
  static const bool off = getenv("APX_QR_UNFUSED") != nullptr;
  if (off) return false;
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(st, &cap) != cudaSuccess || cap != cudaStreamCaptureStatusNone) return false;
  const int tiles = (int)ceil_div(m, 64);
  return ceil_div(tiles, cqr_tpc(tiles)) <= device_sms();
}

// SMs the fused QR of an m x l sketch occupies (0 when it takes the unfused chain)
int qr_sm_footprint(int m, int l) {
  if (l > 64 || getenv("APX_QR_UNFUSED") != nullptr) return 0;
  const int tiles = (int)ceil_div(m, 64);
  return (int)ceil_div(tiles, cqr_tpc(tiles));
}

template <typename TI, typename TO>
int qr_orthonormalize(const TI* Y, int64_t rs, int64_t cs, int m, int l, TO* Q, int64_t qrs, int64_t qcs, TO* Q2,
                      int64_t q2rs, int64_t q2cs, void* wsp, size_t ws_bytes, int method, cudaStream_t st,
                      int tf32) {
  APX_REQUIRE(l >= 1 && l <= kMaxHouseholderL, "sketch width %d outside [1, %d]", l, kMaxHouseholderL);
  APX_REQUIRE(m >= l, "need at least as many rows as columns, got %d x %d", m, l);
  Workspace ws(wsp, ws_bytes);
  const int parts = (int)ceil_div(m, 64);
  double* part = ws.take<double>((size_t)parts * l * l);
  double* G = ws.take<double>((size_t)l * l);
  double* Rinv = ws.take<double>((size_t)l * l);
  double* rdiag = ws.take<double>((size_t)l);
  double* Q1 = ws.take<double>((size_t)m * l);
  double* W = ws.take<double>((size_t)m * l);
  double* V = ws.take<double>((size_t)m * l);
  int* flag = ws.take<int>(4);
  APX_WS_CHECK(ws);
  // wide sketches (l > kMaxL: beyond the register-blocked Cholesky/apply kernels) take the
  // Householder path too
  const bool householder_only = method == 1 || m <= 2 * l || l > kMaxL;
  APX_CUDA(launch_pdl(reset_flag_kernel, dim3(1), dim3(1), 0, st, flag, householder_only ? 1 : 0));
  APX_LAUNCH_CHECK();
  // APX_QR_FUSED=1: fp64 sketches that fit one CTA take the fused CholeskyQR2 (qr_small_kernel). It
  // is off by default: one CTA runs the O(m l^2) work latency-bound on a single SM, 160 us per QR
  // at 512 x 40 against ~110 us for the unfused chain whose Gram and apply kernels spread over the
  // SMs (C1: 2.98 vs 2.38 ms per product, batched 7.9k vs 10.1k products/s).
  static const bool fused = getenv("APX_QR_FUSED") != nullptr;
  const bool small = fused && !householder_only && sizeof(TO) == 8 && qr_small_fits(m, l);
  if (small) {
    const size_t smem = qr_small_smem(m, l);
    APX_CUDA(cudaFuncSetAttribute(qr_small_kernel<TI, TO>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    qr_small_kernel<TI, TO><<<1, kSmallQRThreads, smem, st>>>(Y, rs, cs, m, l, flag, Q, qrs, qcs, Q2, q2rs, q2cs,
                                                               tf32);
    APX_LAUNCH_CHECK();
  } else if (!householder_only && l <= 64 && cqr_fused_ok(m, st)) {
    // fused CholeskyQR2: one cooperative launch (cqr2_fused_kernel); pass-2 rule as below
    const double skip_kappa = sizeof(TO) == 4 ? 3.0e4 : (method == 2 ? 1.0e4 : 0.0);
    double* part2 = W;  // m l >= parts l^2 doubles
    const int tpc = cqr_tpc(parts);
    auto go = [&](auto kern, size_t smem) -> int {
      APX_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3((unsigned)ceil_div(parts, tpc));
      cfg.blockDim = dim3(256);
      cfg.dynamicSmemBytes = smem;
      cfg.stream = st;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeCooperative;
      attr[0].val.cooperative = 1;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      APX_CUDA(cudaLaunchKernelEx(&cfg, kern, Y, rs, cs, m, l, part, part2, G, Rinv, flag, Q, qrs, qcs, Q2, q2rs, q2cs,
                                  tf32, skip_kappa));
      APX_LAUNCH_CHECK();
      return OK;
    };
    if (tpc == 2) APX_TRY(go(cqr2_fused_kernel<TI, TO, 2>, sizeof(CqrSmem<2>)));
    else APX_TRY(go(cqr2_fused_kernel<TI, TO, 1>, sizeof(CqrSmem<1>)));
    for (int mk = 12; mk <= 15; ++mk) stage_mark(mk, st);
  } else if (!householder_only && l <= 64) {
    // fast path: CholeskyQR with R^{-1}; second pass only when the conditioning requires it
    int* skip2 = flag + 1;
    // one fp64 CholeskyQR pass leaves ||Q^T Q - I|| <~ u64 kappa^2: fp32 outputs tolerate kappa_F up
    // to 3e4 (TF32-level orthogonality); fp64 outputs always take the second pass
    // (APX_QR_KAPPA64 = a kappa_F threshold for fp64, tuning knob: at 100-300 the C1 sketches,
    // kappa_F above that, still took both passes -- 1.31 ms either way)
    static const double k64 = [] {
      const char* e = getenv("APX_QR_KAPPA64");
      return e ? atof(e) : 0.0;
    }();
    // method 2 (an intermediate QR of a power iteration: only the spanned subspace matters, and a
    // one-pass Q with ||Q^T Q - I|| ~ u kappa^2 spans it as well as a two-pass one): fp64 outputs
    // skip pass 2 up to kappa_F = 1e4 too
    const double skip_kappa = sizeof(TO) == 4 ? 3.0e4 : (method == 2 ? 1.0e4 : k64);
    const int tiles = (int)ceil_div(m, 64);
    APX_TRY(launch_gram<TI>(Y, rs, cs, m, l, flag, part, G, st));
    stage_mark(12, st);  // fine-grained trace markers (bench.py C4 timeline); no-ops unless armed
    APX_CUDA(launch_cholinv64((const double*)G, l, Rinv, (const int*)flag, flag, skip2, skip_kappa, st));
    APX_LAUNCH_CHECK();
    stage_mark(13, st);
    APX_CUDA(cudaFuncSetAttribute(apply_x_kernel<TI, TO>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kApplySmem));
    APX_CUDA(cudaFuncSetAttribute(apply_x_kernel<double, TO>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kApplySmem));
    APX_CUDA(launch_pdl(apply_x_kernel<TI, TO>, dim3(tiles), dim3(256), kApplySmem, st, Y, rs, cs, m, l,
                        (const double*)Rinv, (const int*)flag, (const int*)skip2, Q1, Q, qrs, qcs, Q2, q2rs, q2cs,
                        tf32));
    APX_LAUNCH_CHECK();
    stage_mark(14, st);
    APX_TRY(launch_gram<double>(Q1, l, 1, m, l, skip2, part, G, st));
    APX_CUDA(launch_cholinv64((const double*)G, l, Rinv, (const int*)skip2, flag, (int*)nullptr, 0.0, st));
    APX_LAUNCH_CHECK();
    APX_CUDA(launch_pdl(apply_x_kernel<double, TO>, dim3(tiles), dim3(256), kApplySmem, st, (const double*)Q1,
                        (int64_t)l, (int64_t)1, m, l, (const double*)Rinv, (const int*)skip2, (const int*)nullptr,
                        (double*)nullptr, Q, qrs, qcs, Q2, q2rs, q2cs, tf32));
    APX_LAUNCH_CHECK();
    stage_mark(15, st);
  } else if (!householder_only) {
    // pass 1: Q1 = Y R1^{-1} (fp64)
    APX_TRY(launch_gram<TI>(Y, rs, cs, m, l, flag, part, G, st));
    APX_TRY(launch_chol(G, l, Rinv, rdiag, flag, st));
    APX_TRY((launch_apply<TI, double>(Y, rs, cs, m, l, Rinv, rdiag, flag, Q1, l, 1, (double*)nullptr, 0, 0, st)));
    // pass 2: Q = Q1 R2^{-1}
    APX_TRY(launch_gram<double>(Q1, l, 1, m, l, flag, part, G, st));
    APX_TRY(launch_chol(G, l, Rinv, rdiag, flag, st));
    APX_TRY((launch_apply<double, TO>(Q1, l, 1, m, l, Rinv, rdiag, flag, Q, qrs, qcs, Q2, q2rs, q2cs, st, tf32)));
  }
  const size_t hh_smem = (size_t)2 * l * sizeof(double);
  APX_CUDA(cudaFuncSetAttribute(householder_qr_kernel<TI, TO>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)std::max<size_t>(hh_smem, 48 * 1024)));
  APX_CUDA(launch_pdl(householder_qr_kernel<TI, TO>, dim3(1), dim3(1024), hh_smem, st, Y, rs, cs, m, l,
                      (const int*)flag, 0, W, V, Q, qrs, qcs, Q2, q2rs, q2cs, tf32));
  APX_LAUNCH_CHECK();
  return OK;
}

// ---- row-sharded CholeskyQR (fp32 sketch, l <= 64): the caller all-reduces the Gram matrices ----
// between the steps, so every rank factors the same G and Q_g = Y_g R^{-1} is the row block g of
// the orthonormal Q of the stacked Y. Same kernels and the same pass-2 rule as the fast path of
// qr_orthonormalize; a Cholesky breakdown is reported through flags[0] (no Householder fallback:
// it would need the whole Y on one device).
namespace {
struct RowsQR {
  double *part, *Rinv, *Q1;
  int* flag;  // [0] breakdown, [1] skip pass 2
};
RowsQR plan_rows_qr(Workspace& ws, int m, int l) {
  RowsQR r;
  r.part = ws.take<double>((size_t)ceil_div(m, 64) * l * l);
  r.Rinv = ws.take<double>((size_t)l * l);
  r.Q1 = ws.take<double>((size_t)m * l);
  r.flag = ws.take<int>(4);
  return r;
}
}  // namespace

size_t cholqr_rows_ws(int m, int l) {
  Workspace ws(nullptr, 0, true);
  plan_rows_qr(ws, m, l);
  return ws.off;
}

int cholqr_rows_gram(const float* Y, int m, int l, double* G, void* wsp, size_t bytes, cudaStream_t st) {
  APX_REQUIRE(l >= 1 && l <= 64 && m >= 1, "row-sharded CholeskyQR: l=%d m=%d", l, m);
  Workspace ws(wsp, bytes);
  RowsQR r = plan_rows_qr(ws, m, l);
  APX_WS_CHECK(ws);
  return launch_gram<float>(Y, l, 1, m, l, nullptr, r.part, G, st);
}

int cholqr_rows_pass1(const float* Y, int m, int l, const double* G, float* Q, double* G2, void* wsp, size_t bytes,
                      cudaStream_t st) {
  Workspace ws(wsp, bytes);
  RowsQR r = plan_rows_qr(ws, m, l);
  APX_WS_CHECK(ws);
  APX_CUDA(cudaMemsetAsync(r.flag, 0, 4 * sizeof(int), st));
  APX_CUDA(cudaMemsetAsync(G2, 0, (size_t)l * l * sizeof(double), st));  // stays zero if pass 2 is skipped
  APX_CUDA(launch_cholinv64(G, l, r.Rinv, r.flag, r.flag, r.flag + 1, 3.0e4, st));
  APX_LAUNCH_CHECK();
  APX_CUDA(cudaFuncSetAttribute(apply_x_kernel<float, float>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)kApplySmem));
  apply_x_kernel<float, float><<<(unsigned)ceil_div(m, 64), 256, kApplySmem, st>>>(
      Y, l, 1, m, l, r.Rinv, r.flag, r.flag + 1, r.Q1, Q, l, 1, (float*)nullptr, 0, 0, 1);
  APX_LAUNCH_CHECK();
  return launch_gram<double>(r.Q1, l, 1, m, l, r.flag + 1, r.part, G2, st);
}

int cholqr_rows_pass2(int m, int l, const double* G2, float* Q, void* wsp, size_t bytes, cudaStream_t st) {
  Workspace ws(wsp, bytes);
  RowsQR r = plan_rows_qr(ws, m, l);
  APX_WS_CHECK(ws);
  APX_CUDA(launch_cholinv64(G2, l, r.Rinv, r.flag + 1, r.flag, (int*)nullptr, 0.0, st));
  APX_LAUNCH_CHECK();
  APX_CUDA(cudaFuncSetAttribute(apply_x_kernel<double, float>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)kApplySmem));
  apply_x_kernel<double, float><<<(unsigned)ceil_div(m, 64), 256, kApplySmem, st>>>(
      r.Q1, l, 1, m, l, r.Rinv, r.flag + 1, (const int*)nullptr, (double*)nullptr, Q, l, 1, (float*)nullptr, 0, 0,
      1);
  APX_LAUNCH_CHECK();
  return OK;
}

const int* cholqr_rows_flags(void* wsp, size_t bytes, int m, int l) {
  Workspace ws(wsp, bytes);
  RowsQR r = plan_rows_qr(ws, m, l);
  return r.flag;
}

template int qr_orthonormalize<float, float>(const float*, int64_t, int64_t, int, int, float*, int64_t, int64_t,
                                             float*, int64_t, int64_t, void*, size_t, int, cudaStream_t, int);
template int qr_orthonormalize<double, double>(const double*, int64_t, int64_t, int, int, double*, int64_t, int64_t,
                                               double*, int64_t, int64_t, void*, size_t, int, cudaStream_t, int);

}  // namespace apx
