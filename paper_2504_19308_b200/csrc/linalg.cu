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

constexpr int kMaxL = 128;

// ---- Gram partials: G_p = Y[rows_p]^T Y[rows_p] -------------------------------------------
// 64 rows per CTA staged as fp64 in shared memory; thread t owns a 4x4 block (bi, bj) of G
// (upper block triangle only), so each pair of 4-wide row loads feeds 16 FMAs.
template <typename T>
__global__ void __launch_bounds__(256) gram_partial_kernel(const T* __restrict__ Y, int64_t rs, int64_t cs, int m,
                                                           int l, int rows_per, const int* __restrict__ skip,
                                                           double* __restrict__ part) {
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
// 128 threads: thread (c = tid & 63, h = tid >> 6) keeps rows [32h, 32h+32) of column c of G in
// registers; each of the l pivot steps costs three 128-thread barriers and <= 32 predicated FMAs
// per thread. Then X = R^{-1} is formed column-parallel in shared memory (reciprocal diagonal,
// no divisions), and kappa_F = ||R||_F ||X||_F >= cond_2(Y) decides whether CholeskyQR's second
// pass can be skipped: with fp32 outputs one fp64 pass already leaves ||Q^T Q - I|| <~
// u64 * kappa^2, so kappa_F <= skip_kappa skips pass 2 (flag_skip = 1).
__global__ void __launch_bounds__(128) cholinv64_kernel(const double* __restrict__ Gin, int l, double* __restrict__ Xout,
                                                        const int* __restrict__ gate, int* __restrict__ breakdown,
                                                        int* __restrict__ skip_out, double skip_kappa) {
  if (*gate) return;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* Rs = reinterpret_cast<double*>(smem_raw);  // 64 x 65
  double* Xs = Rs + 64 * 65;                          // 64 x 65
  __shared__ double rowj[64];
  __shared__ double rinv[64];
  __shared__ double red[32];
  __shared__ double s_inv;
  __shared__ int s_bad;
  const int tid = threadIdx.x, c = tid & 63, h = tid >> 6;
  double g[32];
#pragma unroll
  for (int rr = 0; rr < 32; ++rr) {
    const int r = 32 * h + rr;
    g[rr] = (c < l && r <= c) ? Gin[r * l + c] : 0.0;
  }
  // max diagonal -> breakdown tolerance
  double dg = 0.0;
#pragma unroll
  for (int rr = 0; rr < 32; ++rr)
    if (32 * h + rr == c) dg = g[rr];
  rowj[c] = 0.0;
  __syncthreads();
  if (c < l && (c >> 5) == h) rowj[c] = dg;
  if (tid == 0) s_bad = 0;
  __syncthreads();
  double md = 0.0;
  for (int i = 0; i < l; ++i) md = fmax(md, rowj[i]);
  const double tol = 4.0 * l * 2.220446049250313e-16 * md;
  __syncthreads();
#pragma unroll 1
  for (int j = 0; j < l; ++j) {
    const int hj = j >> 5, jj = j & 31;
    if (c == j && h == hj) {
      double d2 = 0.0;
#pragma unroll
      for (int rr = 0; rr < 32; ++rr)
        if (rr == jj) d2 = g[rr];
      if (!(d2 > tol)) s_bad = 1;
      const double inv = rsqrt(fmax(d2, 1e-300));
      s_inv = inv;
      rinv[j] = inv;
#pragma unroll
      for (int rr = 0; rr < 32; ++rr)
        if (rr == jj) g[rr] = d2 * inv;
    }
    __syncthreads();
    if (s_bad) break;
    if (c > j && c < l && h == hj) {
      const double inv = s_inv;
      double rjc = 0.0;
#pragma unroll
      for (int rr = 0; rr < 32; ++rr)
        if (rr == jj) { g[rr] *= inv; rjc = g[rr]; }
      rowj[c] = rjc;
    }
    __syncthreads();
    if (c > j && c < l) {
      const double rjc = rowj[c];
#pragma unroll
      for (int rr = 0; rr < 32; ++rr) {
        const int r = 32 * h + rr;
        if (r > j && r <= c) g[rr] = fma(-rowj[r], rjc, g[rr]);
      }
    }
    __syncthreads();
  }
  if (s_bad) {
    if (tid == 0) {
      *breakdown = 1;
      if (skip_out) *skip_out = 1;
    }
    return;
  }
  // R (upper) to shared memory
#pragma unroll
  for (int rr = 0; rr < 32; ++rr) {
    const int r = 32 * h + rr;
    if (r < 64) Rs[r * 65 + c] = (c < l && r <= c) ? g[rr] : 0.0;
  }
  __syncthreads();
  // X = R^{-1}: thread c < l solves R x = e_c by back substitution (column c of X)
  if (tid < l) {
    for (int i = l - 1; i >= 0; --i) {
      double sacc = (i == c) ? 1.0 : 0.0;
      if (i <= c) {
        for (int k = i + 1; k <= c; ++k) sacc = fma(-Rs[i * 65 + k], Xs[k * 65 + c], sacc);
      } else {
        sacc = 0.0;
      }
      Xs[i * 65 + c] = (i <= c) ? sacc * rinv[i] : 0.0;
    }
  }
  __syncthreads();
  // kappa_F = ||R||_F ||X||_F
  double r2 = 0.0, x2 = 0.0;
  for (int e = tid; e < l * l; e += blockDim.x) {
    const int i = e / l, k = e - i * l;
    const double rv = Rs[i * 65 + k], xv = Xs[i * 65 + k];
    r2 = fma(rv, rv, r2);
    x2 = fma(xv, xv, x2);
    Xout[e] = xv;
  }
  r2 = block_sum(r2, red);
  __syncthreads();
  x2 = block_sum(x2, red);
  if (tid == 0 && skip_out) *skip_out = (sqrt(r2) * sqrt(x2) <= skip_kappa) ? 1 : 0;
}

// ---- Q = Y X (X = R^{-1} upper), one warp per row; X staged in shared memory ----------------
// Writes the fp64 copy Q1 (input of CholeskyQR's second pass) and/or the typed outputs Q, Q2.
template <typename TI, typename TO, int LW>
__global__ void __launch_bounds__(256) apply_x_kernel(const TI* __restrict__ Y, int64_t rs, int64_t cs, int m, int l,
                                                      const double* __restrict__ X, const int* __restrict__ skip,
                                                      double* __restrict__ Q1, TO* __restrict__ Q, int64_t qrs,
                                                      int64_t qcs, TO* __restrict__ Q2, int64_t q2rs, int64_t q2cs) {
  if (*skip) return;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* Xs = reinterpret_cast<double*>(smem_raw);
  for (int e = threadIdx.x; e < l * l; e += blockDim.x) Xs[e] = X[e];
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int warps = blockDim.x >> 5;
  for (int r = blockIdx.x * warps + (threadIdx.x >> 5); r < m; r += gridDim.x * warps) {
    double y[LW], acc[LW];
#pragma unroll
    for (int q = 0; q < LW; ++q) {
      const int c = lane + 32 * q;
      y[q] = c < l ? (double)Y[(size_t)r * rs + (size_t)c * cs] : 0.0;
      acc[q] = 0.0;
    }
#pragma unroll
    for (int q = 0; q < LW; ++q) {
#pragma unroll 8
      for (int i = 0; i < 32; ++i) {
        const int ii = 32 * q + i;
        const double yi = __shfl_sync(0xffffffffu, y[q], i);
#pragma unroll
        for (int p = 0; p < LW; ++p) {
          const int c = lane + 32 * p;
          if (ii < l && c < l) acc[p] = fma(yi, Xs[ii * l + c], acc[p]);
        }
      }
    }
#pragma unroll
    for (int q = 0; q < LW; ++q) {
      const int c = lane + 32 * q;
      if (c < l) {
        if (Q1) Q1[(size_t)r * l + c] = acc[q];
        if (Q) Q[(size_t)r * qrs + (size_t)c * qcs] = (TO)acc[q];
        if (Q2) Q2[(size_t)r * q2rs + (size_t)c * q2cs] = (TO)acc[q];
      }
    }
  }
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
                                                         int64_t q2cs) {
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
        Q[(size_t)r * qrs + (size_t)c * qcs] = (TO)acc[q];
        if (Q2) Q2[(size_t)r * q2rs + (size_t)c * q2cs] = (TO)acc[q];
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
                                                              int64_t q2rs, int64_t q2cs) {
  if (!force && !(*flag)) return;
  __shared__ double red[32];
  __shared__ double s_dot[kMaxL];
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
  __shared__ double s_tau[kMaxL];
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
    Q[r * qrs + c * qcs] = (TO)W[e];
    if (Q2) Q2[r * q2rs + c * q2cs] = (TO)W[e];
  }
}

__global__ void reset_flag_kernel(int* flag, int v) { *flag = v; }

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
                        cudaStream_t st) {
  const size_t smem = (size_t)(l * l + l) * sizeof(double);
  const int blocks = (int)std::min<int64_t>(ceil_div(m, 8), kNumSMs);
  const int lw = (int)ceil_div(l, 32);
#define APX_APPLY(LWV)                                                                                     \
  {                                                                                                        \
    auto fn = apply_rinv_kernel<TI, TO, LWV>;                                                              \
    APX_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));            \
    fn<<<blocks, 256, smem, st>>>(Y, rs, cs, m, l, Rinv, rdiag, flag, Q, qrs, qcs, Q2, q2rs, q2cs);        \
  }
  if (lw == 1) APX_APPLY(1) else if (lw == 2) APX_APPLY(2) else if (lw == 3) APX_APPLY(3) else APX_APPLY(4)
#undef APX_APPLY
  APX_LAUNCH_CHECK();
  return OK;
}

template <typename TI>
static int launch_gram(const TI* Y, int64_t rs, int64_t cs, int m, int l, const int* skip, double* part, double* G,
                       cudaStream_t st) {
  const int rows_per = 64;
  const int parts = (int)ceil_div(m, rows_per);
  const size_t smem = (size_t)rows_per * (ceil_div(l, 4) * 4 + 4) * sizeof(double);
  auto fn = gram_partial_kernel<TI>;
  APX_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  fn<<<parts, 256, smem, st>>>(Y, rs, cs, m, l, rows_per, skip, part);
  APX_LAUNCH_CHECK();
  gram_reduce_kernel<<<(unsigned)ceil_div(l * l, 32), 256, 0, st>>>(part, parts, l, skip, G);
  APX_LAUNCH_CHECK();
  return OK;
}

static int launch_chol(const double* G, int l, double* R, double* rdiag, int* flag, cudaStream_t st) {
  if (l <= 64) {
    chol64_kernel<<<1, 64, 0, st>>>(G, l, R, rdiag, flag);
    APX_LAUNCH_CHECK();
    return OK;
  }
  const size_t smem = (size_t)l * l * sizeof(double);
  APX_CUDA(cudaFuncSetAttribute(chol_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  chol_kernel<<<1, 32, smem, st>>>(G, l, R, rdiag, flag);
  APX_LAUNCH_CHECK();
  return OK;
}

// Q (m x l, strides qrs/qcs) = orth(Y); optional second copy Q2 (e.g. Q^T). method: 0 auto,
// 1 force Householder.
template <typename TI, typename TO>
int qr_orthonormalize(const TI* Y, int64_t rs, int64_t cs, int m, int l, TO* Q, int64_t qrs, int64_t qcs, TO* Q2,
                      int64_t q2rs, int64_t q2cs, void* wsp, size_t ws_bytes, int method, cudaStream_t st) {
  APX_REQUIRE(l >= 1 && l <= kMaxL, "sketch width %d outside [1, %d]", l, kMaxL);
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
  const bool householder_only = method == 1 || m <= 2 * l;
  reset_flag_kernel<<<1, 1, 0, st>>>(flag, householder_only ? 1 : 0);
  APX_LAUNCH_CHECK();
  if (!householder_only && l <= 64) {
    // fast path: CholeskyQR with R^{-1}; second pass only when the conditioning requires it
    int* skip2 = flag + 1;
    const double skip_kappa = sizeof(TO) == 4 ? 3.0e4 : 0.0;
    const size_t smem = (size_t)l * l * sizeof(double);
    const int blocks = (int)std::min<int64_t>(ceil_div(m, 8), kNumSMs);
    const int lw = (int)ceil_div(l, 32);
    const size_t csmem = 2 * 64 * 65 * sizeof(double);
    APX_CUDA(cudaFuncSetAttribute(cholinv64_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)csmem));
    APX_TRY(launch_gram<TI>(Y, rs, cs, m, l, flag, part, G, st));
    cholinv64_kernel<<<1, 128, csmem, st>>>(G, l, Rinv, flag, flag, skip2, skip_kappa);
    APX_LAUNCH_CHECK();
    {
      auto fn = lw == 1 ? apply_x_kernel<TI, TO, 1> : apply_x_kernel<TI, TO, 2>;
      APX_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      fn<<<blocks, 256, smem, st>>>(Y, rs, cs, m, l, Rinv, flag, Q1, Q, qrs, qcs, Q2, q2rs, q2cs);
      APX_LAUNCH_CHECK();
    }
    APX_TRY(launch_gram<double>(Q1, l, 1, m, l, skip2, part, G, st));
    cholinv64_kernel<<<1, 128, csmem, st>>>(G, l, Rinv, skip2, flag, (int*)nullptr, 0.0);
    APX_LAUNCH_CHECK();
    {
      auto fn = lw == 1 ? apply_x_kernel<double, TO, 1> : apply_x_kernel<double, TO, 2>;
      APX_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      fn<<<blocks, 256, smem, st>>>(Q1, l, 1, m, l, Rinv, skip2, (double*)nullptr, Q, qrs, qcs, Q2, q2rs, q2cs);
      APX_LAUNCH_CHECK();
    }
  } else if (!householder_only) {
    // pass 1: Q1 = Y R1^{-1} (fp64)
    APX_TRY(launch_gram<TI>(Y, rs, cs, m, l, flag, part, G, st));
    APX_TRY(launch_chol(G, l, Rinv, rdiag, flag, st));
    APX_TRY((launch_apply<TI, double>(Y, rs, cs, m, l, Rinv, rdiag, flag, Q1, l, 1, (double*)nullptr, 0, 0, st)));
    // pass 2: Q = Q1 R2^{-1}
    APX_TRY(launch_gram<double>(Q1, l, 1, m, l, flag, part, G, st));
    APX_TRY(launch_chol(G, l, Rinv, rdiag, flag, st));
    APX_TRY((launch_apply<double, TO>(Q1, l, 1, m, l, Rinv, rdiag, flag, Q, qrs, qcs, Q2, q2rs, q2cs, st)));
  }
  householder_qr_kernel<TI, TO><<<1, 1024, 0, st>>>(Y, rs, cs, m, l, flag, 0, W, V, Q, qrs, qcs, Q2, q2rs, q2cs);
  APX_LAUNCH_CHECK();
  return OK;
}

template int qr_orthonormalize<float, float>(const float*, int64_t, int64_t, int, int, float*, int64_t, int64_t,
                                             float*, int64_t, int64_t, void*, size_t, int, cudaStream_t);
template int qr_orthonormalize<double, double>(const double*, int64_t, int64_t, int, int, double*, int64_t, int64_t,
                                               double*, int64_t, int64_t, void*, size_t, int, cudaStream_t);

}  // namespace apx
