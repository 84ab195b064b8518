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
template <typename T>
__global__ void __launch_bounds__(256) gram_partial_kernel(const T* __restrict__ Y, int64_t rs, int64_t cs, int m,
                                                           int l, int rows_per, const int* __restrict__ skip,
                                                           double* __restrict__ part) {
  if (skip && *skip) return;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* Ys = reinterpret_cast<double*>(smem_raw);  // rows_per x (l+1)
  const int r0 = blockIdx.x * rows_per;
  const int rows = min(rows_per, m - r0);
  const int S = l + 1;
  for (int e = threadIdx.x; e < rows * l; e += blockDim.x) {
    const int r = e / l, c = e - r * l;
    Ys[r * S + c] = (double)Y[(size_t)(r0 + r) * rs + (size_t)c * cs];
  }
  __syncthreads();
  double* out = part + (size_t)blockIdx.x * l * l;
  for (int e = threadIdx.x; e < l * l; e += blockDim.x) {
    const int i = e / l, j = e - i * l;
    double s = 0.0;
    if (j >= i) {
      for (int r = 0; r < rows; ++r) s = fma(Ys[r * S + i], Ys[r * S + j], s);
    }
    out[e] = s;
  }
}

__global__ void gram_reduce_kernel(const double* __restrict__ part, int parts, int l, const int* __restrict__ skip,
                                   double* __restrict__ G) {
  if (skip && *skip) return;
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= l * l) return;
  double s = 0.0;
  for (int p = 0; p < parts; ++p) s += part[(size_t)p * l * l + e];
  G[e] = s;
}

// ---- one-CTA Cholesky (upper R, G = R^T R) + inverse of R ---------------------------------
__global__ void __launch_bounds__(1024) chol_inv_kernel(const double* __restrict__ Gin, int l,
                                                        double* __restrict__ Rinv, int* __restrict__ flag) {
  if (*flag) return;
  // One l x l buffer: the upper triangle holds G and is factored in place into R (G = R^T R);
  // the strictly lower triangle then receives X = R^{-1} transposed (X[i][c] at (c, i)), with
  // X's diagonal in a separate vector. 128 KB at l = 128.
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* Gs = reinterpret_cast<double*>(smem_raw);
  __shared__ double xdiag[kMaxL];
  __shared__ double s_maxd;
  __shared__ int s_bad;
  const int tid = threadIdx.x;
  for (int e = tid; e < l * l; e += blockDim.x) {
    const int i = e / l, j = e - i * l;
    Gs[e] = i <= j ? Gin[e] : 0.0;
  }
  __syncthreads();
  if (tid == 0) {
    double md = 0.0;
    for (int i = 0; i < l; ++i) md = fmax(md, Gs[i * l + i]);
    s_maxd = md;
    s_bad = 0;
  }
  __syncthreads();
  const double tol = 4.0 * l * 2.220446049250313e-16 * s_maxd;
  for (int j = 0; j < l; ++j) {
    if (tid == 0) {
      const double d2 = Gs[j * l + j];
      if (!(d2 > tol)) s_bad = 1;
      Gs[j * l + j] = sqrt(fmax(d2, 0.0));
    }
    __syncthreads();
    if (s_bad) break;
    const double inv = 1.0 / Gs[j * l + j];
    for (int c = j + 1 + tid; c < l; c += blockDim.x) Gs[j * l + c] *= inv;
    __syncthreads();
    const int rem = l - j - 1;
    for (int e = tid; e < rem * rem; e += blockDim.x) {
      const int r = j + 1 + e / rem, c = j + 1 + e % rem;
      if (c >= r) Gs[r * l + c] -= Gs[j * l + r] * Gs[j * l + c];
    }
    __syncthreads();
  }
  if (s_bad) {
    if (tid == 0) *flag = 1;
    return;
  }
  // X = R^{-1} (upper), column c by back substitution; thread c owns row c of the lower part
  for (int c = tid; c < l; c += blockDim.x) {
    const double xc = 1.0 / Gs[c * l + c];
    xdiag[c] = xc;
    for (int i = c - 1; i >= 0; --i) {
      double s = Gs[i * l + c] * xc;  // j = c term
      for (int j2 = i + 1; j2 < c; ++j2) s = fma(Gs[i * l + j2], Gs[c * l + j2], s);
      Gs[c * l + i] = -s / Gs[i * l + i];
    }
  }
  __syncthreads();
  for (int e = tid; e < l * l; e += blockDim.x) {
    const int i = e / l, c = e - i * l;
    Rinv[e] = i < c ? Gs[c * l + i] : (i == c ? xdiag[c] : 0.0);
  }
}

// ---- Q = Y R^{-1}; warp per row, R^{-1} in shared memory ---------------------------------
template <typename TI, typename TO, int LW>
__global__ void __launch_bounds__(256) apply_rinv_kernel(const TI* __restrict__ Y, int64_t rs, int64_t cs, int m,
                                                         int l, const double* __restrict__ Rinv,
                                                         const int* __restrict__ flag, TO* __restrict__ Q,
                                                         int64_t qrs, int64_t qcs, TO* __restrict__ Q2, int64_t q2rs,
                                                         int64_t q2cs) {
  if (*flag) return;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* Rs = reinterpret_cast<double*>(smem_raw);
  for (int e = threadIdx.x; e < l * l; e += blockDim.x) Rs[e] = Rinv[e];
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
      for (int i = 0; i < 32; ++i) {
        const int ii = 32 * q + i;
        if (ii >= l) break;
        const double yi = __shfl_sync(0xffffffffu, y[q], i);
#pragma unroll
        for (int p = 0; p < LW; ++p) {
          const int c = lane + 32 * p;
          if (c < l) acc[p] = fma(yi, Rs[ii * l + c], acc[p]);
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
  ws.take<double>((size_t)l * l);       // Rinv
  ws.take<double>((size_t)m * l);       // Q1 (fp64)
  ws.take<double>((size_t)m * l);       // W (householder)
  ws.take<double>((size_t)m * l);       // V (householder)
  ws.take<int>(4);                      // flag
  return ws.off;
}

template <typename TI, typename TO>
static int launch_apply(const TI* Y, int64_t rs, int64_t cs, int m, int l, const double* Rinv, const int* flag,
                        TO* Q, int64_t qrs, int64_t qcs, TO* Q2, int64_t q2rs, int64_t q2cs, cudaStream_t st) {
  const size_t smem = (size_t)l * l * sizeof(double);
  const int blocks = (int)std::min<int64_t>(ceil_div(m, 8), kNumSMs * 4);
  const int lw = (int)ceil_div(l, 32);
#define APX_APPLY(LWV)                                                                                     \
  {                                                                                                        \
    auto fn = apply_rinv_kernel<TI, TO, LWV>;                                                              \
    APX_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));            \
    fn<<<blocks, 256, smem, st>>>(Y, rs, cs, m, l, Rinv, flag, Q, qrs, qcs, Q2, q2rs, q2cs);               \
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
  const size_t smem = (size_t)rows_per * (l + 1) * sizeof(double);
  auto fn = gram_partial_kernel<TI>;
  APX_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  fn<<<parts, 256, smem, st>>>(Y, rs, cs, m, l, rows_per, skip, part);
  APX_LAUNCH_CHECK();
  gram_reduce_kernel<<<(unsigned)ceil_div(l * l, 256), 256, 0, st>>>(part, parts, l, skip, G);
  APX_LAUNCH_CHECK();
  return OK;
}

static int launch_chol(const double* G, int l, double* Rinv, int* flag, cudaStream_t st) {
  const size_t smem = (size_t)l * l * sizeof(double);
  APX_CUDA(cudaFuncSetAttribute(chol_inv_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  chol_inv_kernel<<<1, 1024, smem, st>>>(G, l, Rinv, flag);
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
  double* Q1 = ws.take<double>((size_t)m * l);
  double* W = ws.take<double>((size_t)m * l);
  double* V = ws.take<double>((size_t)m * l);
  int* flag = ws.take<int>(4);
  APX_WS_CHECK(ws);
  const bool householder_only = method == 1 || m <= 2 * l;
  reset_flag_kernel<<<1, 1, 0, st>>>(flag, householder_only ? 1 : 0);
  APX_LAUNCH_CHECK();
  if (!householder_only) {
    // pass 1: Q1 = Y R1^{-1} (fp64)
    APX_TRY(launch_gram<TI>(Y, rs, cs, m, l, flag, part, G, st));
    APX_TRY(launch_chol(G, l, Rinv, flag, st));
    APX_TRY((launch_apply<TI, double>(Y, rs, cs, m, l, Rinv, flag, Q1, l, 1, (double*)nullptr, 0, 0, st)));
    // pass 2: Q = Q1 R2^{-1}
    APX_TRY(launch_gram<double>(Q1, l, 1, m, l, flag, part, G, st));
    APX_TRY(launch_chol(G, l, Rinv, flag, st));
    APX_TRY((launch_apply<double, TO>(Q1, l, 1, m, l, Rinv, flag, Q, qrs, qcs, Q2, q2rs, q2cs, st)));
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
