// Row-wise Fourier sparsification and the sparsified first-order product (reference fsparse.py).
//
//   At = A W* (row transforms), Bt = W B (column transforms)                 (fsparse.py:195-196)
//   SA = per-row top-k of |At| (ties -> lower column), SB likewise by rows or by columns
//   order 0: M = SA . dense(SB)           (sparse row gather: k nonzeros per row of SA)
//   order 1: M = SA . Bt + (At - SA) . SB (row gather + dense complex GEMM as 4 real DMMA GEMMs)
// Residual norms are the exact Frobenius norms of the dropped entries (fsparse.py:207-208).
#include "../../include/apx.h"
#include "common.cuh"
#include "fft.cuh"
#include "kernels.cuh"
#include "select.cuh"

namespace apx {

// |x| for complex entries, hypot semantics (np.abs)
__global__ void cabs_kernel(const double2* __restrict__ x, size_t cnt, double* __restrict__ out) {
  for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < cnt; e += (size_t)gridDim.x * blockDim.x)
    out[e] = hypot(x[e].x, x[e].y);
}

// batched top-k: CTA b selects budget[b] (or k) largest of w[b*n .. b*n+n), writing ascending
// column indices to sel[b*k ..]; unused slots get -1.
__global__ void __launch_bounds__(kSelThreads) topk_rows_kernel(const double* __restrict__ w, int n, int k,
                                                                const int* __restrict__ budget, int* __restrict__ sel) {
  const int b = blockIdx.x;
  const int kb = budget ? min(budget[b], n) : min(k, n);
  int* out = sel + (size_t)b * k;
  for (int q = threadIdx.x; q < k; q += blockDim.x) out[q] = -1;
  __syncthreads();
  topk_select_block(w + (size_t)b * n, n, kb, out);
}

// kept entries -> dense sparse-matrix image S (zeros elsewhere, optional) and per-row packed
// values; mode_cols: selection is per column of X (sel indexes rows).
__global__ void scatter_kept_kernel(const double2* __restrict__ X, int rows, int cols, const int* __restrict__ sel,
                                    int k, int by_cols, double2* __restrict__ Sdense, double2* __restrict__ vals) {
  const int nb = by_cols ? cols : rows;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < nb * k; e += gridDim.x * blockDim.x) {
    const int b = e / k, q = e - b * k;
    const int j = sel[(size_t)b * k + q];
    double2 v = make_double2(0.0, 0.0);
    APX_DCHECK(j < (by_cols ? rows : cols));
    if (j >= 0) {
      const size_t idx = by_cols ? (size_t)j * cols + b : (size_t)b * cols + j;
      v = X[idx];
      if (Sdense) Sdense[idx] = v;
    }
    if (vals) vals[e] = v;
  }
}

// out[e] = x[e] - s[e] (dropped part), plus per-block partial of |out|^2
__global__ void __launch_bounds__(256) residual_kernel(const double2* __restrict__ x, const double2* __restrict__ s,
                                                       size_t cnt, double2* __restrict__ out,
                                                       double* __restrict__ part) {
  __shared__ double red[32];
  double acc = 0.0;
  for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < cnt; e += (size_t)gridDim.x * blockDim.x) {
    const double2 d = csub(x[e], s[e]);
    if (out) out[e] = d;
    acc = fma(d.x, d.x, fma(d.y, d.y, acc));
  }
  acc = block_sum(acc, red);
  if (threadIdx.x == 0) part[blockIdx.x] = acc;
}

// M[i, :] (+)= sum_q vals[i][q] * X[sel[i][q], :]   (k nonzeros per row of the left factor, any k:
// the entries are staged through shared memory in tiles of kSpTile)
constexpr int kSpTile = 256;
__global__ void __launch_bounds__(256) sparse_rows_gemm_kernel(const int* __restrict__ sel,
                                                               const double2* __restrict__ vals, int k,
                                                               const double2* __restrict__ X, int p, int accumulate,
                                                               double2* __restrict__ M) {
  const int i = blockIdx.x;
  __shared__ int sj[kSpTile];
  __shared__ double2 sv[kSpTile];
  // a CTA covers up to 4 column sweeps of 256 in registers; wider rows loop over column chunks
  for (int c0 = 0; c0 < p; c0 += 4 * blockDim.x) {
    double2 acc[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) acc[u] = make_double2(0.0, 0.0);
    for (int q0 = 0; q0 < k; q0 += kSpTile) {
      const int qn = min(kSpTile, k - q0);
      __syncthreads();  // previous tile consumed
      for (int q = threadIdx.x; q < qn; q += blockDim.x) {
        sj[q] = sel[(size_t)i * k + q0 + q];
        sv[q] = vals[(size_t)i * k + q0 + q];
      }
      __syncthreads();
      for (int q = 0; q < qn; ++q) {
        const int j = sj[q];
        if (j < 0) continue;
        APX_DCHECK(q < kSpTile);
        const double2 v = sv[q];
        const double2* xr = X + (size_t)j * p;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int c = c0 + u * blockDim.x + threadIdx.x;
          if (c < p) acc[u] = cadd(acc[u], cmul(v, xr[c]));
        }
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int c = c0 + u * blockDim.x + threadIdx.x;
      if (c < p) {
        double2* pm = M + (size_t)i * p + c;
        *pm = accumulate ? cadd(*pm, acc[u]) : acc[u];
      }
    }
  }
}

__global__ void split_planes_kernel(const double2* __restrict__ z, size_t cnt, double* __restrict__ re,
                                    double* __restrict__ im) {
  for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < cnt; e += (size_t)gridDim.x * blockDim.x) {
    re[e] = z[e].x;
    im[e] = z[e].y;
  }
}
__global__ void merge_planes_kernel(const double* __restrict__ re, const double* __restrict__ im, size_t cnt,
                                    double2* __restrict__ z) {
  for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < cnt; e += (size_t)gridDim.x * blockDim.x)
    z[e] = cadd(z[e], make_double2(re[e], im[e]));
}

// fourier_row_decompose (fsparse.py:92-105), three passes over F = W(rows):
//  1. per column k (one thread per column, rows in order: coalesced across the warp): F /= sqrt(n)
//     in place and nrm[k] = ||f_k||_2;
//  2. one CTA: ||A||^2 = sum_k n nrm[k]^2 (fixed order) and the transform's rounding floor
//     4 eps log2(n) ||A||: a column whose exact transform is zero (pocketfft returns exact zeros for,
//     e.g., constant rows) comes out of a floating-point FFT at that noise level instead;
//  3. weights[k] = sqrt(n) nrm[k] and directions f_k / nrm[k], or 0 and a zero column at or below
//     the floor ("zero column where the weight vanishes").
__global__ void fourier_colnorm_kernel(double2* __restrict__ F, int m, int n, double inv_sqrt_n,
                                       double* __restrict__ nrm) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  double s = 0.0;
  for (int i = 0; i < m; ++i) {
    double2 v = F[(size_t)i * n + k];
    v.x *= inv_sqrt_n;
    v.y *= inv_sqrt_n;
    F[(size_t)i * n + k] = v;
    s = fma(v.x, v.x, fma(v.y, v.y, s));
  }
  nrm[k] = sqrt(s);
}

__global__ void fourier_floor_kernel(const double* __restrict__ nrm, int n, double* __restrict__ floor_out) {
  __shared__ double sh[32];
  double s = 0.0;
  for (int k = threadIdx.x; k < n; k += blockDim.x) s = fma(nrm[k], nrm[k], s);
  s = block_sum(s, sh);
  if (threadIdx.x == 0)
    *floor_out = 4.0 * 2.220446049250313e-16 * log2(fmax(2.0, (double)n)) * sqrt((double)n * s);
}

__global__ void fourier_scale_kernel(double2* __restrict__ F, int m, int n, double sqrt_n,
                                     const double* __restrict__ nrm, const double* __restrict__ floor_in,
                                     double* __restrict__ weights) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  const double c = nrm[k];
  const bool keep = sqrt_n * c > *floor_in;
  weights[k] = keep ? sqrt_n * c : 0.0;
  for (int i = 0; i < m; ++i) {
    const double2 v = F[(size_t)i * n + k];
    F[(size_t)i * n + k] = keep ? make_double2(v.x / c, v.y / c) : make_double2(0.0, 0.0);
  }
}

static unsigned grid_for(size_t cnt) { return (unsigned)std::min<int64_t>(ceil_div(cnt, 256), kNumSMs * 8); }

}  // namespace apx

using namespace apx;

extern "C" size_t apx_unitary_dft_workspace(int64_t n, int64_t batch);
extern "C" int apx_unitary_dft(const void* x, void* y, int64_t n, int64_t batch, int64_t stride, int64_t dist,
                               int inverse, void* wsp, size_t ws_bytes, void* stream);

namespace apx {
struct SfftPlan {
  double2 *At, *Bt, *SA, *SB, *dAt, *va, *vb;
  double *mag, *part, *re1, *im1, *re2, *im2, *mre, *mim;
  int *sa, *sb;
  char* dft_ws;
  size_t dft_bytes;
  double* gpart;
  size_t gcap;
};

static void plan_sfft(Workspace& ws, SfftPlan& p, int m, int n, int q, int k) {
  const size_t mn = (size_t)m * n, nq = (size_t)n * q, mq = (size_t)m * q;
  p.At = ws.take<double2>(mn);
  p.Bt = ws.take<double2>(nq);
  p.SA = ws.take<double2>(mn);
  p.SB = ws.take<double2>(nq);
  p.dAt = ws.take<double2>(mn);
  p.va = ws.take<double2>((size_t)m * std::max(k, 1));
  p.vb = ws.take<double2>((size_t)std::max(n, q) * std::max(k, 1));
  p.mag = ws.take<double>(std::max(mn, nq));
  p.part = ws.take<double>(kNumSMs * 8);
  p.re1 = ws.take<double>(mn);
  p.im1 = ws.take<double>(mn);
  p.re2 = ws.take<double>(nq);
  p.im2 = ws.take<double>(nq);
  p.mre = ws.take<double>(mq);
  p.mim = ws.take<double>(mq);
  p.sa = ws.take<int>((size_t)m * std::max(k, 1));
  p.sb = ws.take<int>((size_t)std::max(n, q) * std::max(k, 1));
  p.dft_bytes = apx_unitary_dft_workspace(std::max(n, 1), std::max(m, q));
  p.dft_ws = ws.take<char>(p.dft_bytes);
  p.gcap = 8 * std::max(mq, (size_t)1);
  p.gpart = ws.take<double>(p.gcap);
}

// M (+)= (Ar + i Ai)(Br + i Bi) with 4 real DMMA GEMMs into the planes, then merged
static int complex_gemm(const SfftPlan& p, const double* ar, const double* ai, const double* br, const double* bi,
                        double2* M, int m, int n, int q, cudaStream_t st) {
  auto g = [&](const double* A, const double* B, double* C, int acc) {
    int s = gemm_splits(m, q, n, 64, 64);
    if (acc || (size_t)s * m * q > p.gcap) s = 1;
    return gemm_skinny<double>(0, A, n, B, q, C, q, m, q, n, acc, nullptr, 0, 1, p.gpart, s, false, st);
  };
  APX_TRY(g(ar, br, p.mre, 0));
  APX_TRY(g(ai, bi, p.mim, 0));
  const size_t cnt = (size_t)m * q;
  APX_TRY(launch_axpy2d(p.mre, q, p.mim, q, m, q, -1.0, nullptr, 0, st));  // re = ar br - ai bi
  APX_TRY(g(ar, bi, p.mim, 0));
  APX_TRY(g(ai, br, p.mim, 1));
  merge_planes_kernel<<<grid_for(cnt), 256, 0, st>>>(p.mre, p.mim, cnt, M);
  APX_LAUNCH_CHECK();
  return OK;
}
}  // namespace apx

extern "C" {

size_t apx_sfft_first_order_workspace(int64_t m, int64_t n, int64_t p, int k) {
  Workspace ws(nullptr, 0, true);
  SfftPlan pl;
  plan_sfft(ws, pl, (int)m, (int)n, (int)p, k);
  return ws.off;
}

// fft_sparse_first_order_multiply (fsparse.py:168-240): A m x n, B n x p (fp64 or complex128),
// k entries kept per row of At (and per row / column of Bt), M m x p complex128.
// scalars: FRO2_A, FRO2_B, RES2_A = ||At - SA||^2, RES2_B = ||Bt - SB||^2, FRO2_M.
int apx_sfft_first_order(int dtype, const void* A, const void* B, int64_t m, int64_t n, int64_t p, int k, int order,
                         int sparsify_cols, void* M_, int32_t* sel_a, int32_t* sel_b, double* scal, void* wsp,
                         size_t ws_bytes, void* stream) {
  APX_NVTX("apx_sfft_first_order");
  APX_REQUIRE(dtype == F64 || dtype == C128, "sfft product: fp64 or complex128 inputs");
  APX_REQUIRE(m >= 1 && n >= 1 && p >= 1, "empty operand");
  APX_REQUIRE(k >= 0, "k=%d must be >= 0", k);
  APX_REQUIRE(order == 0 || order == 1, "order must be 0 or 1");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  Workspace ws(wsp, ws_bytes);
  SfftPlan pl;
  const int mi = (int)m, ni = (int)n, pi = (int)p;
  const int ka = std::min(k, ni);
  const int kb = std::min(k, sparsify_cols ? ni : pi);
  plan_sfft(ws, pl, mi, ni, pi, std::max(ka, kb));
  APX_WS_CHECK(ws);
  double2* M = (double2*)M_;
  const size_t mn = (size_t)m * n, nq = (size_t)n * p, mq = (size_t)m * p;
  APX_CUDA(cudaMemsetAsync(scal, 0, APX_NSCALARS * sizeof(double), st));
  // complex copies of the operands (the DFT kernels read complex128)
  if (dtype == F64) {
    APX_CUDA(cudaMemsetAsync(pl.dAt, 0, mn * sizeof(double2), st));
    APX_CUDA(cudaMemcpy2DAsync(pl.dAt, sizeof(double2), A, sizeof(double), sizeof(double), mn,
                               cudaMemcpyDeviceToDevice, st));
    APX_CUDA(cudaMemsetAsync(pl.SB, 0, nq * sizeof(double2), st));
    APX_CUDA(cudaMemcpy2DAsync(pl.SB, sizeof(double2), B, sizeof(double), sizeof(double), nq,
                               cudaMemcpyDeviceToDevice, st));
  } else {
    APX_CUDA(cudaMemcpyAsync(pl.dAt, A, mn * sizeof(double2), cudaMemcpyDeviceToDevice, st));
    APX_CUDA(cudaMemcpyAsync(pl.SB, B, nq * sizeof(double2), cudaMemcpyDeviceToDevice, st));
  }
  int parts = 0;
  APX_TRY(launch_sumsq<double>((const double*)pl.dAt, 2 * mn, pl.part, &parts, st));
  APX_TRY(launch_sum_vector(pl.part, parts, scal + APX_S_FRO2_A, st));
  APX_TRY(launch_sumsq<double>((const double*)pl.SB, 2 * nq, pl.part, &parts, st));
  APX_TRY(launch_sum_vector(pl.part, parts, scal + APX_S_FRO2_B, st));
  // At = A W* (rows, inverse), Bt = W B (columns, forward)
  APX_TRY(apx_unitary_dft(pl.dAt, pl.At, n, m, 1, n, 1, pl.dft_ws, pl.dft_bytes, stream));
  APX_TRY(apx_unitary_dft(pl.SB, pl.Bt, n, p, p, 1, 0, pl.dft_ws, pl.dft_bytes, stream));
  // SA: per-row top-k of |At|
  cabs_kernel<<<grid_for(mn), 256, 0, st>>>(pl.At, mn, pl.mag);
  APX_LAUNCH_CHECK();
  APX_CUDA(cudaMemsetAsync(pl.SA, 0, mn * sizeof(double2), st));
  if (ka > 0) {
    topk_rows_kernel<<<mi, kSelThreads, 0, st>>>(pl.mag, ni, ka, nullptr, pl.sa);
    APX_LAUNCH_CHECK();
    scatter_kept_kernel<<<grid_for((size_t)m * ka), 256, 0, st>>>(pl.At, mi, ni, pl.sa, ka, 0, pl.SA, pl.va);
    APX_LAUNCH_CHECK();
  }
  // SB: per-row (or per-column) top-k of |Bt|
  APX_CUDA(cudaMemsetAsync(pl.SB, 0, nq * sizeof(double2), st));
  if (kb > 0) {
    if (!sparsify_cols) {
      cabs_kernel<<<grid_for(nq), 256, 0, st>>>(pl.Bt, nq, pl.mag);
      APX_LAUNCH_CHECK();
      topk_rows_kernel<<<ni, kSelThreads, 0, st>>>(pl.mag, pi, kb, nullptr, pl.sb);
      APX_LAUNCH_CHECK();
      scatter_kept_kernel<<<grid_for((size_t)n * kb), 256, 0, st>>>(pl.Bt, ni, pi, pl.sb, kb, 0, pl.SB, pl.vb);
    } else {
      // magnitudes of the columns of Bt as rows of |Bt|^T, then per-column selection of rows
      cabs_kernel<<<grid_for(nq), 256, 0, st>>>(pl.Bt, nq, pl.mag);
      APX_LAUNCH_CHECK();
      APX_TRY(launch_transpose_f64(pl.mag, pi, ni, pi, pl.re2, ni, st));
      topk_rows_kernel<<<pi, kSelThreads, 0, st>>>(pl.re2, ni, kb, nullptr, pl.sb);
      APX_LAUNCH_CHECK();
      scatter_kept_kernel<<<grid_for((size_t)p * kb), 256, 0, st>>>(pl.Bt, ni, pi, pl.sb, kb, 1, pl.SB, nullptr);
    }
    APX_LAUNCH_CHECK();
  }
  // residual norms (exact): ||At - SA||^2, ||Bt - SB||^2; dAt kept for order 1
  residual_kernel<<<kNumSMs * 4, 256, 0, st>>>(pl.At, pl.SA, mn, pl.dAt, pl.part);
  APX_LAUNCH_CHECK();
  APX_TRY(launch_sum_vector(pl.part, kNumSMs * 4, scal + APX_S_RES2_A, st));
  residual_kernel<<<kNumSMs * 4, 256, 0, st>>>(pl.Bt, pl.SB, nq, nullptr, pl.part);
  APX_LAUNCH_CHECK();
  APX_TRY(launch_sum_vector(pl.part, kNumSMs * 4, scal + APX_S_RES2_B, st));
  if (order == 0) {
    // M = SA . dense(SB)
    sparse_rows_gemm_kernel<<<mi, 256, 0, st>>>(pl.sa, pl.va, ka, pl.SB, pi, 0, M);
    APX_LAUNCH_CHECK();
  } else {
    // M = SA . Bt (sparse rows) + dAt . SB (dense complex GEMM)
    sparse_rows_gemm_kernel<<<mi, 256, 0, st>>>(pl.sa, pl.va, ka, pl.Bt, pi, 0, M);
    APX_LAUNCH_CHECK();
    split_planes_kernel<<<grid_for(mn), 256, 0, st>>>(pl.dAt, mn, pl.re1, pl.im1);
    APX_LAUNCH_CHECK();
    split_planes_kernel<<<grid_for(nq), 256, 0, st>>>(pl.SB, nq, pl.re2, pl.im2);
    APX_LAUNCH_CHECK();
    APX_TRY(complex_gemm(pl, pl.re1, pl.im1, pl.re2, pl.im2, M, mi, ni, pi, st));
  }
  APX_TRY(launch_sumsq<double>((const double*)M, 2 * mq, pl.part, &parts, st));
  APX_TRY(launch_sum_vector(pl.part, parts, scal + APX_S_FRO2_M, st));
  if (sel_a && ka > 0) APX_CUDA(cudaMemcpyAsync(sel_a, pl.sa, (size_t)m * ka * sizeof(int), cudaMemcpyDeviceToDevice, st));
  if (sel_b && kb > 0)
    APX_CUDA(cudaMemcpyAsync(sel_b, pl.sb, (size_t)(sparsify_cols ? p : n) * kb * sizeof(int),
                             cudaMemcpyDeviceToDevice, st));
  return OK;
}

// sparse_dense_multiply (fsparse.py:142-165), left side: out (rows x p, complex128) =
// S . X with S given as rows x k (sel, vals), -1 marking unused slots; X is ? x p complex128.
int apx_sparse_rows_multiply(const int32_t* sel, const void* vals, int k, int64_t rows, const void* X, int64_t p,
                             void* out, void* stream) {
  APX_REQUIRE(rows >= 1 && p >= 1 && k >= 0, "bad sparse multiply arguments");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  sparse_rows_gemm_kernel<<<(unsigned)rows, 256, 0, st>>>(sel, (const double2*)vals, k, (const double2*)X, (int)p, 0,
                                                          (double2*)out);
  APX_LAUNCH_CHECK();
  return OK;
}

size_t apx_fourier_row_decompose_workspace(int64_t m, int64_t n) {
  Workspace ws(nullptr, 0, true);
  ws.take<double2>((size_t)m * n);
  ws.take<char>(apx_unitary_dft_workspace(n, m));
  return ws.off;
}

// fourier_row_decompose (fsparse.py:92-105): A m x n (fp64 or complex128) -> weights (n fp64),
// directions (m x n complex128).
int apx_fourier_row_decompose(int dtype, const void* A, int64_t m, int64_t n, double* weights, void* directions,
                              void* wsp, size_t ws_bytes, void* stream) {
  APX_NVTX("apx_fourier_row_decompose");
  APX_REQUIRE(dtype == F64 || dtype == C128, "fourier_row_decompose: fp64 or complex128 input");
  APX_REQUIRE(m >= 1 && n >= 1, "empty matrix");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  Workspace ws(wsp, ws_bytes);
  double2* X = ws.take<double2>((size_t)m * n);
  const size_t dft_bytes = apx_unitary_dft_workspace(n, m);
  char* dft_ws = ws.take<char>(dft_bytes);
  APX_WS_CHECK(ws);
  const size_t mn = (size_t)m * n;
  if (dtype == F64) {
    APX_CUDA(cudaMemsetAsync(X, 0, mn * sizeof(double2), st));
    APX_CUDA(cudaMemcpy2DAsync(X, sizeof(double2), A, sizeof(double), sizeof(double), mn, cudaMemcpyDeviceToDevice,
                               st));
  } else {
    APX_CUDA(cudaMemcpyAsync(X, A, mn * sizeof(double2), cudaMemcpyDeviceToDevice, st));
  }
  APX_TRY(apx_unitary_dft(X, directions, n, m, 1, n, 0, dft_ws, dft_bytes, stream));
  double* nrm = (double*)X;  // X is consumed by the DFT; reuse it for the norms and the floor
  const unsigned g = (unsigned)ceil_div(n, 128);
  fourier_colnorm_kernel<<<g, 128, 0, st>>>((double2*)directions, (int)m, (int)n, 1.0 / sqrt((double)n), nrm);
  APX_LAUNCH_CHECK();
  fourier_floor_kernel<<<1, 1024, 0, st>>>(nrm, (int)n, nrm + n);
  APX_LAUNCH_CHECK();
  fourier_scale_kernel<<<g, 128, 0, st>>>((double2*)directions, (int)m, (int)n, sqrt((double)n), nrm, nrm + n,
                                          weights);
  APX_LAUNCH_CHECK();
  return OK;
}

size_t apx_topk_rows_workspace(int64_t rows, int64_t cols) {
  Workspace ws(nullptr, 0, true);
  ws.take<double>((size_t)rows * cols);
  return ws.off;
}

int apx_topk_rows(const void* M, int64_t rows, int64_t cols, int k, const int32_t* budget, int32_t* sel, void* vals,
                  void* wsp, size_t ws_bytes, void* stream) {
  APX_NVTX("apx_topk_rows");
  APX_REQUIRE(rows >= 1 && cols >= 1 && k >= 1, "bad topk_rows arguments");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  Workspace ws(wsp, ws_bytes);
  double* mag = ws.take<double>((size_t)rows * cols);
  APX_WS_CHECK(ws);
  const size_t cnt = (size_t)rows * cols;
  cabs_kernel<<<grid_for(cnt), 256, 0, st>>>((const double2*)M, cnt, mag);
  APX_LAUNCH_CHECK();
  topk_rows_kernel<<<(unsigned)rows, kSelThreads, 0, st>>>(mag, (int)cols, k, budget, sel);
  APX_LAUNCH_CHECK();
  scatter_kept_kernel<<<grid_for((size_t)rows * k), 256, 0, st>>>((const double2*)M, (int)rows, (int)cols, sel, k, 0,
                                                                 nullptr, (double2*)vals);
  APX_LAUNCH_CHECK();
  return OK;
}

}  // extern "C"
