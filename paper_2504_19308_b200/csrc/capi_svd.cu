// C-ABI for the randomized-SVD path (reference svd.py): randomized_partial_svd (svd.py:83-119)
// and svd_first_order_multiply (svd.py:138-200), fp64, on device.
//
//   range finder   Y = A Omega, Q = orth(Y); q x { Q = orth(A^T Q), Q = orth(A Q) }   (svd.py:105-111)
//   projection     Ba = Q^T A                                                         (svd.py:112)
//   small SVD      Ba^T = Q2 R2 (thin QR), Hestenes Jacobi on W = R2^T = Ba Q2 (l x l)  (svd.py:113)
//                  => U = Q U', V = Q2 V', sigma                                        (svd.py:114-116)
// The product only needs the projector Q Q^T when l == k, so
// svd_first_order_multiply skips the small SVD unless the sketch is oversampled (config C1):
//   order 0  M = Qa (Ba Qb) Bb                                   (= Ahat Bhat, svd.py:170-172)
//   order 1  M = Qa (Ba B) + (A Qb - Qa (Ba Qb)) Bb              (= Ahat B + dA Bhat, :174-177)
// All contractions are DMMA (mma.sync m8n8k4 f64) GEMMs; Omega is drawn by the host with numpy.
#include "../../include/apx.h"
#include "common.cuh"
#include "kernels.cuh"

namespace apx {

namespace {

struct Dgemm {
  double* part;
  size_t cap;  // doubles
  int operator()(const double* A, int64_t lda, const double* B, int64_t ldb, double* C, int64_t ldc, int M, int N,
                 int K, int acc, cudaStream_t st) const {
    int s = gemm_splits(M, N, K, 64, 64);
    if (acc || ldc != N || (size_t)s * M * N > cap) s = 1;
    return gemm_skinny<double>(0, A, lda, B, ldb, C, ldc, M, N, K, acc, nullptr, 0, 1, part, s, false, st);
  }
};

// Per-operand buffers of the rSVD (sized for an m x n operand, sketch width l).
struct Side {
  double *Y, *Q, *Qt, *P, *Pt, *Ba, *Q2, *Q2t, *W, *Up, *S, *Vp, *VpT, *Qk, *Bk, *svd_scratch;
  void* qr;
  size_t qr_bytes;
};

void plan_side(Workspace& ws, Side& s, int m, int n, int l) {
  const size_t mx = (size_t)std::max(m, n);
  s.Y = ws.take<double>(mx * l);
  s.Q = ws.take<double>(mx * l);
  s.Qt = ws.take<double>(mx * l);
  s.P = ws.take<double>(mx * l);
  s.Pt = ws.take<double>(mx * l);
  s.Ba = ws.take<double>((size_t)l * n);
  s.Q2 = ws.take<double>((size_t)n * l);
  s.Q2t = ws.take<double>((size_t)n * l);
  s.W = ws.take<double>((size_t)l * l);
  s.Up = ws.take<double>((size_t)l * l);
  s.S = ws.take<double>((size_t)l + 1);
  s.Vp = ws.take<double>((size_t)l * l);
  s.VpT = ws.take<double>((size_t)l * l);
  s.Qk = ws.take<double>((size_t)m * l);
  s.Bk = ws.take<double>((size_t)l * n);
  s.svd_scratch = ws.take<double>(small_svd_scratch_doubles(l) + 1);
  s.qr_bytes = qr_ws_bytes((int)mx, l);
  s.qr = ws.take<char>(s.qr_bytes);
}

// Q (m x l) orthonormal basis of range(A Omega) after q power iterations; Qt = Q^T.
int range_finder(const double* A, int m, int n, int l, int q, const double* Om, const Side& s, const Dgemm& g,
                 cudaStream_t st) {
  // the QRs inside the power iteration only carry the subspace to the next product (method 2: one
  // CholeskyQR pass when the sketch is well conditioned); the last one is the full QR
  APX_TRY(g(A, n, Om, l, s.Y, l, m, l, n, 0, st));
  APX_TRY((qr_orthonormalize<double, double>(s.Y, l, 1, m, l, s.Q, l, 1, s.Qt, 1, m, s.qr, s.qr_bytes, q > 0 ? 2 : 0,
                                             st)));
  for (int it = 0; it < q; ++it) {
    APX_TRY(g(s.Qt, m, A, n, s.Pt, n, l, n, m, 0, st));  // Pt = Q^T A  (= (A^T Q)^T)
    APX_TRY((qr_orthonormalize<double, double>(s.Pt, 1, n, n, l, s.P, l, 1, (double*)nullptr, 0, 0, s.qr, s.qr_bytes,
                                               2, st)));
    APX_TRY(g(A, n, s.P, l, s.Y, l, m, l, n, 0, st));
    APX_TRY((qr_orthonormalize<double, double>(s.Y, l, 1, m, l, s.Q, l, 1, s.Qt, 1, m, s.qr, s.qr_bytes,
                                               it + 1 < q ? 2 : 0, st)));
  }
  return OK;
}

// Ba = Q^T A, then the small SVD of Ba: U' (l x l), S, V', V'^T and Q2 (n x l), Q2t.
int project_and_svd(const double* A, int m, int n, int l, const Side& s, const Dgemm& g, bool need_svd,
                    cudaStream_t st) {
  APX_TRY(g(s.Qt, m, A, n, s.Ba, n, l, n, m, 0, st));
  if (!need_svd) return OK;
  APX_TRY((qr_orthonormalize<double, double>(s.Ba, 1, n, n, l, s.Q2, l, 1, s.Q2t, 1, n, s.qr, s.qr_bytes, 0, st)));
  APX_TRY(g(s.Ba, n, s.Q2, l, s.W, l, l, l, n, 0, st));  // W = Ba Q2 = R2^T
  APX_TRY(launch_small_svd(s.W, l, s.Up, s.S, s.Vp, s.VpT, st, s.svd_scratch));
  return OK;
}

size_t svd_first_order_ws(int m, int n, int p, int la, int lb) {
  Workspace ws(nullptr, 0, true);
  Side a, b;
  plan_side(ws, a, m, n, la);
  plan_side(ws, b, n, p, lb);
  const int mx = std::max(m, std::max(n, p)), lm = std::max(la, lb);
  ws.take<double>((size_t)lm * p * 3 + (size_t)lm * lm * 2 + (size_t)m * lm * 2);
  ws.take<double>((size_t)16 * mx * lm);  // split-K scratch
  ws.take<double>(4 * kNumSMs + 64);
  ws.take<double>((size_t)16 * mx * lm);  // split-K scratch of B's decomposition (side stream)
  return ws.off;
}

template <typename T>
__global__ void transpose_kernel(const T* __restrict__ in, int64_t ldi, int rows, int cols, T* __restrict__ out,
                                 int64_t ldo) {
  __shared__ T tile[32][33];
  const int bx = blockIdx.x * 32, by = blockIdx.y * 32;
  for (int y = threadIdx.y; y < 32; y += blockDim.y) {
    const int r = by + y, c = bx + threadIdx.x;
    tile[y][threadIdx.x] = (r < rows && c < cols) ? in[(size_t)r * ldi + c] : T{};
  }
  __syncthreads();
  for (int y = threadIdx.y; y < 32; y += blockDim.y) {
    const int r = bx + y, c = by + threadIdx.x;  // out is cols x rows
    if (r < cols && c < rows) out[(size_t)r * ldo + c] = tile[threadIdx.x][y];
  }
}

template <typename T>
int launch_transpose(const T* in, int64_t ldi, int rows, int cols, T* out, int64_t ldo, cudaStream_t st) {
  dim3 grid((unsigned)ceil_div(cols, 32), (unsigned)ceil_div(rows, 32));
  transpose_kernel<T><<<grid, dim3(32, 8), 0, st>>>(in, ldi, rows, cols, out, ldo);
  APX_LAUNCH_CHECK();
  return OK;
}

__global__ void triu_kernel(double* R, int k) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < k * k; e += gridDim.x * blockDim.x)
    if (e / k > e % k) R[e] = 0.0;
}

}  // namespace

int launch_transpose_f64(const double* in, int64_t ldi, int rows, int cols, double* out, int64_t ldo, cudaStream_t st) {
  return launch_transpose<double>(in, ldi, rows, cols, out, ldo, st);
}
int launch_transpose_f32(const float* in, int64_t ldi, int rows, int cols, float* out, int64_t ldo, cudaStream_t st) {
  return launch_transpose<float>(in, ldi, rows, cols, out, ldo, st);
}
int launch_transpose_c128(const double2* in, int64_t ldi, int rows, int cols, double2* out, int64_t ldo,
                          cudaStream_t st) {
  return launch_transpose<double2>(in, ldi, rows, cols, out, ldo, st);
}

}  // namespace apx

using namespace apx;

extern "C" {

size_t apx_rsvd_workspace(int dtype, int64_t m, int64_t n, int l) {
  (void)dtype;
  Workspace ws(nullptr, 0, true);
  Side s;
  plan_side(ws, s, (int)m, (int)n, l);
  ws.take<double>((size_t)16 * std::max(m, n) * l);
  ws.take<double>(4 * kNumSMs + 64);
  return ws.off;
}

int apx_rsvd(int dtype, const void* A_, int64_t m, int64_t n, int l, int k, int power_iterations, const void* omega,
             void* U_, double* sigma, void* V_, double* scalars, void* wsp, size_t ws_bytes, void* stream) {
  APX_NVTX("apx_rsvd");
  APX_REQUIRE(dtype == F64, "randomized_partial_svd: fp64 required");
  APX_REQUIRE(m >= 1 && n >= 1, "empty matrix");
  APX_REQUIRE(l >= 1 && l <= m && l <= n, "sketch width %d out of range", l);
  APX_REQUIRE(k >= 1 && k <= l, "kept rank %d out of range [1, %d]", k, l);
  APX_REQUIRE(power_iterations >= 0, "power_iterations must be >= 0");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const double* A = (const double*)A_;
  Workspace ws(wsp, ws_bytes);
  Side s;
  plan_side(ws, s, (int)m, (int)n, l);
  Dgemm g{ws.take<double>((size_t)16 * std::max(m, n) * l), (size_t)16 * std::max(m, n) * l};
  double* red = ws.take<double>(4 * kNumSMs + 64);
  APX_WS_CHECK(ws);
  APX_CUDA(cudaMemsetAsync(scalars, 0, APX_NSCALARS * sizeof(double), st));
  APX_TRY(range_finder(A, (int)m, (int)n, l, power_iterations, (const double*)omega, s, g, st));
  APX_TRY(project_and_svd(A, (int)m, (int)n, l, s, g, true, st));
  // U = Q U'[:, :k], V = Q2 V'[:, :k], sigma = S[:k]
  APX_TRY(g(s.Q, l, s.Up, l, (double*)U_, k, (int)m, k, l, 0, st));
  APX_TRY(g(s.Q2, l, s.Vp, l, (double*)V_, k, (int)n, k, l, 0, st));
  APX_CUDA(cudaMemcpyAsync(sigma, s.S, (size_t)k * sizeof(double), cudaMemcpyDeviceToDevice, st));
  int parts = 0;
  APX_TRY(launch_sumsq<double>(A, (size_t)m * n, red, &parts, st));
  APX_TRY(launch_sum_vector(red, parts, scalars + APX_S_FRO2_A, st));
  APX_TRY(launch_sumsq_prefix(s.S, k, scalars + APX_S_KEPT_A, st));
  return OK;
}

size_t apx_qr_workspace(int dtype, int64_t m, int64_t k) {
  (void)dtype;
  Workspace ws(nullptr, 0, true);
  ws.take<char>(qr_ws_bytes((int)m, (int)k));
  ws.take<double>((size_t)m * k);
  ws.take<double>((size_t)16 * m * k);
  return ws.off;
}

int apx_qr(int dtype, const void* Y_, int64_t m, int64_t k, void* Q_, void* R_, void* wsp, size_t ws_bytes,
           void* stream) {
  APX_NVTX("apx_qr");
  APX_REQUIRE(dtype == F64, "qr_decompose: fp64 required");
  APX_REQUIRE(m >= k, "need at least as many rows as columns, got %lld x %lld", (long long)m, (long long)k);
  APX_REQUIRE(k >= 1, "qr_decompose: at least one column");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  Workspace ws(wsp, ws_bytes);
  const size_t qb = qr_ws_bytes((int)m, (int)k);
  void* qws = ws.take<char>(qb);
  double* Qt = ws.take<double>((size_t)m * k);
  Dgemm g{ws.take<double>((size_t)16 * m * k), (size_t)16 * m * k};
  APX_WS_CHECK(ws);
  const double* Y = (const double*)Y_;
  // Householder with LAPACK's reflector convention (geqrf/orgqr signs), R = triu(Q^T Y)
  APX_TRY((qr_orthonormalize<double, double>(Y, k, 1, (int)m, (int)k, (double*)Q_, k, 1, Qt, 1, m, qws, qb, 1, st)));
  APX_TRY(g(Qt, m, Y, k, (double*)R_, k, (int)k, (int)k, (int)m, 0, st));
  triu_kernel<<<1, 256, 0, st>>>((double*)R_, (int)k);
  APX_LAUNCH_CHECK();
  return OK;
}

// ||A (B G)||_F^2 (errest.py:139-154 before its division by k): X = B G (n x k), T = A X
// (m x k), both fp64 DMMA GEMMs, then a fixed-order sum of squares. O(k n^2) instead of O(n^3).
size_t apx_sketch_norm_workspace(int64_t m, int64_t n, int64_t p, int k) {
  Workspace ws(nullptr, 0, true);
  ws.take<double>((size_t)n * k);
  ws.take<double>((size_t)m * k);
  ws.take<double>((size_t)8 * std::max(m, n) * k);
  ws.take<double>(4096);
  return ws.off;
}

int apx_sketch_norm(const double* A, const double* B, int64_t m, int64_t n, int64_t p, const double* G, int k,
                    double* out, void* wsp, size_t ws_bytes, void* stream) {
  APX_NVTX("apx_sketch_norm");
  APX_REQUIRE(m >= 1 && n >= 1 && p >= 1, "sketch_norm: empty operand");
  APX_REQUIRE(k >= 1, "k must be >= 1");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  Workspace ws(wsp, ws_bytes);
  double* X = ws.take<double>((size_t)n * k);
  double* T = ws.take<double>((size_t)m * k);
  double* part = ws.take<double>((size_t)8 * std::max(m, n) * k);
  double* red = ws.take<double>(4096);
  APX_WS_CHECK(ws);
  Dgemm g{part, (size_t)8 * std::max(m, n) * k};
  APX_TRY(g(B, p, G, k, X, k, (int)n, k, (int)p, 0, st));
  APX_TRY(g(A, n, X, k, T, k, (int)m, k, (int)n, 0, st));
  int parts = 0;
  APX_TRY(launch_sumsq<double>(T, (size_t)m * k, red, &parts, st));
  APX_REQUIRE(parts <= 4096, "sketch_norm: reduction workspace");
  return launch_sum_vector(red, parts, out, st);
}

size_t apx_gemm_workspace(int dtype, int64_t M, int64_t N, int64_t K, int trans_a, int trans_b) {
  const size_t e = dtype == F32 ? 4 : 8;
  Workspace ws(nullptr, 0, true);
  if (trans_a) ws.take<char>((size_t)M * K * e);
  if (trans_b) ws.take<char>((size_t)K * N * e);
  ws.take<char>((size_t)8 * M * N * e);
  return ws.off;
}

// C (+)= op(A) op(B): op(A) is M x K (A stored K x M when trans_a), op(B) is K x N (B stored N x K
// when trans_b). fp64: DMMA; fp32: TF32 mma.sync with 3xTF32 splitting (fp32-level accuracy).
int apx_gemm(int dtype, int trans_a, int trans_b, int64_t M, int64_t N, int64_t K, const void* A, int64_t lda,
             const void* B, int64_t ldb, void* C, int64_t ldc, int accumulate, void* wsp, size_t ws_bytes,
             void* stream) {
  APX_NVTX("apx_gemm");
  APX_REQUIRE(dtype == F32 || dtype == F64, "gemm: real dtype required");
  APX_REQUIRE(M >= 1 && N >= 1 && K >= 1, "gemm: empty operand");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  Workspace ws(wsp, ws_bytes);
  const size_t e = dtype == F32 ? 4 : 8;
  char* At = trans_a ? ws.take<char>((size_t)M * K * e) : nullptr;
  char* Bt = trans_b ? ws.take<char>((size_t)K * N * e) : nullptr;
  char* part = ws.take<char>((size_t)8 * M * N * e);
  APX_WS_CHECK(ws);
  if (dtype == F64) {
    const double* a = (const double*)A;
    const double* b = (const double*)B;
    int64_t la = lda, lb = ldb;
    if (trans_a) { APX_TRY(launch_transpose<double>(a, lda, (int)K, (int)M, (double*)At, K, st)); a = (double*)At; la = K; }
    if (trans_b) { APX_TRY(launch_transpose<double>(b, ldb, (int)N, (int)K, (double*)Bt, N, st)); b = (double*)Bt; lb = N; }
    Dgemm g{(double*)part, (size_t)8 * M * N};
    return g(a, la, b, lb, (double*)C, ldc, (int)M, (int)N, (int)K, accumulate, st);
  }
  const float* a = (const float*)A;
  const float* b = (const float*)B;
  int64_t la = lda, lb = ldb;
  if (trans_a) { APX_TRY(launch_transpose<float>(a, lda, (int)K, (int)M, (float*)At, K, st)); a = (float*)At; la = K; }
  if (trans_b) { APX_TRY(launch_transpose<float>(b, ldb, (int)N, (int)K, (float*)Bt, N, st)); b = (float*)Bt; lb = N; }
  int s = gemm_splits((int)M, (int)N, (int)K, 128, 128);
  if (accumulate || ldc != N || s > 8) s = 1;
  return gemm_skinny<float>(2, a, la, b, lb, (float*)C, ldc, (int)M, (int)N, (int)K, accumulate, nullptr, 0, 1,
                            (float*)part, s, true, st);
}

size_t apx_svd_first_order_workspace(int dtype, int64_t m, int64_t n, int64_t p, int l_a, int l_b) {
  (void)dtype;
  return svd_first_order_ws((int)m, (int)n, (int)p, l_a, l_b);
}

int apx_svd_first_order(int dtype, const void* A_, const void* B_, int64_t m, int64_t n, int64_t p, int l_a, int k_a,
                        int l_b, int k_b, int power_iterations, int order, const void* omega_a,
                        const void* omega_b, void* M_, double* scalars, void* wsp, size_t ws_bytes, void* stream) {
  APX_NVTX("apx_svd_first_order");
  APX_REQUIRE(dtype == F64, "svd_first_order_multiply: fp64 required");
  APX_REQUIRE(m >= 1 && n >= 1 && p >= 1, "empty matrix");
  APX_REQUIRE(l_a >= 1 && l_a <= m && l_a <= n && k_a >= 1 && k_a <= l_a, "A sketch out of range");
  APX_REQUIRE(l_b >= 1 && l_b <= n && l_b <= p && k_b >= 1 && k_b <= l_b, "B sketch out of range");
  APX_REQUIRE(order == 0 || order == 1, "order must be 0 or 1");
  APX_REQUIRE(power_iterations >= 0, "power_iterations must be >= 0");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const double* A = (const double*)A_;
  const double* B = (const double*)B_;
  double* M = (double*)M_;
  const int mi = (int)m, ni = (int)n, pi = (int)p;
  Workspace ws(wsp, ws_bytes);
  Side a, b;
  plan_side(ws, a, mi, ni, l_a);
  plan_side(ws, b, ni, pi, l_b);
  const int lm = std::max(l_a, l_b), mx = std::max(mi, std::max(ni, pi));
  double* T = ws.take<double>((size_t)lm * pi * 3 + (size_t)lm * lm * 2 + (size_t)mi * lm * 2);
  double* T2 = T + (size_t)lm * lm;
  double* S1 = T2 + (size_t)lm * pi;
  double* P = S1 + (size_t)lm * pi;
  double* P2 = P + (size_t)mi * lm;
  Dgemm g{ws.take<double>((size_t)16 * mx * lm), (size_t)16 * mx * lm};
  double* red = ws.take<double>(4 * kNumSMs + 64);
  Dgemm g2{ws.take<double>((size_t)16 * mx * lm), (size_t)16 * mx * lm};
  APX_WS_CHECK(ws);
  APX_CUDA(cudaMemsetAsync(scalars, 0, APX_NSCALARS * sizeof(double), st));
  stage_mark(0, st);
  // operand decompositions (independent sketches: default_rng([seed,0]) / ([seed,1]), svd.py:161-162):
  // two latency-bound chains of small kernels (~5 QRs each), so B's runs on the side stream
  // concurrently with A's (each with its own buffers and split-K scratch)
  cudaStream_t sb = st;
  APX_TRY(side_fork(st, &sb));
  APX_TRY(range_finder(A, mi, ni, l_a, power_iterations, (const double*)omega_a, a, g, st));
  APX_TRY(project_and_svd(A, mi, ni, l_a, a, g, k_a < l_a, st));
  APX_TRY(range_finder(B, ni, pi, l_b, power_iterations, (const double*)omega_b, b, g2, sb));
  APX_TRY(project_and_svd(B, ni, pi, l_b, b, g2, k_b < l_b, sb));
  APX_TRY(side_join(st, sb));
  stage_mark(1, st);
  // truncation of an oversampled sketch: Qk = Q U'[:, :k], Bk = diag(S_k) V'^T[:k] Q2^T
  const double *Qa = a.Q, *Ba = a.Ba, *Qb = b.Q, *Bb = b.Ba;
  if (k_a < l_a) {
    APX_TRY(g(a.Q, l_a, a.Up, l_a, a.Qk, k_a, mi, k_a, l_a, 0, st));
    APX_TRY(g(a.VpT, l_a, a.Q2t, ni, a.Bk, ni, k_a, ni, l_a, 0, st));
    APX_TRY(launch_axpy2d(a.Bk, ni, a.Bk, ni, k_a, ni, 1.0, a.S, 1, st));
    APX_TRY(launch_sumsq_prefix(a.S, k_a, scalars + APX_S_KEPT_A, st));
    Qa = a.Qk;
    Ba = a.Bk;
  } else {
    int parts = 0;
    APX_TRY(launch_sumsq<double>(a.Ba, (size_t)l_a * ni, red, &parts, st));
    APX_TRY(launch_sum_vector(red, parts, scalars + APX_S_KEPT_A, st));
  }
  if (k_b < l_b) {
    APX_TRY(g(b.Q, l_b, b.Up, l_b, b.Qk, k_b, ni, k_b, l_b, 0, st));
    APX_TRY(g(b.VpT, l_b, b.Q2t, pi, b.Bk, pi, k_b, pi, l_b, 0, st));
    APX_TRY(launch_axpy2d(b.Bk, pi, b.Bk, pi, k_b, pi, 1.0, b.S, 1, st));
    APX_TRY(launch_sumsq_prefix(b.S, k_b, scalars + APX_S_KEPT_B, st));
    Qb = b.Qk;
    Bb = b.Bk;
  } else {
    int parts = 0;
    APX_TRY(launch_sumsq<double>(b.Ba, (size_t)l_b * pi, red, &parts, st));
    APX_TRY(launch_sum_vector(red, parts, scalars + APX_S_KEPT_B, st));
  }
  const int ka = k_a, kb = k_b;
  const int64_t lqa = k_a < l_a ? k_a : l_a, lqb = k_b < l_b ? k_b : l_b;  // leading dims of Qa / Qb
  APX_TRY(g(Ba, ni, Qb, lqb, T, kb, ka, kb, ni, 0, st));  // T = Ba Qb  (ka x kb)
  if (order == 0) {
    APX_TRY(g(T, kb, Bb, pi, T2, pi, ka, pi, kb, 0, st));  // T2 = T Bb
    APX_TRY(g(Qa, lqa, T2, pi, M, pi, mi, pi, ka, 0, st));  // M = Qa T2
  } else {
    APX_TRY(g(Ba, ni, B, pi, S1, pi, ka, pi, ni, 0, st));   // S1 = Ba B
    APX_TRY(g(Qa, lqa, S1, pi, M, pi, mi, pi, ka, 0, st));  // M = Qa S1  (Ahat B)
    APX_TRY(g(A, ni, Qb, lqb, P, kb, mi, kb, ni, 0, st));   // P = A Qb
    APX_TRY(g(Qa, lqa, T, kb, P2, kb, mi, kb, ka, 0, st));  // P2 = Qa (Ba Qb)
    APX_TRY(launch_axpy2d(P, kb, P2, kb, mi, kb, -1.0, nullptr, 0, st));  // P = dA Qb
    APX_TRY(g(P, kb, Bb, pi, M, pi, mi, pi, kb, 1, st));    // M += (dA Qb) Bb
  }
  stage_mark(2, st);
  int parts = 0;
  APX_TRY(launch_sumsq<double>(A, (size_t)m * n, red, &parts, st));
  APX_TRY(launch_sum_vector(red, parts, scalars + APX_S_FRO2_A, st));
  APX_TRY(launch_sumsq<double>(B, (size_t)n * p, red, &parts, st));
  APX_TRY(launch_sum_vector(red, parts, scalars + APX_S_FRO2_B, st));
  APX_TRY(launch_sumsq<double>(M, (size_t)m * p, red, &parts, st));
  APX_TRY(launch_sum_vector(red, parts, scalars + APX_S_FRO2_M, st));
  stage_mark(3, st);
  return OK;
}

}  // extern "C"
