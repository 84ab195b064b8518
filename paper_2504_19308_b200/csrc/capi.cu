// C-ABI entry points (include/apx.h). Validation, workspace planning, and the launch sequence
// of each product; the kernels live in the other translation units.
#include <atomic>
#include <cstdarg>

#include "../../include/apx.h"
#include "common.cuh"
#include "kernels.cuh"

namespace apx {

static thread_local char g_err[1024] = "";
static std::atomic<long long> g_launches{0};
static thread_local cudaEvent_t* g_stage_ev = nullptr;
static thread_local int g_stage_n = 0;

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

void stage_mark(int i, cudaStream_t st) {
  if (g_stage_ev != nullptr && i < g_stage_n && g_stage_ev[i] != nullptr) cudaEventRecord(g_stage_ev[i], st);
}

static inline cudaStream_t S(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// gather lambda tables are padded to a multiple of 8 rows (zeros) for the unguarded fast path
static inline int pad8(int k) { return (int)ceil_div(std::max(k, 1), 8) * 8; }

template <typename T>
static int zero_pad_rows(T* lam, int k, int n, cudaStream_t st) {
  const int kp = pad8(k);
  if (kp > k) APX_CUDA(cudaMemsetAsync(lam + (size_t)k * n, 0, (size_t)(kp - k) * n * sizeof(T), st));
  return OK;
}

// ------------------------------------------------------------------------------------------
// cycle product plan
// ------------------------------------------------------------------------------------------
struct CyclePlan {
  double* partial;   // energy partials (shared by A then B)
  double* en_a;      // energies A
  double* nr_a;      // norms A
  double* en_b;
  double* nr_b;
  void* lam_a;       // k_a x n
  void* lam_b;       // k_b x n
  void* bhat;        // n x n (order 0 only)
  void* xt;          // n x n: X^T for the transposed left product (large n only)
  void* tt;          // n x n: (A_hat . X)^T
  int* jneg;         // (n - J_A) mod n
  bool left_t;       // A_hat . X evaluated as (X^T A_hat^T)^T with the right gather
  double* msq;       // ||M||^2 partials
  int n_msq;
  unsigned short* lam_h;  // f16 lambda' table of the f16-staged residual gather (fp32, large n)
};

static void plan_cycle(Workspace& ws, CyclePlan& p, int dtype, int n, int ka, int kb, int order) {
  const size_t e = dtype == F32 ? 4 : 8;
  p.partial = ws.take<double>(cycle_energy_ws(n) / sizeof(double) + 1);
  p.en_a = ws.take<double>(n);
  p.nr_a = ws.take<double>(n);
  p.en_b = ws.take<double>(n);
  p.nr_b = ws.take<double>(n);
  p.lam_a = ws.take<char>((size_t)pad8(ka) * n * e);
  p.lam_b = ws.take<char>((size_t)pad8(kb) * n * e);
  p.bhat = order == 0 ? (void*)ws.take<char>((size_t)n * n * e) : nullptr;
  p.left_t = left_via_transpose(n, e, ka);
  p.xt = p.left_t ? (void*)ws.take<char>((size_t)n * n * e) : nullptr;
  p.tt = p.left_t ? (void*)ws.take<char>((size_t)n * n * e) : nullptr;
  p.jneg = ws.take<int>((size_t)pad8(ka));
  p.n_msq = std::max<int>((int)ceil_div(n, 1), kNumSMs * 4);
  p.msq = ws.take<double>(p.n_msq);
  p.lam_h = (dtype == F32 && order == 1 && ka > 0 && right_gather_seg_rows(n, 4, kb) > 0)
                ? (unsigned short*)ws.take<char>(right_gather_seg_f16_ws(n, kb))
                : nullptr;
}

template <typename T>
static int run_cycle(const T* A, const T* B, int n, int ka, int kb, int order, const int* fa, const int* fb, T* M,
                     int* sa, int* sb, double* scal, const CyclePlan& p, cudaStream_t st) {
  stage_mark(0, st);
  APX_CUDA(cudaMemsetAsync(scal, 0, APX_NSCALARS * sizeof(double), st));
  APX_TRY(launch_cycle_energies<T>(A, n, p.en_a, p.nr_a, scal + APX_S_FRO2_A, p.partial, st));
  APX_TRY(launch_cycle_energies<T>(B, n, p.en_b, p.nr_b, scal + APX_S_FRO2_B, p.partial, st));
  if (fa) { if (ka) APX_CUDA(cudaMemcpyAsync(sa, fa, ka * sizeof(int), cudaMemcpyDeviceToDevice, st)); }
  else APX_TRY(launch_topk(p.nr_a, n, ka, sa, st));
  if (fb) { if (kb) APX_CUDA(cudaMemcpyAsync(sb, fb, kb * sizeof(int), cudaMemcpyDeviceToDevice, st)); }
  else APX_TRY(launch_topk(p.nr_b, n, kb, sb, st));
  APX_TRY(launch_kept_energy(p.nr_a, sa, ka, 1.0, scal + APX_S_KEPT_A, st));
  APX_TRY(launch_kept_energy(p.nr_b, sb, kb, 1.0, scal + APX_S_KEPT_B, st));
  T* la = (T*)p.lam_a;
  T* lb = (T*)p.lam_b;
  APX_TRY(launch_cycle_extract<T>(A, n, sa, ka, la, st));
  APX_TRY(zero_pad_rows<T>(la, ka, n, st));
  APX_TRY(launch_cycle_extract<T>(B, n, sb, kb, lb, st, /*aligned=*/order == 1));  // order 0: materialize
  APX_TRY(zero_pad_rows<T>(lb, kb, n, st));
  stage_mark(1, st);
  // Ahat . X: column strips of X in shared memory (left gather), or for large n -- where a strip
  // is one or two columns and every lambda would be re-read per column -- as (X^T Ahat^T)^T:
  // Ahat^T has shifts n - J_t and, aligned to its output index, the left-layout table itself, so
  // the row-block right gather runs on X^T (R rows resident, each lambda feeding R FMAs)
  auto left_product = [&](const T* X, T* out) -> int {
    if (!p.left_t) return launch_cycle_left_gather<T>(X, la, sa, ka, n, 0, out, st);
    T *xt = (T*)p.xt, *tt = (T*)p.tt;
    APX_TRY(launch_transpose_any(X, n, n, n, xt, n, st));
    APX_TRY(launch_negate_shifts(sa, ka, n, p.jneg, st));
    APX_TRY(launch_cycle_right_gather<T>(xt, nullptr, 0, la, p.jneg, ka, n, n, 0, tt, nullptr, nullptr, st, true));
    return launch_transpose_any(tt, n, n, n, out, n, st);
  };
  if (order == 1) {
    // M = Ahat . B
    APX_TRY(left_product(B, M));
    stage_mark(2, st);
    // M += dA . Bhat (right gather over row blocks of A, masked to dA on load) + ||M||^2
    // (large fp32 n: staged as scaled f16 when dA is a small residual -- cycle.cu K11h)
    if (p.lam_h != nullptr && right_gather_seg_f16_ok(n, sizeof(T), kb))
      APX_TRY(launch_cycle_right_gather_seg_f16((const float*)A, sa, ka, (const float*)lb, sb, kb, n, n, 1, (float*)M,
                                                p.msq, st, 0, p.lam_h, scal + APX_S_FRO2_A, scal + APX_S_KEPT_A,
                                                scal + APX_S_FRO2_B));
    else
      APX_TRY(launch_cycle_right_gather<T>(A, sa, ka, lb, sb, kb, n, n, 1, M, p.msq, nullptr, st, true));
    stage_mark(3, st);
    const int rblocks = (int)ceil_div(n, right_gather_rows_plain(n, sizeof(T), kb));
    APX_TRY(launch_sum_vector(p.msq, rblocks, scal + APX_S_FRO2_M, st));
  } else {
    T* bh = (T*)p.bhat;
    APX_TRY(launch_cycle_materialize<T>(lb, sb, kb, n, bh, st));
    APX_TRY(left_product(bh, M));
    int parts = 0;
    APX_TRY(launch_sumsq<T>(M, (size_t)n * n, p.msq, &parts, st));
    APX_TRY(launch_sum_vector(p.msq, parts, scal + APX_S_FRO2_M, st));
  }
  stage_mark(4, st);
  return OK;
}

// ------------------------------------------------------------------------------------------
// row-sharded cycle product (C2 / C5 rows over ranks): rank g holds the row
// block A_rows = A[r0:r0+m] and the whole B, and produces M[r0:r0+m]. A's cycle energies are
// row-separable, so the only exchange before the product is the sum of the rank's energy
// partials (n fp64); the selection is then made from identical sums on every rank, B's selection
// from the (replicated) B. After the product, ||M_g||^2 is summed.
// ------------------------------------------------------------------------------------------
struct CycleRowsPlan {
  double *partial, *nr_a, *en_b, *nr_b, *msq;
  void *lam_a, *lam_b, *bhat, *xt, *tt;
  int *jneg;
  bool left_t;
  unsigned short* lam_h;
};

static void plan_cycle_rows(Workspace& ws, CycleRowsPlan& p, int dtype, int n, int m, int ka, int kb, int order) {
  const size_t e = dtype == F32 ? 4 : 8;
  p.partial = ws.take<double>(cycle_energy_ws(n) / sizeof(double) + 1);
  p.nr_a = ws.take<double>(n);
  p.en_b = ws.take<double>(n);
  p.nr_b = ws.take<double>(n);
  p.msq = ws.take<double>(std::max<int>(m, kNumSMs * 4));
  p.lam_a = ws.take<char>((size_t)std::max(ka, 1) * m * e);
  p.lam_b = ws.take<char>((size_t)pad8(kb) * n * e);
  p.bhat = order == 0 ? (void*)ws.take<char>((size_t)n * n * e) : nullptr;
  p.left_t = left_via_transpose(n, e, ka);
  p.xt = p.left_t ? (void*)ws.take<char>((size_t)n * n * e) : nullptr;
  p.tt = p.left_t ? (void*)ws.take<char>((size_t)n * m * e) : nullptr;
  p.jneg = ws.take<int>((size_t)pad8(ka));
  p.lam_h = (dtype == F32 && order == 1 && ka > 0 && right_gather_seg_rows(n, 4, kb) > 0)
                ? (unsigned short*)ws.take<char>(right_gather_seg_f16_ws(n, kb))
                : nullptr;
}

__global__ void sqrt_vector_kernel(const double* __restrict__ e, int n, double* __restrict__ out) {
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) out[j] = sqrt(e[j]);
}

template <typename T>
static int run_cycle_rows(int phase, const T* A, int m, int r0, const T* B, int n, int ka, int kb, int order, T* M,
                          int* sa, int* sb, const double* red_in, double* red_out, double* scal,
                          const CycleRowsPlan& p, cudaStream_t st) {
  if (phase == 1) return launch_cycle_energies_rows<T>(A, m, r0, n, red_out, p.partial, st);
  // phase 2: red_in = A's energies summed over the ranks
  APX_CUDA(cudaMemsetAsync(scal, 0, APX_NSCALARS * sizeof(double), st));
  sqrt_vector_kernel<<<(unsigned)std::min<int64_t>(ceil_div(n, 256), 1024), 256, 0, st>>>(red_in, n, p.nr_a);
  APX_LAUNCH_CHECK();
  APX_TRY(launch_topk(p.nr_a, n, ka, sa, st, p.nr_a, 1.0, scal + APX_S_KEPT_A, red_in, scal + APX_S_FRO2_A));
  APX_TRY(launch_cycle_energies<T>(B, n, p.en_b, p.nr_b, nullptr, p.partial, st));
  APX_TRY(launch_topk(p.nr_b, n, kb, sb, st, p.nr_b, 1.0, scal + APX_S_KEPT_B, p.en_b, scal + APX_S_FRO2_B));
  T* la = (T*)p.lam_a;
  T* lb = (T*)p.lam_b;
  APX_TRY(launch_cycle_extract_rows<T>(A, m, r0, n, sa, ka, la, st));
  APX_TRY(launch_cycle_extract<T>(B, n, sb, kb, lb, st, /*aligned=*/order == 1));
  APX_TRY(zero_pad_rows<T>(lb, kb, n, st));
  const T* X = B;
  if (order == 0) {
    APX_TRY(launch_cycle_materialize<T>(lb, sb, kb, n, (T*)p.bhat, st));
    X = (const T*)p.bhat;
  }
  // term1 rows: Ahat[r0:r0+m] . X
  if (ka == 0) {
    APX_CUDA(cudaMemsetAsync(M, 0, (size_t)m * n * sizeof(T), st));
  } else if (!p.left_t) {
    APX_TRY(launch_cycle_left_gather_rows<T>(X, la, sa, ka, n, r0, r0 + m, M, st));
  } else {
    // (X^T Ahat^T)^T restricted to the output columns r0..r0+m of X^T Ahat^T
    T *xt = (T*)p.xt, *tt = (T*)p.tt;
    APX_TRY(launch_transpose_any(X, n, n, n, xt, n, st));
    APX_TRY(launch_negate_shifts(sa, ka, n, p.jneg, st));
    APX_TRY(launch_cycle_right_gather_cols<T>(xt, la, p.jneg, ka, n, n, r0, r0 + m, tt, st));
    APX_TRY(launch_transpose_any(tt, m, n, m, M, n, st));
  }
  if (order == 1) {
    // M_rows += dA_rows . Bhat (A's kept cycles masked on load, global row r0 + r) + ||M_g||^2
    if (p.lam_h != nullptr && right_gather_seg_f16_ok(n, sizeof(T), kb))
      APX_TRY(launch_cycle_right_gather_seg_f16((const float*)A, sa, ka, (const float*)lb, sb, kb, n, m, 1, (float*)M,
                                                p.msq, st, r0, p.lam_h, scal + APX_S_FRO2_A, scal + APX_S_KEPT_A,
                                                scal + APX_S_FRO2_B));
    else
      APX_TRY(launch_cycle_right_gather<T>(A, sa, ka, lb, sb, kb, n, m, 1, M, p.msq, nullptr, st, true, 0, nullptr, 1,
                                           false, nullptr, false, r0));
    const int rblocks = (int)ceil_div(m, right_gather_rows_plain(n, sizeof(T), kb));
    APX_TRY(launch_sum_vector(p.msq, rblocks, red_out, st));
  } else {
    int parts = 0;
    APX_TRY(launch_sumsq<T>(M, (size_t)m * n, p.msq, &parts, st));
    APX_TRY(launch_sum_vector(p.msq, parts, red_out, st));
  }
  return OK;
}

// ------------------------------------------------------------------------------------------
// mixed product plan: A by rSVD (l = k_svd columns, q power iterations), B by k_cyc cycles.
//   order 1:  M = Q (Bm . dB) + A . Bhat      (== Ahat.B + dA.Bhat, Ahat = Q Q^T A = Q Bm)
//   order 0:  M = Q (Bm . Bhat)               (== Ahat . Bhat)
// Only the projector Q Q^T enters M when l = k, so no small SVD is needed;
// sum sigma^2 = ||Bm||_F^2 gives the residual norm (svd.py:122-130).
// ------------------------------------------------------------------------------------------
struct MixedPlan {
  double* partial;
  double* en_b;
  double* nr_b;
  void* lam_b;
  void *Y, *Q, *Qt, *Z, *Bm, *W, *part;
  void* qr_ws;
  size_t qr_bytes;
  double* msq;
  double* asq;
  double* bsq;
  int* ticket;
  int* ready;  // per gather row block: 1 once its M rows are final (consumed by M += Q.W on lo)
  int n_part_rows;
  // residual plan (mixed_f16.cu): [Q | Q], the TF32 hi/lo split of W, f16 lambda', f16 dA
  // (row-block interleaved); null when the shape does not fit it
  float *Q2 = nullptr, *W2 = nullptr;
  uint16_t *lamh = nullptr, *dAh = nullptr;
};

// The residual plan's shape conditions (run_mixed_f32_resid): fp32, l = 64, a row fits shared
// memory as 8 f16 rows, n a multiple of the gather's 4 x 128-column thread groups.
static bool resid_shape_ok(int dtype, int n, int l, int kc) {
  return dtype == F32 && l == 64 && kc >= 1 && kc <= 128 && gather_f16_threads(n) > 0 &&
         gather_f16_smem(n, pad8(kc)) <= 220 * 1024;
}

static int mixed_gemm_splits(int n, int l) {
  return std::max(gemm_splits(n, l, n, 128, 64), gemm_splits(l, n, n, 64, 128));
}

// row groups of the residual plan's energy pass (APX_EN_GROUPS, tuning knob; 0 = one wave of
// long-lived CTAs, the default). Short-lived CTAs (128-512 groups, several waves) let the QR's
// single-CTA Cholesky find an SM sooner (it ends 20 us earlier) but the QR's remaining kernels then
// overlap the pass's HBM traffic and finish no earlier (measured 1118-1142 vs 1128 products/s).
// CTAs of B's energy pass in the residual plan (row-stream kernel): the SMs the fused QR leaves
// (qr_sm_footprint), so neither waits for the other's CTAs to drain
static int resid_energy_ctas(int n) {
  return std::max(16, device_sms() - qr_sm_footprint(n, 64));
}

static int resid_energy_groups(int n) {
  static const int env = [] {
    const char* e = getenv("APX_EN_GROUPS");
    return e ? atoi(e) : 0;
  }();
  return std::min(std::max(env, 0), n);
}

static void plan_mixed(Workspace& ws, MixedPlan& p, int dtype, int n, int l, int kc) {
  const size_t e = dtype == F32 ? 4 : 8;
  p.partial = ws.take<double>(std::max(cycle_energy_ws(n), cycle_energy_ws_groups(n, resid_energy_groups(n))) /
                                  sizeof(double) + 1);
  p.en_b = ws.take<double>(n);
  p.nr_b = ws.take<double>(n);
  p.lam_b = ws.take<char>((size_t)pad8(kc) * n * e);
  const size_t nl = (size_t)n * l * e;
  p.Y = ws.take<char>(nl);
  p.Q = ws.take<char>(nl);
  p.Qt = ws.take<char>(nl);
  p.Z = ws.take<char>(nl);
  p.Bm = ws.take<char>(nl);
  p.W = ws.take<char>(nl);
  p.part = ws.take<char>(nl * (size_t)std::max(8, mixed_gemm_splits(n, l)));
  p.qr_bytes = qr_ws_bytes(n, l);
  p.qr_ws = ws.take<char>(p.qr_bytes);
  p.n_part_rows = (int)ceil_div(n, 1);
  const int64_t qw_ctas = ceil_div(n, 128) * ceil_div(n, 128);  // ||M||^2 partials of the Q.W GEMM
  p.msq = ws.take<double>((size_t)std::max<int64_t>(std::max<int64_t>(n, kNumSMs * 4), qw_ctas));
  p.asq = ws.take<double>(std::max<int>(n, kNumSMs * 4));
  p.bsq = ws.take<double>(std::max<int>(n, kNumSMs * 4));
  p.ticket = ws.take<int>(8);  // [0] gather ticket, [1] persistent Q.W ticket, [2] finalize counter, [3] use_f16
  p.ready = ws.take<int>((size_t)n + 1 + qw_ctas);  // row-block flags, then the deferred-tile list
  if (resid_shape_ok(dtype, n, l, kc)) {
    p.Q2 = ws.take<float>((size_t)n * 2 * l);
    p.W2 = ws.take<float>((size_t)n * 2 * l);
    p.lamh = ws.take<uint16_t>((size_t)pad8(kc) * n);
    p.dAh = ws.take<uint16_t>((size_t)ceil_div(n, 8) * 8 * n);
  }
}

// fp32 GEMM stages of the mixed product on tcgen05 (umma.cu). Layout bits: 1 = A operand stored
// [k][m] (MN-major), 2 = B operand stored [k][n] (MN-major), 4 = transposed store.
struct UmmaStages {
  // K splits for a skinny GEMM with ceil(n/128) row tiles on an SM budget (two CTAs per SM)
  static int splits(int n, int sms = kNumSMs) {
    return std::max(1, std::min(8, (int)((2 * sms) / ceil_div(n, 128))));
  }
  static int umma_gemm(int layout, int bn, const float* A, int64_t lda, const float* B, int64_t ldb, float* C,
                       int64_t ldc, int64_t css, int M, int N, int K, int splits, int acc, const int* mJ, int mk,
                       int mod_n, cudaStream_t st) {
    return umma_tma_gemm(layout, bn, A, lda, B, ldb, C, ldc, css, M, N, K, splits, acc, mJ, mk, mod_n, st);
  }
  // Y[n x l] = A . X, X stored n x l (row-major)
  static int a_times_x(const float* A, const float* X, float* Y, float* part, int n, int l, cudaStream_t st,
                       int sms = kNumSMs) {
    const int s = splits(n, sms);
    APX_TRY(umma_gemm(2, 64, A, n, X, l, s > 1 ? part : Y, l, (int64_t)n * l, n, l, n, s, 0, nullptr, 0, 1, st));
    if (s > 1) APX_TRY(launch_split_reduce_f32(part, s, (size_t)n * l, Y, st));
    return OK;
  }
  // Z[n x l] = A^T . X   (= (X^T A)^T), X stored n x l
  static int at_times_x(const float* A, const float* X, float* Z, float* part, int n, int l, cudaStream_t st,
                        int sms = kNumSMs) {
    const int s = splits(n, sms);
    APX_TRY(umma_gemm(3, 64, A, n, X, l, s > 1 ? part : Z, l, (int64_t)n * l, n, l, n, s, 0, nullptr, 0, 1, st));
    if (s > 1) APX_TRY(launch_split_reduce_f32(part, s, (size_t)n * l, Z, st));
    return OK;
  }
  // Bm[l x n] = Q^T . A, computed as (A^T Q) stored transposed; Q stored n x l
  static int qt_times_a(const float* A, const float* Q, float* Bm, float* part, int n, int l, cudaStream_t st,
                        int sms = kNumSMs) {
    const int s = splits(n, sms);
    // layout bit 8: operands rounded to TF32 nearest in shared memory, so ||Bm||^2 = sum sigma^2
    // (the residual energy ||A||^2 - ||Bm||^2, svd.py:122-130) carries no truncation bias
    APX_TRY(umma_gemm(7 | 8, 64, A, n, Q, l, s > 1 ? part : Bm, n, (int64_t)l * n, n, l, n, s, 0, nullptr, 0, 1, st));
    if (s > 1) APX_TRY(launch_split_reduce_f32(part, s, (size_t)n * l, Bm, st));
    return OK;
  }
  // W[l x n] = Bm . dB, computed as (dB^T Bm^T) stored transposed; dB = B with kept cycles masked
  static int bm_times_db(const float* B, const float* Bm, float* W, float* part, int n, int l, const int* J, int kc,
                         cudaStream_t st, int sms = kNumSMs) {
    const int s = splits(n, sms);
    APX_TRY(umma_gemm(5, 64, B, n, Bm, n, s > 1 ? part : W, n, (int64_t)l * n, n, l, n, s, 0, J, kc, n, st));
    if (s > 1) APX_TRY(launch_split_reduce_f32(part, s, (size_t)n * l, W, st));
    return OK;
  }
  // M[n x n] (+)= Q . W  (Q stored n x l, W stored l x n); optional ||M||^2 partials per CTA
  static int q_times_w(const float* Q, const float* W, float* M, int n, int l, cudaStream_t st, int acc = 0,
                       double* sq = nullptr, const int* ready = nullptr, int ready_rows = 0,
                       const int* progress = nullptr, int* defer = nullptr) {
    // accumulate: BN 128 / 2 stages, whose drained ring holds the C tile for the staged epilogue
    // (measured faster than a persistent double-buffered variant: 3 CTAs per SM = 12 epilogue warps)
    return umma_tma_gemm(2, acc ? 128 : 256, Q, l, W, n, M, n, 0, n, n, l, 1, acc, nullptr, 0, 1, st, sq, ready,
                         ready_rows, progress, defer);
  }
  static int q_times_w_ctas(int n, int l, int acc) {
    return (int)(ceil_div(n, acc ? 128 : 256) * ceil_div(n, 128));
  }
};

// Per-thread side stream + fork/join events: B's cycle decomposition (HBM-bound energy pass,
// latency-bound select) runs concurrently with A's range finder (GEMMs + the latency-bound QR).
// Two internal streams per host thread: `hi` (greatest priority) carries the cycle side of the
// product (B's decomposition, then the persistent row gather), `lo` (least priority) the
// range finder. The gather's persistent CTAs leave a few SMs free; the range finder's
// HBM-bound GEMMs and latency-bound QR run there concurrently, so they cost almost no gather
// time. Priorities make freed SMs go to pending gather CTAs first.
struct SideStream {
  cudaStream_t s = nullptr, hi = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr, b_ready = nullptr, hi_done = nullptr, b_read = nullptr;
  cudaEvent_t aux_fork = nullptr, aux_join = nullptr;  // side_fork / side_join (other products)
  cudaEvent_t en_done = nullptr;                        // residual plan: B's energy pass done (hi)
};
// Keyed by the current device: one host thread may drive several GPUs (or re-target with
// cudaSetDevice), and each device gets its own pair of streams and events.
constexpr int kMaxDevices = 64;
static thread_local SideStream g_side[kMaxDevices];

static int get_side(SideStream** out) {
  int dev = 0;
  APX_CUDA(cudaGetDevice(&dev));
  APX_REQUIRE(dev >= 0 && dev < kMaxDevices, "device ordinal %d out of range", dev);
  SideStream& g = g_side[dev];
  if (!g.s) {
    int least = 0, greatest = 0;
    APX_CUDA(cudaDeviceGetStreamPriorityRange(&least, &greatest));
    APX_CUDA(cudaStreamCreateWithPriority(&g.s, cudaStreamNonBlocking, least));
    APX_CUDA(cudaStreamCreateWithPriority(&g.hi, cudaStreamNonBlocking, greatest));
    APX_CUDA(cudaEventCreateWithFlags(&g.fork, cudaEventDisableTiming));
    APX_CUDA(cudaEventCreateWithFlags(&g.join, cudaEventDisableTiming));
    APX_CUDA(cudaEventCreateWithFlags(&g.b_ready, cudaEventDisableTiming));
    APX_CUDA(cudaEventCreateWithFlags(&g.hi_done, cudaEventDisableTiming));
    APX_CUDA(cudaEventCreateWithFlags(&g.b_read, cudaEventDisableTiming));
    APX_CUDA(cudaEventCreateWithFlags(&g.aux_fork, cudaEventDisableTiming));
    APX_CUDA(cudaEventCreateWithFlags(&g.aux_join, cudaEventDisableTiming));
    APX_CUDA(cudaEventCreateWithFlags(&g.en_done, cudaEventDisableTiming));
  }
  *out = &g;
  return OK;
}

// Fork / join of the calling thread's low-priority side stream on the current device, for products
// whose two operand decompositions are independent (apx_svd_first_order): *side = st when `st` is
// being captured into a CUDA graph (batched products already run concurrently there, and a shared
// side stream would serialise the captured products).
int side_fork(cudaStream_t st, cudaStream_t* side) {
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  APX_CUDA(cudaStreamIsCapturing(st, &cap));
  if (cap != cudaStreamCaptureStatusNone) {
    *side = st;
    return OK;
  }
  SideStream* ss = nullptr;
  APX_TRY(get_side(&ss));
  APX_CUDA(cudaEventRecord(ss->aux_fork, st));
  APX_CUDA(cudaStreamWaitEvent(ss->s, ss->aux_fork, 0));
  *side = ss->s;
  return OK;
}
int side_join(cudaStream_t st, cudaStream_t side) {
  if (side == st) return OK;
  SideStream* ss = nullptr;
  APX_TRY(get_side(&ss));
  APX_CUDA(cudaEventRecord(ss->aux_join, side));
  APX_CUDA(cudaStreamWaitEvent(st, ss->aux_join, 0));
  return OK;
}

// Persistent gather grid: all but kMinFreeSMs SMs (the row blocks are pulled from a ticket, so
// the count need not divide them); APX_GATHER_CTAS overrides, for tuning.
static int gather_ctas(int nblk) {
  // measured at n = 8192 (bench sweep): 16 free SMs = 32 slots for the range finder's 64-CTA GEMMs
  // (exactly two waves); 14 free SMs need a third wave, 18 slow the gather
  constexpr int kMinFreeSMs = 16;
  static const int env = [] {
    const char* e = getenv("APX_GATHER_CTAS");
    return e ? atoi(e) : 0;
  }();
  if (env > 0) return env;
  return std::max(1, std::min(nblk, device_sms() - kMinFreeSMs));
}

// SM budget the Y = A Omega GEMM sizes its K split for (APX_Y_SMS, tuning knob). Default 64: two
// K slices (128 CTAs) -- Y starts before the gather holds its SMs (tools/c4_sweep.sh: 978 vs 963
// products/s for 32, the round-1 setting, and 967 for 148)
static int y_sm_budget() {
  static const int v = [] {
    const char* e = getenv("APX_Y_SMS");
    return e ? std::max(1, atoi(e)) : 64;
  }();
  return v;
}

// Stage markers (bench.py): 0 start | hi: 1 B decomposed, 2 gather done | lo: 3 Y, 4 QR, 5 Bm,
// 9 W GEMM, 6 W correction, 7 M += Q.W (order 1; on the main stream after the join for order 0)
// | main: 8 end.
static int run_mixed_f32_umma(const float* A, const float* B, int n, int l, int kc, int order, int q,
                              const float* Omega, const int* fb, float* M, int* sb, double* scal,
                              const MixedPlan& p, cudaStream_t st) {
  stage_mark(0, st);
  APX_CUDA(cudaMemsetAsync(scal, 0, APX_NSCALARS * sizeof(double), st));
  const int grows = right_gather_rows(n, sizeof(float), kc);
  const int rblocks = (int)ceil_div(n, grows);
  int* defer = p.ready + rblocks;  // [count, tiles...] of the bounded-wait Q.W epilogue
  if (order == 1) {
    APX_CUDA(cudaMemsetAsync(p.ready, 0, (rblocks + 1) * sizeof(int), st));
    APX_CUDA(cudaMemsetAsync(p.ticket, 0, sizeof(int), st));  // the gather's (x_early launch)
  }
  SideStream* ss = nullptr;
  APX_TRY(get_side(&ss));
  APX_CUDA(cudaEventRecord(ss->fork, st));
  APX_CUDA(cudaStreamWaitEvent(ss->s, ss->fork, 0));
  APX_CUDA(cudaStreamWaitEvent(ss->hi, ss->fork, 0));
  const cudaStream_t hi = ss->hi, lo = ss->s;
  const int gctas = gather_ctas(rblocks);
  const int free_sms = std::max(8, kNumSMs - gctas);
  // ---- hi: B's cycle decomposition -> (order 1) the gather M = A . Bhat --------------------------
  if (fb) {
    APX_TRY(launch_cycle_energies<float>(B, n, p.en_b, p.nr_b, scal + APX_S_FRO2_B, p.partial, hi));
    if (kc) APX_CUDA(cudaMemcpyAsync(sb, fb, kc * sizeof(int), cudaMemcpyDeviceToDevice, hi));
    APX_TRY(launch_kept_energy(p.nr_b, sb, kc, 1.0, scal + APX_S_KEPT_B, hi));
  } else {  // selection with ||B||^2 and the kept energy fused into the select kernel
    APX_TRY(launch_cycle_energies<float>(B, n, p.en_b, p.nr_b, nullptr, p.partial, hi));
    APX_CUDA(cudaEventRecord(ss->b_read, hi));
    APX_TRY(launch_topk(p.nr_b, n, kc, sb, hi, p.nr_b, 1.0, scal + APX_S_KEPT_B, p.en_b, scal + APX_S_FRO2_B));
  }
  if (fb) APX_CUDA(cudaEventRecord(ss->b_read, hi));
  float* lb = (float*)p.lam_b;
  APX_TRY(launch_cycle_extract<float>(B, n, sb, kc, lb, hi, /*aligned=*/true));
  APX_TRY(zero_pad_rows<float>(lb, kc, n, hi));
  APX_CUDA(cudaEventRecord(ss->b_ready, hi));
  stage_mark(1, hi);
  if (order == 1) {
    APX_TRY(launch_cycle_right_gather<float>(A, nullptr, 0, lb, sb, kc, n, n, 0, M, nullptr, p.asq, hi, true, gctas,
                                             p.ticket, 1, false, p.ready, /*x_early=*/true));
  }
  stage_mark(2, hi);
  if (order == 1) APX_TRY(launch_sum_vector(p.asq, rblocks, scal + APX_S_FRO2_A, hi));  // ||A||^2 (gather partials)
  APX_CUDA(cudaEventRecord(ss->hi_done, hi));
  // ---- lo: randomized range finder on the SMs the gather leaves free ------------------------------
  float *Y = (float*)p.Y, *Q = (float*)p.Q, *Qt = (float*)p.Qt, *Z = (float*)p.Z, *Bm = (float*)p.Bm,
        *W = (float*)p.W, *part = (float*)p.part;
  // Y starts when B's energy pass (the HBM-bound, critical part of B's decomposition) is done and
  // overlaps the latency-bound select/extract and the gather's start; the rest of the range
  // finder then fits on the SMs the persistent gather leaves free
  // (waiting for the extraction instead -- Y entirely after B's stage -- measured the same)
  APX_CUDA(cudaStreamWaitEvent(lo, ss->b_read, 0));
  APX_TRY(UmmaStages::a_times_x(A, Omega, Y, part, n, l, lo, y_sm_budget()));
  stage_mark(3, lo);
  APX_TRY((qr_orthonormalize<float, float>(Y, l, 1, n, l, Q, l, 1, Qt, 1, n, p.qr_ws, p.qr_bytes, 0, lo, /*tf32=*/1)));
  for (int it = 0; it < q; ++it) {
    APX_TRY(UmmaStages::at_times_x(A, Q, Z, part, n, l, lo, free_sms));
    APX_TRY((qr_orthonormalize<float, float>(Z, l, 1, n, l, Q, l, 1, Qt, 1, n, p.qr_ws, p.qr_bytes, 0, lo, /*tf32=*/1)));
    APX_TRY(UmmaStages::a_times_x(A, Q, Y, part, n, l, lo, free_sms));
    APX_TRY((qr_orthonormalize<float, float>(Y, l, 1, n, l, Q, l, 1, Qt, 1, n, p.qr_ws, p.qr_bytes, 0, lo, /*tf32=*/1)));
  }
  stage_mark(4, lo);
  APX_TRY(UmmaStages::qt_times_a(A, Q, Bm, part, n, l, lo, free_sms));
  int parts = 0;
  APX_TRY(launch_sumsq<float>(Bm, (size_t)l * n, p.bsq, &parts, lo));
  APX_TRY(launch_sum_vector(p.bsq, parts, scal + APX_S_KEPT_A, lo));
  stage_mark(5, lo);
  // W = Bm . dB = Bm . B - Bm . Bhat (order 1) or Bm . Bhat (order 0): an unmasked TF32 GEMM plus a
  // 64-row gather over column chunks (cheaper on a few SMs than masking every GEMM stage). The
  // subtracted gather uses the same TF32-truncated operands as the tensor core, so the large kept
  // part cancels exactly and W keeps TF32 accuracy relative to Bm . dB, not to Bm . B.
  // ~5 CTA waves over the free SMs: each of the l/R row blocks split into column chunks
  const int wblocks = (int)ceil_div(l, right_gather_rows(n, sizeof(float), kc));
  const int wchunks = std::max(1, std::min(8, (int)ceil_div(5 * free_sms, wblocks)));
  if (order == 1) APX_TRY(UmmaStages::bm_times_db(B, Bm, W, part, n, l, nullptr, 0, lo, free_sms));
  stage_mark(9, lo);
  APX_CUDA(cudaStreamWaitEvent(lo, ss->b_ready, 0));  // B's selection and lambda' (long done by now)
  APX_TRY(launch_cycle_right_gather<float>(Bm, nullptr, 0, lb, sb, kc, n, l, order == 1 ? -1 : 0, W, nullptr, nullptr,
                                           lo, true, 0, nullptr, wchunks, /*tf32_operands=*/order == 1));
  stage_mark(6, lo);
  // M += Q . W (order 1) with ||M||^2 fused into the epilogue, on lo while the gather is still
  // running: each tile's operand pipeline and MMA run at once, and its epilogue waits (acquire)
  // only for the gather row blocks under it, so the HBM-bound read-modify-write of the finished
  // rows overlaps the shared-memory-bound gather on the SMs it leaves free, and the rest follows
  // the gather's frontier onto the SMs it releases. The gather is enqueued on hi well before the
  // range finder ends, so its CTAs are normally resident first; CUDA does not guarantee that
  // across streams (MPS SM limits, co-tenants), so each tile's wait is bounded: a tile whose
  // gather makes no progress for 20 ms defers itself, and qw_fixup_sum_kernel completes it after
  // the gather (lo waits for hi first). Normally nothing is deferred and the fixup kernel is the
  // fixed-order ||M||^2 sum it replaces.
  if (order == 1) {
    APX_TRY(UmmaStages::q_times_w(Q, W, M, n, l, lo, 1, p.msq, p.ready, grows, p.ticket, defer));
    stage_mark(7, lo);
    APX_CUDA(cudaStreamWaitEvent(lo, ss->hi_done, 0));
    APX_TRY(launch_qw_fixup_sum(Q, l, W, n, M, n, n, n, l, 128, defer, p.msq, UmmaStages::q_times_w_ctas(n, l, 1),
                                scal + APX_S_FRO2_M, lo));
  }
  APX_CUDA(cudaEventRecord(ss->join, lo));
  // ---- main: join; (order 0) M = Q . W; the fixed-order sums ----------------------------------
  APX_CUDA(cudaStreamWaitEvent(st, ss->join, 0));
  APX_CUDA(cudaStreamWaitEvent(st, ss->hi_done, 0));
  if (order != 1) {
    APX_TRY(UmmaStages::q_times_w(Q, W, M, n, l, st, 0, p.msq));
    stage_mark(7, st);
    APX_TRY(launch_sum_vector(p.msq, UmmaStages::q_times_w_ctas(n, l, 0), scal + APX_S_FRO2_M, st));
    APX_TRY(launch_sumsq<float>(A, (size_t)n * n, p.asq, &parts, st));
    APX_TRY(launch_sum_vector(p.asq, parts, scal + APX_S_FRO2_A, st));
  }
  stage_mark(8, st);
  return OK;
}

// ---- residual plan of the C4 product (order 1; mixed_f16.cu explains the algebra) ----------------
// M = Q.(Bm.B) + (A - Q.Bm).Bhat: the gather runs over the f16 residual dA instead of the fp32 A,
// i.e. 2 shared-memory bytes per FMA instead of 4.
//   hi: Y = A Omega, CholeskyQR, Bm = Q^T A (+||A||^2 from the rounded A tiles), Bm := tf32(Bm),
//       dA = A - Q.Bm stored as f16 (fused epilogue), then the persistent f16 gather M = dA.Bhat
//       on all but 16 SMs, publishing a flag per 8-row block
//   lo: B's cycle decomposition and lambda' (fp32 and scaled f16) during the QR | on the 16 SMs
//       the gather leaves: W = Bm.B (TF32 GEMM minus the TF32-exact gather plus the fp32 gather),
//       hi/lo split, M += [Q|Q].[W_hi; W_lo] (+||M||^2) following the gather's row flags (bounded
//       wait + fixup as in run_mixed_f32_umma). (Measured alternative: M = Q.W first, then the
//       gather as a read-modify-write on every SM -- the W chain then sits on the critical path:
//       979 vs 1132 products/s.)
// Stage markers: 0 start | hi: 3 Y, 4 QR, 5 Bm, 10 dA, 11 gather start, 2 gather end |
// lo: 1 B decomposed, 9 W GEMM, 6 W, 7 M += Q.W | 8 end.
static int run_mixed_f32_resid(const float* A, const float* B, int n, int l, int kc, int q, const float* Omega,
                               const int* fb, float* M, int* sb, double* scal, const MixedPlan& p, cudaStream_t st) {
  stage_mark(0, st);
  const int grows = 8;  // the f16 gather's row block
  const int rblocks = (int)ceil_div(n, grows);
  int* defer = p.ready + rblocks;
  SideStream* ss = nullptr;
  APX_TRY(get_side(&ss));
  APX_CUDA(cudaEventRecord(ss->fork, st));
  APX_CUDA(cudaStreamWaitEvent(ss->s, ss->fork, 0));
  APX_CUDA(cudaStreamWaitEvent(ss->hi, ss->fork, 0));
  // the resets go to lo, off the critical path: the scalars, the gather's row flags and deferral
  // list, the tickets and the finalize counter; hi picks them up through `b_read` (before the Bm
  // finalize) and `b_ready` (before the gather)
  APX_CUDA(cudaMemsetAsync(scal, 0, APX_NSCALARS * sizeof(double), ss->s));
  APX_CUDA(cudaMemsetAsync(p.ready, 0, (rblocks + 1) * sizeof(int), ss->s));
  APX_CUDA(cudaMemsetAsync(p.ticket, 0, 8 * sizeof(int), ss->s));
  APX_CUDA(cudaEventRecord(ss->b_read, ss->s));
  // The critical path is A's chain (Y -> QR -> Bm -> dA -> gather), so it runs on the
  // high-priority stream; B's decomposition and the W chain fill in on the low-priority one.
  const cudaStream_t hi = ss->hi, lo = ss->s;
  const int gctas = gather_ctas(rblocks);
  const int free_sms = std::max(8, kNumSMs - gctas);
  const int kp = pad8(kc);
  float *Y = (float*)p.Y, *Q = (float*)p.Q, *Qt = (float*)p.Qt, *Z = (float*)p.Z, *Bm = (float*)p.Bm,
        *W = (float*)p.W, *part = (float*)p.part;
  // ---- hi: Y = A Omega on the whole GPU, then CholeskyQR -------------------------------------------
  // B's energy pass (HBM-bound) runs after Y = A Omega, overlapping the latency-bound QR, at the
  // full 8 CTAs per SM so it is over quickly (a long, thin energy pass slows the QR's loads: the
  // QR's span grew 117 -> 240 us as its CTAs per SM went 8 -> 1). Concurrent with Y instead
  // (APX_B_ORDER=0) delays Y by the shared bandwidth and measured the same (1122 vs 1121).
  static const int b_after_y = [] {
    const char* e = getenv("APX_B_ORDER");
    return e ? atoi(e) : 1;
  }();
  static const int en_cps = [] {  // energy-pass CTAs per SM (APX_EN_CPS, tuning knob)
    const char* e = getenv("APX_EN_CPS");
    return e ? std::max(1, std::min(8, atoi(e))) : 8;
  }();
  // APX_B_ORDER=3: B's energy pass runs first, alone on hi (both it and Y are HBM streams, so the
  // order costs nothing there), and the QR then runs without an energy pass beside it
  if (b_after_y == 3) {
    APX_CUDA(cudaStreamWaitEvent(hi, ss->b_read, 0));  // lo's resets
    APX_TRY(launch_cycle_energies<float>(B, n, p.en_b, p.nr_b, fb ? scal + APX_S_FRO2_B : nullptr, p.partial, hi,
                                         en_cps, resid_energy_groups(n)));
    APX_CUDA(cudaEventRecord(ss->en_done, hi));
  }
  stage_mark(17, hi);
  static const int y_sms = getenv("APX_Y_SMS") ? y_sm_budget() : kNumSMs;  // tuning knob
  APX_TRY(UmmaStages::a_times_x(A, Omega, Y, part, n, l, hi, y_sms));
  stage_mark(3, hi);
  APX_CUDA(cudaStreamWaitEvent(hi, ss->b_read, 0));  // lo's resets (long done)
  // APX_B_ORDER=2: B's decomposition waits for the QR instead (its energy pass, one wave of
  // long-lived CTAs on every SM, otherwise holds the QR's single-CTA Cholesky out of the SMs)
  if (b_after_y == 1) {
    APX_CUDA(cudaEventRecord(ss->b_read, hi));
    APX_CUDA(cudaStreamWaitEvent(lo, ss->b_read, 0));
  }
  // ---- lo: B's cycle decomposition and the f16 lambda' table -----------------------------------
  float* lb = (float*)p.lam_b;
  auto b_stage = [&]() -> int {
    if (b_after_y == 3) {
      APX_CUDA(cudaStreamWaitEvent(lo, ss->en_done, 0));  // the energy pass ran on hi
    } else {
      // on the SMs the QR (64 CTAs of two row tiles each at n = 8192) leaves: the two run side by side
      APX_TRY(launch_cycle_energies<float>(B, n, p.en_b, p.nr_b, fb ? scal + APX_S_FRO2_B : nullptr, p.partial, lo,
                                           en_cps, resid_energy_groups(n), resid_energy_ctas(n)));
    }
    if (fb) {
      APX_CUDA(cudaMemcpyAsync(sb, fb, kc * sizeof(int), cudaMemcpyDeviceToDevice, lo));
      APX_TRY(launch_kept_energy(p.nr_b, sb, kc, 1.0, scal + APX_S_KEPT_B, lo));
    } else {
      APX_TRY(launch_topk(p.nr_b, n, kc, sb, lo, p.nr_b, 1.0, scal + APX_S_KEPT_B, p.en_b, scal + APX_S_FRO2_B));
    }
    APX_TRY(launch_cycle_extract<float>(B, n, sb, kc, lb, lo, /*aligned=*/true));
    APX_TRY(zero_pad_rows<float>(lb, kc, n, lo));
    APX_TRY(launch_lam_f16(lb, kp, n, scal + APX_S_FRO2_B, p.lamh, lo));
    APX_CUDA(cudaEventRecord(ss->b_ready, lo));
    stage_mark(1, lo);
    return OK;
  };
  if (b_after_y != 2) APX_TRY(b_stage());
  // ---- hi: QR, Bm (+||A||^2), dA in f16 -----------------------------------------------------------
  APX_TRY((qr_orthonormalize<float, float>(Y, l, 1, n, l, Q, l, 1, Qt, 1, n, p.qr_ws, p.qr_bytes, 0, hi, /*tf32=*/1)));
  for (int it = 0; it < q; ++it) {
    APX_TRY(UmmaStages::at_times_x(A, Q, Z, part, n, l, hi));
    APX_TRY((qr_orthonormalize<float, float>(Z, l, 1, n, l, Q, l, 1, Qt, 1, n, p.qr_ws, p.qr_bytes, 0, hi, /*tf32=*/1)));
    APX_TRY(UmmaStages::a_times_x(A, Q, Y, part, n, l, hi));
    APX_TRY((qr_orthonormalize<float, float>(Y, l, 1, n, l, Q, l, 1, Qt, 1, n, p.qr_ws, p.qr_bytes, 0, hi, /*tf32=*/1)));
  }
  stage_mark(4, hi);
  if (b_after_y == 2) {
    APX_CUDA(cudaEventRecord(ss->b_read, hi));
    APX_CUDA(cudaStreamWaitEvent(lo, ss->b_read, 0));
    APX_TRY(b_stage());
  }
  {
    // Bm = Q^T A with the A tiles rounded to TF32 (FIX 3): the rounding warps also sum the
    // squares of every A element they touch (each exactly once) -> ||A||^2 partials. Then one
    // finalize kernel: split-K sum, ||Bm||^2 (= sum sigma^2, the report's kept energy) from Bm as
    // formed, Bm := tf32(Bm) (the algebra holds for any Bm -- but the energy difference
    // ||A||^2 - ||Bm||^2 would feel the rounding: ~2e-5 of ||Bm||^2 when a few rows carry the
    // energy; with Q TF32-exact too, Q.Bm is then exact on the tensor core at K = l), [Q | Q], and
    // the fixed-order sums of both norms.
    const int s = UmmaStages::splits(n);
    APX_TRY(umma_tma_gemm(7 | 8 | 16, 64, A, n, Q, l, part, n, (int64_t)l * n, n, l, n, s, 0, nullptr, 0, 1, hi,
                          p.asq));
    stage_mark(16, hi);
    // APX_RESID_F16=1 / 0 forces the f16 residual / the fp32 fallback (tests); default: decided on
    // the device from the residual energy (bm_finalize_kernel)
    static const int f16_mode = [] {
      const char* e = getenv("APX_RESID_F16");
      return e ? (atoi(e) ? 1 : 2) : 0;
    }();
    APX_TRY(launch_bm_finalize(part, s, l, n, Bm, Q, p.Q2, p.bsq, p.asq, (int)(ceil_div(n, 128) * s),
                               reinterpret_cast<unsigned*>(p.ticket + 2), scal + APX_S_KEPT_A, scal + APX_S_FRO2_A,
                               p.ticket + 3, f16_mode, hi));
  }
  stage_mark(5, hi);
  // APX_W0_EARLY=1: the low-priority chain (W0 = Bm.B ...) starts once Bm exists, beside the dA
  // pass, instead of behind it (tuning knob; APX_W0_SMS: the SM budget W0's K split is sized for)
  static const int w0_early = getenv("APX_W0_EARLY") ? atoi(getenv("APX_W0_EARLY")) : 0;
  static const int w0_sms = getenv("APX_W0_SMS") ? atoi(getenv("APX_W0_SMS")) : 0;
  cudaEvent_t da_ready = ss->join;  // reused: recorded again at the end of lo
  if (w0_early) APX_CUDA(cudaEventRecord(da_ready, hi));
  // dA as scaled f16 (or, in the fallback, as fp32 into M, which is free until the gather)
  APX_TRY(umma_tma_gemm(2 | 32, 128, Q, l, Bm, n, const_cast<float*>(A), n, 0, n, n, l, 1, 0, nullptr, 0, 1, hi,
                        nullptr, nullptr, 0, nullptr, nullptr, p.dAh, scal + APX_S_FRO2_A, p.ticket + 3, M));
  stage_mark(10, hi);
  if (!w0_early) APX_CUDA(cudaEventRecord(da_ready, hi));
  // ---- hi: the f16 gather M = dA . Bhat -------------------------------------------------------------
  APX_CUDA(cudaStreamWaitEvent(hi, ss->b_ready, 0));
  stage_mark(11, hi);
  APX_TRY(launch_gather_f16(p.dAh, p.lamh, sb, kc, kp, n, n, M, scal + APX_S_FRO2_A, scal + APX_S_FRO2_B, p.ticket,
                            p.ready, gctas, hi, nullptr, p.ticket + 3));
  // fallback (dA too large a part of M for f16): the fp32 gather over dA, in place in M (each
  // persistent CTA stages its whole row block before writing those rows), then all row flags;
  // both launches return at once when the f16 gather ran
  APX_TRY(launch_cycle_right_gather<float>(M, nullptr, 0, lb, sb, kc, n, n, 0, M, nullptr, nullptr, hi, true, gctas,
                                           p.ticket, 1, false, nullptr, false, 0, p.ticket + 3));
  APX_TRY(launch_fallback_flags(p.ticket + 3, p.ready, rblocks, hi));
  stage_mark(2, hi);
  APX_CUDA(cudaEventRecord(ss->hi_done, hi));
  // ---- lo: W = Bm . B at fp32 accuracy, then M += [Q|Q].[W_hi; W_lo] behind the gather's frontier --
  // (after dA: the W GEMM's HBM pass would otherwise slow the critical dA pass)
  APX_CUDA(cudaStreamWaitEvent(lo, da_ready, 0));
  const int wblocks = (int)ceil_div(l, right_gather_rows(n, sizeof(float), kc));
  const int wchunks = std::max(1, std::min(8, (int)ceil_div(5 * free_sms, wblocks)));
  APX_TRY(UmmaStages::bm_times_db(B, Bm, W, part, n, l, nullptr, 0, lo, w0_sms > 0 ? w0_sms : free_sms));
  stage_mark(9, lo);
  // W0 - Bm.Bhat_tf32 + Bm.Bhat as ONE gather over lambda - tf32(lambda): Bm is TF32-exact (the
  // finalize rounded it), so the TF32 and fp32 gathers differ only in lambda's truncated bits (two
  // gathers, each a few waves of 192 KB CTAs on the SMs the f16 gather leaves, were 163 us of the
  // low-priority chain, which sets the product's end)
  APX_TRY(launch_cycle_right_gather<float>(Bm, nullptr, 0, lb, sb, kc, n, l, 1, W, nullptr, nullptr, lo, true, 0,
                                           nullptr, wchunks, /*tf32_operands=*/2));
  APX_TRY(launch_split_tf32(W, (size_t)l * n, p.W2, lo));
  stage_mark(6, lo);
  // one tile per CTA (3 CTAs per SM on the SMs the gather leaves free). APX_QW_PERSIST=1: the
  // persistent, TMEM double-buffered, dynamically scheduled kernel with TMA epilogues instead (same
  // tile numbering, so the fixup is shared) -- faster alone (111 vs 114 us RMW, 75 vs 121 us plain
  // store at n = 8192) but one CTA per SM beside the gather: 1109 vs 1133 products/s.
  static const bool persist = getenv("APX_QW_PERSIST") != nullptr;
  if (persist) {
    APX_TRY(umma_persist_gemm(p.Q2, 2 * l, p.W2, n, M, n, n, n, 2 * l, 1, lo, p.msq, p.ready, grows, p.ticket, defer,
                              device_sms(), 128, p.ticket + 1));
  } else {
    APX_TRY(UmmaStages::q_times_w(p.Q2, p.W2, M, n, 2 * l, lo, 1, p.msq, p.ready, grows, p.ticket, defer));
  }
  stage_mark(7, lo);
  APX_CUDA(cudaStreamWaitEvent(lo, ss->hi_done, 0));
  APX_TRY(launch_qw_fixup_sum(p.Q2, 2 * l, p.W2, n, M, n, n, n, 2 * l, 128, defer, p.msq,
                              UmmaStages::q_times_w_ctas(n, 2 * l, 1), scal + APX_S_FRO2_M, lo));
  APX_CUDA(cudaEventRecord(ss->join, lo));
  APX_CUDA(cudaStreamWaitEvent(st, ss->join, 0));
  APX_CUDA(cudaStreamWaitEvent(st, ss->hi_done, 0));
  stage_mark(8, st);
  return OK;
}

// ---- the C4 product sharded by rows of A and M -------------------------------------
// Rank g holds the row block A_g (m x n) and the whole B; it computes M_g = Q_g W + A_g Bhat. The
// plan of run_mixed_f32_umma is cut at the four points where the rows must be combined; between
// phases the caller sums `red_out` over the ranks in place (an NCCL all-reduce on `stream`):
//   1: B's cycle decomposition and the gather M_g = A_g Bhat start on hi (the gather runs through
//      the later phases); Y_g = A_g Omega and its Gram matrix (out: l x l fp64)
//   2: R1^{-1} from the summed Gram, Q_g = Y_g R1^{-1}, the pass-2 Gram (out: l x l fp64, zero
//      when the conditioning lets pass 2 be skipped -- the same decision on every rank)
//   3: pass 2 when needed; Bm_g = Q_g^T A_g (out: l x n fp32)
//   4: W = Bm dB from the summed Bm (B is whole on every rank), M_g += Q_g W as the gather
//      releases row blocks (out: [||A_g||^2, ||M_g||^2, Cholesky breakdown])
struct RowsPlan {
  MixedPlan mp;
  void* qr;
  size_t qr_bytes;
  double* asum;  // ||A_g||^2 (hi, phase 1) until phase 4 reports it
};

static void plan_rows(Workspace& ws, RowsPlan& r, int n, int m, int l, int kc) {
  plan_mixed(ws, r.mp, F32, n, l, kc);
  r.qr_bytes = cholqr_rows_ws(m, l);
  r.qr = ws.take<char>(r.qr_bytes);
  r.asum = ws.take<double>(1);
}

static int run_mixed_rows_phase(int phase, const float* A, int m, const float* B, int n, int l, int kc, int order,
                                int flags, const float* Omega, float* M, int* sb, const void* red_in, void* red_out,
                                double* scal, const RowsPlan& r, cudaStream_t st) {
  const MixedPlan& p = r.mp;
  SideStream* ss = nullptr;
  APX_TRY(get_side(&ss));
  const cudaStream_t hi = ss->hi, lo = ss->s;
  const int grows = right_gather_rows(n, sizeof(float), kc);
  const int rblocks = (int)ceil_div(m, grows);
  const int gctas = gather_ctas(rblocks);
  const int free_sms = std::max(8, kNumSMs - gctas);
  float *Y = (float*)p.Y, *Q = (float*)p.Q, *W = (float*)p.W, *part = (float*)p.part;
  float* lb = (float*)p.lam_b;
  if (phase == 1) {
    APX_CUDA(cudaMemsetAsync(scal, 0, APX_NSCALARS * sizeof(double), st));
    APX_CUDA(cudaMemsetAsync(p.ready, 0, (rblocks + 1) * sizeof(int), st));
    APX_CUDA(cudaMemsetAsync(p.ticket, 0, sizeof(int), st));
    APX_CUDA(cudaEventRecord(ss->fork, st));
    APX_CUDA(cudaStreamWaitEvent(lo, ss->fork, 0));
    APX_CUDA(cudaStreamWaitEvent(hi, ss->fork, 0));
    APX_TRY(launch_cycle_energies<float>(B, n, p.en_b, p.nr_b, nullptr, p.partial, hi));
    APX_CUDA(cudaEventRecord(ss->b_read, hi));
    APX_TRY(launch_topk(p.nr_b, n, kc, sb, hi, p.nr_b, 1.0, scal + APX_S_KEPT_B, p.en_b, scal + APX_S_FRO2_B));
    APX_TRY(launch_cycle_extract<float>(B, n, sb, kc, lb, hi, /*aligned=*/true));
    APX_TRY(zero_pad_rows<float>(lb, kc, n, hi));
    APX_CUDA(cudaEventRecord(ss->b_ready, hi));
    if (order == 1) {
      APX_TRY(launch_cycle_right_gather<float>(A, nullptr, 0, lb, sb, kc, n, m, 0, M, nullptr, p.asq, hi, true, gctas,
                                               p.ticket, 1, false, p.ready, /*x_early=*/true));
      APX_TRY(launch_sum_vector(p.asq, rblocks, r.asum, hi));  // ||A_g||^2 (gather partials)
    } else {
      int parts = 0;
      APX_TRY(launch_sumsq<float>(A, (size_t)m * n, p.asq, &parts, hi));
      APX_TRY(launch_sum_vector(p.asq, parts, r.asum, hi));
    }
    APX_CUDA(cudaEventRecord(ss->hi_done, hi));
    APX_CUDA(cudaStreamWaitEvent(lo, ss->b_read, 0));
    const int s = std::max(1, std::min(8, (int)((2 * 32) / ceil_div(m, 128))));
    APX_TRY(umma_tma_gemm(2, 64, A, n, Omega, l, s > 1 ? part : Y, l, (int64_t)m * l, m, l, n, s, 0, nullptr, 0, 1,
                          lo));
    if (s > 1) APX_TRY(launch_split_reduce_f32(part, s, (size_t)m * l, Y, lo));
    APX_TRY(cholqr_rows_gram(Y, m, l, (double*)red_out, r.qr, r.qr_bytes, lo));
  } else {
    APX_CUDA(cudaEventRecord(ss->fork, st));  // the caller's all-reduce of the previous phase's output
    APX_CUDA(cudaStreamWaitEvent(lo, ss->fork, 0));
  }
  if (phase == 2)
    APX_TRY(cholqr_rows_pass1(Y, m, l, (const double*)red_in, Q, (double*)red_out, r.qr, r.qr_bytes, lo));
  if (phase == 3) {
    APX_TRY(cholqr_rows_pass2(m, l, (const double*)red_in, Q, r.qr, r.qr_bytes, lo));
    // Bm_g = Q_g^T A_g, computed as (A_g^T Q_g) stored transposed
    const int s = UmmaStages::splits(n, free_sms);
    APX_TRY(umma_tma_gemm(7 | 8, 64, A, n, Q, l, s > 1 ? part : (float*)red_out, n, (int64_t)l * n, n, l, m, s, 0,
                          nullptr, 0, 1, lo));
    if (s > 1) APX_TRY(launch_split_reduce_f32(part, s, (size_t)n * l, (float*)red_out, lo));
  }
  if (phase == 4) {
    const float* Bm = (const float*)red_in;
    double* fin = (double*)red_out;  // [||A_g||^2, ||M_g||^2, breakdown]
    int parts = 0;
    APX_TRY(launch_sumsq<float>(Bm, (size_t)l * n, p.bsq, &parts, lo));
    APX_TRY(launch_sum_vector(p.bsq, parts, scal + APX_S_KEPT_A, lo));
    const int wblocks = (int)ceil_div(l, grows);
    const int wchunks = std::max(1, std::min(8, (int)ceil_div(5 * free_sms, wblocks)));
    if (order == 1) APX_TRY(UmmaStages::bm_times_db(B, Bm, W, part, n, l, nullptr, 0, lo, free_sms));
    APX_CUDA(cudaStreamWaitEvent(lo, ss->b_ready, 0));
    APX_TRY(launch_cycle_right_gather<float>(Bm, nullptr, 0, lb, sb, kc, n, l, order == 1 ? -1 : 0, W, nullptr,
                                             nullptr, lo, true, 0, nullptr, wchunks, /*tf32_operands=*/order == 1));
    // flags & 1: M += Q.W only after the whole gather (several shards on one device, whose gathers
    // are queued behind each other on hi: a waiting Q.W grid could hold the SMs a later gather needs)
    if (flags & 1) APX_CUDA(cudaStreamWaitEvent(lo, ss->hi_done, 0));
    const int qw_ctas = (int)(ceil_div(n, order == 1 ? 128 : 256) * ceil_div(m, 128));
    int* defer = order == 1 ? p.ready + rblocks : nullptr;  // bounded wait (see run_mixed_f32_umma)
    APX_TRY(umma_tma_gemm(2, order == 1 ? 128 : 256, Q, l, W, n, M, n, 0, m, n, l, 1, order == 1 ? 1 : 0, nullptr, 0,
                          1, lo, p.msq, order == 1 ? p.ready : nullptr, grows, order == 1 ? p.ticket : nullptr,
                          defer));
    APX_CUDA(cudaStreamWaitEvent(lo, ss->hi_done, 0));
    if (order == 1)
      APX_TRY(launch_qw_fixup_sum(Q, l, W, n, M, n, m, n, l, 128, defer, p.msq, qw_ctas, fin + 1, lo));
    else
      APX_TRY(launch_sum_vector(p.msq, qw_ctas, fin + 1, lo));
    APX_CUDA(cudaMemcpyAsync(fin, r.asum, sizeof(double), cudaMemcpyDeviceToDevice, lo));
    APX_TRY(launch_flag_to_double(cholqr_rows_flags(r.qr, r.qr_bytes, m, l), fin + 2, lo));
    APX_CUDA(cudaEventRecord(ss->join, lo));
    APX_CUDA(cudaStreamWaitEvent(st, ss->join, 0));
    return OK;
  }
  APX_CUDA(cudaEventRecord(ss->join, lo));
  APX_CUDA(cudaStreamWaitEvent(st, ss->join, 0));
  return OK;
}

template <typename T>
static int run_mixed(const T* A, const T* B, int n, int l, int kc, int order, int q, const T* Omega, const int* fb,
                     T* M, int* sb, double* scal, const MixedPlan& p, bool split3, cudaStream_t st) {
  stage_mark(0, st);
  APX_CUDA(cudaMemsetAsync(scal, 0, APX_NSCALARS * sizeof(double), st));
  // B: cycle norms, selection, kept diagonals
  APX_TRY(launch_cycle_energies<T>(B, n, p.en_b, p.nr_b, scal + APX_S_FRO2_B, p.partial, st));
  if (fb) { if (kc) APX_CUDA(cudaMemcpyAsync(sb, fb, kc * sizeof(int), cudaMemcpyDeviceToDevice, st)); }
  else APX_TRY(launch_topk(p.nr_b, n, kc, sb, st));
  APX_TRY(launch_kept_energy(p.nr_b, sb, kc, 1.0, scal + APX_S_KEPT_B, st));
  T* lb = (T*)p.lam_b;
  APX_TRY(launch_cycle_extract<T>(B, n, sb, kc, lb, st, /*aligned=*/true));
  APX_TRY(zero_pad_rows<T>(lb, kc, n, st));
  stage_mark(1, st);
  // A: randomized range finder (svd.py:105-111)
  T *Y = (T*)p.Y, *Q = (T*)p.Q, *Qt = (T*)p.Qt, *Z = (T*)p.Z, *Bm = (T*)p.Bm, *W = (T*)p.W, *part = (T*)p.part;
  const int s0 = gemm_splits(n, l, n, 128, 64);
  const int s1 = gemm_splits(l, n, n, 64, 128);
  APX_TRY(gemm_skinny<T>(0, A, n, Omega, l, Y, l, n, l, n, 0, nullptr, 0, 1, part, s0, split3, st));
  stage_mark(2, st);
  APX_TRY((qr_orthonormalize<T, T>(Y, l, 1, n, l, Q, l, 1, Qt, 1, n, p.qr_ws, p.qr_bytes, 0, st)));
  for (int it = 0; it < q; ++it) {
    // Q <- qr(A^T Q) with A^T Q = (Q^T A)^T, then Q <- qr(A Q)
    APX_TRY(gemm_skinny<T>(1, Qt, n, A, n, Z, n, l, n, n, 0, nullptr, 0, 1, part, s1, split3, st));
    APX_TRY((qr_orthonormalize<T, T>(Z, 1, n, n, l, Q, l, 1, Qt, 1, n, p.qr_ws, p.qr_bytes, 0, st)));
    APX_TRY(gemm_skinny<T>(0, A, n, Q, l, Y, l, n, l, n, 0, nullptr, 0, 1, part, s0, split3, st));
    APX_TRY((qr_orthonormalize<T, T>(Y, l, 1, n, l, Q, l, 1, Qt, 1, n, p.qr_ws, p.qr_bytes, 0, st)));
  }
  stage_mark(3, st);
  // Bm = Q^T A; ||Bm||_F^2 = sum sigma^2
  APX_TRY(gemm_skinny<T>(1, Qt, n, A, n, Bm, n, l, n, n, 0, nullptr, 0, 1, part, s1, split3, st));
  int parts = 0;
  APX_TRY(launch_sumsq<T>(Bm, (size_t)l * n, p.msq, &parts, st));
  APX_TRY(launch_sum_vector(p.msq, parts, scal + APX_S_KEPT_A, st));
  stage_mark(4, st);
  if (order == 1) {
    // W = Bm . dB (kept cycles of B masked on load), M = Q W, M += A . Bhat (+ ||M||^2, ||A||^2)
    APX_TRY(gemm_skinny<T>(1, Bm, n, B, n, W, n, l, n, n, 0, sb, kc, n, part, s1, split3, st));
    stage_mark(5, st);
    APX_TRY(gemm_skinny<T>(2, Q, l, W, n, M, n, n, n, l, 0, nullptr, 0, 1, nullptr, 1, split3, st));
    stage_mark(6, st);
    APX_TRY(launch_cycle_right_gather<T>(A, nullptr, 0, lb, sb, kc, n, n, 1, M, p.msq, p.asq, st, true));
    stage_mark(7, st);
    const int rblocks = (int)ceil_div(n, right_gather_rows_plain(n, sizeof(T), kc));
    APX_TRY(launch_sum_vector(p.msq, rblocks, scal + APX_S_FRO2_M, st));
    APX_TRY(launch_sum_vector(p.asq, rblocks, scal + APX_S_FRO2_A, st));
  } else {
    APX_TRY(launch_cycle_right_gather<T>(Bm, nullptr, 0, lb, sb, kc, n, l, 0, W, p.msq, nullptr, st, true));
    APX_TRY(gemm_skinny<T>(2, Q, l, W, n, M, n, n, n, l, 0, nullptr, 0, 1, nullptr, 1, split3, st));
    APX_TRY(launch_sumsq<T>(M, (size_t)n * n, p.msq, &parts, st));
    APX_TRY(launch_sum_vector(p.msq, parts, scal + APX_S_FRO2_M, st));
    APX_TRY(launch_sumsq<T>(A, (size_t)n * n, p.asq, &parts, st));
    APX_TRY(launch_sum_vector(p.asq, parts, scal + APX_S_FRO2_A, st));
  }
  stage_mark(8, st);
  return OK;
}

}  // namespace apx

using namespace apx;

extern "C" {

int apx_abi_version(void) { return 1; }

long long apx_launch_count(void) { return g_launches.load(std::memory_order_relaxed); }

int apx_set_stage_events(void** events, int count) {
  g_stage_ev = reinterpret_cast<cudaEvent_t*>(events);
  g_stage_n = events ? count : 0;
  return OK;
}

const char* apx_last_error(void) { return g_err; }

int apx_top_indices(const double* w, int64_t n, int k, int32_t* sel, void* stream) {
  APX_REQUIRE(n >= 1, "n must be >= 1");
  APX_REQUIRE(k >= 0 && k <= n, "k=%d out of range [0, %lld]", k, (long long)n);
  return launch_topk(w, (int)n, k, sel, S(stream));
}

size_t apx_cycle_norms_workspace(int dtype, int64_t n) {
  (void)dtype;
  Workspace ws(nullptr, 0, true);
  ws.take<double>(cycle_energy_ws((int)n) / sizeof(double) + 1);
  ws.take<double>(n);
  return ws.off;
}

int apx_cycle_norms(int dtype, const void* A, int64_t n, double* norms, double* fro2, void* wsp, size_t ws_bytes,
                    void* stream) {
  APX_REQUIRE(dtype == F32 || dtype == F64, "cycle_norms: real dtype required");
  APX_REQUIRE(n >= 1 && n <= 46340, "n=%lld out of range", (long long)n);
  Workspace ws(wsp, ws_bytes);
  double* partial = ws.take<double>(cycle_energy_ws((int)n) / sizeof(double) + 1);
  double* en = ws.take<double>(n);
  APX_WS_CHECK(ws);
  if (dtype == F32) return launch_cycle_energies<float>((const float*)A, (int)n, en, norms, fro2, partial, S(stream));
  return launch_cycle_energies<double>((const double*)A, (int)n, en, norms, fro2, partial, S(stream));
}

size_t apx_cycle_first_order_workspace(int dtype, int64_t n, int k_a, int k_b, int order) {
  Workspace ws(nullptr, 0, true);
  CyclePlan p;
  plan_cycle(ws, p, dtype, (int)n, k_a, k_b, order);
  return ws.off;
}

int apx_cycle_first_order(int dtype, const void* A, const void* B, int64_t n, int k_a, int k_b, int order,
                          const int32_t* force_sel_a, const int32_t* force_sel_b, void* M, int32_t* sel_a,
                          int32_t* sel_b, double* scalars, void* wsp, size_t ws_bytes, void* stream) {
  APX_NVTX("apx_cycle_first_order");
  APX_REQUIRE(dtype == F32 || dtype == F64, "cycle product: real dtype required");
  APX_REQUIRE(n >= 1 && n <= 46340, "n=%lld out of range", (long long)n);
  APX_REQUIRE(k_a >= 0 && k_a <= n && k_b >= 0 && k_b <= n, "k out of range [0, %lld]", (long long)n);
  APX_REQUIRE(order == 0 || order == 1, "order must be 0 or 1");
  Workspace ws(wsp, ws_bytes);
  CyclePlan p;
  plan_cycle(ws, p, dtype, (int)n, k_a, k_b, order);
  APX_WS_CHECK(ws);
  if (dtype == F32)
    return run_cycle<float>((const float*)A, (const float*)B, (int)n, k_a, k_b, order, force_sel_a, force_sel_b,
                            (float*)M, sel_a, sel_b, scalars, p, S(stream));
  return run_cycle<double>((const double*)A, (const double*)B, (int)n, k_a, k_b, order, force_sel_a, force_sel_b,
                           (double*)M, sel_a, sel_b, scalars, p, S(stream));
}

size_t apx_cycle_rows_workspace(int dtype, int64_t n, int64_t m_rows, int k_a, int k_b, int order) {
  Workspace ws(nullptr, 0, true);
  CycleRowsPlan p;
  plan_cycle_rows(ws, p, dtype, (int)n, (int)m_rows, k_a, k_b, order);
  return ws.off;
}

int apx_cycle_rows_phase(int phase, int dtype, const void* A_rows, int64_t m_rows, int64_t row0, const void* B,
                         int64_t n, int k_a, int k_b, int order, void* M_rows, int32_t* sel_a, int32_t* sel_b,
                         const double* red_in, double* red_out, double* scalars, void* wsp, size_t ws_bytes,
                         void* stream) {
  APX_NVTX("apx_cycle_rows_phase");
  APX_REQUIRE(phase == 1 || phase == 2, "phase must be 1 or 2");
  APX_REQUIRE(dtype == F32 || dtype == F64, "cycle product: real dtype required");
  APX_REQUIRE(n >= 1 && n <= 46340, "n=%lld out of range", (long long)n);
  APX_REQUIRE(m_rows >= 1 && row0 >= 0 && row0 + m_rows <= n, "row block [%lld, %lld) outside [0, %lld)",
              (long long)row0, (long long)(row0 + m_rows), (long long)n);
  APX_REQUIRE(k_a >= 0 && k_a <= n && k_b >= 0 && k_b <= n, "k out of range [0, %lld]", (long long)n);
  APX_REQUIRE(order == 0 || order == 1, "order must be 0 or 1");
  APX_REQUIRE(phase == 1 || red_in != nullptr, "phase 2 needs the summed energies");
  Workspace ws(wsp, ws_bytes);
  CycleRowsPlan p;
  plan_cycle_rows(ws, p, dtype, (int)n, (int)m_rows, k_a, k_b, order);
  APX_WS_CHECK(ws);
  if (dtype == F32)
    return run_cycle_rows<float>(phase, (const float*)A_rows, (int)m_rows, (int)row0, (const float*)B, (int)n, k_a,
                                 k_b, order, (float*)M_rows, sel_a, sel_b, red_in, red_out, scalars, p, S(stream));
  return run_cycle_rows<double>(phase, (const double*)A_rows, (int)m_rows, (int)row0, (const double*)B, (int)n, k_a,
                                k_b, order, (double*)M_rows, sel_a, sel_b, red_in, red_out, scalars, p, S(stream));
}

int apx_debug_umma_gemm(int layout, int bn, const float* A, int64_t lda, const float* B, int64_t ldb, float* C,
                        int64_t ldc, int64_t M, int64_t N, int64_t K, int splits, int accumulate, const int32_t* mask_j,
                        int mask_k, int mod_n, void* stream) {
  APX_REQUIRE(M >= 1 && N >= 1 && K >= 1 && splits >= 1, "bad GEMM shape");
  const int64_t slice = (int64_t)((layout & 4) ? N : M) * ldc;
  if (layout & 64) {  // persistent tile loop (layout 2 only); mod_n = CTA count (0: one per SM);
    // layout bit 128: dynamic tile scheduling with mask_j as the (int) ticket counter
    APX_REQUIRE((layout & 7) == 2 && splits == 1 && mask_k == 0, "persistent GEMM: layout 2, no split, no mask");
    return umma_persist_gemm(A, lda, B, ldb, C, ldc, (int)M, (int)N, (int)K, accumulate, S(stream), nullptr, nullptr,
                             0, nullptr, nullptr, mod_n, bn, (layout & 128) ? const_cast<int32_t*>(mask_j) : nullptr);
  }
  if (layout & 32)
    return umma_tma_gemm(layout & 15, bn, A, lda, B, ldb, C, ldc, slice, (int)M, (int)N, (int)K, splits,
                         accumulate, mask_j, mask_k, mod_n, S(stream));
  return umma_gemm(layout, bn, A, lda, B, ldb, C, ldc, slice, (int)M, (int)N, (int)K, splits, accumulate,
                   mask_j, mask_k, mod_n, S(stream));
}

size_t apx_mixed_first_order_workspace(int dtype, int64_t n, int k_svd, int k_cyc, int order) {
  (void)order;
  Workspace ws(nullptr, 0, true);
  MixedPlan p;
  plan_mixed(ws, p, dtype, (int)n, k_svd, k_cyc);
  return ws.off;
}

size_t apx_mixed_rows_workspace(int64_t n, int64_t m_rows, int k_svd, int k_cyc) {
  Workspace ws(nullptr, 0, true);
  RowsPlan r;
  plan_rows(ws, r, (int)n, (int)m_rows, k_svd, k_cyc);
  return ws.off;
}

int apx_mixed_rows_phase(int phase, const float* A_rows, int64_t m_rows, const float* B, int64_t n, int k_svd,
                         int k_cyc, int order, int flags, const float* omega, float* M_rows, int32_t* sel_b,
                         const void* red_in, void* red_out, double* scalars, void* wsp, size_t ws_bytes,
                         void* stream) {
  APX_NVTX("apx_mixed_rows_phase");
  APX_REQUIRE(phase >= 1 && phase <= 4, "phase must be 1..4");
  APX_REQUIRE(n >= 128 && n <= 46340 && (n % 32) == 0, "n=%lld: the sharded product needs n %% 32 == 0, n >= 128",
              (long long)n);
  APX_REQUIRE(m_rows >= 64 && m_rows <= n, "m_rows=%lld out of range [64, n]", (long long)m_rows);
  APX_REQUIRE(k_svd == 64, "the sharded product is planned for k_svd = 64");
  APX_REQUIRE(k_cyc >= 0 && k_cyc <= 128 && k_cyc <= n, "k_cyc=%d out of range [0, 128]", k_cyc);
  APX_REQUIRE(order == 0 || order == 1, "order must be 0 or 1");
  APX_REQUIRE(phase == 1 || red_in != nullptr, "phase %d needs the all-reduced output of phase %d", phase, phase - 1);
  Workspace ws(wsp, ws_bytes);
  RowsPlan r;
  plan_rows(ws, r, (int)n, (int)m_rows, k_svd, k_cyc);
  APX_WS_CHECK(ws);
  return run_mixed_rows_phase(phase, A_rows, (int)m_rows, B, (int)n, k_svd, k_cyc, order, flags, omega, M_rows, sel_b,
                              red_in, red_out, scalars, r, S(stream));
}

int apx_mixed_first_order(int dtype, const void* A, const void* B, int64_t n, int k_svd, int k_cyc, int order,
                          int power_iterations, const void* omega, const int32_t* force_sel_b, int flags, void* M,
                          int32_t* sel_b, double* scalars, void* wsp, size_t ws_bytes, void* stream) {
  APX_NVTX("apx_mixed_first_order");
  APX_REQUIRE(dtype == F32 || dtype == F64, "mixed product: real dtype required");
  APX_REQUIRE(n >= 2 && n <= 46340, "n=%lld out of range", (long long)n);
  APX_REQUIRE(k_svd >= 1 && k_svd <= 128 && k_svd <= n, "k_svd=%d out of range [1, min(n,128)]", k_svd);
  APX_REQUIRE(k_cyc >= 0 && k_cyc <= n, "k_cyc=%d out of range [0, %lld]", k_cyc, (long long)n);
  APX_REQUIRE(order == 0 || order == 1, "order must be 0 or 1");
  APX_REQUIRE(power_iterations >= 0, "power_iterations must be >= 0");
  Workspace ws(wsp, ws_bytes);
  MixedPlan p;
  plan_mixed(ws, p, dtype, (int)n, k_svd, k_cyc);
  APX_WS_CHECK(ws);
  const bool split3 = (flags & 1) != 0;
  // tcgen05 path: fp32, l == 64 (one N=64 tile), n a multiple of 4 (16-byte rows), <= 128 masked
  // cycles; 3xTF32 requests and other shapes use the mma.sync path
  const bool umma_ok = dtype == F32 && !split3 && k_svd == 64 && (n % 4) == 0 && k_cyc <= 128 && !(flags & 2);
  // residual plan (f16 gather over dA) unless flag 4 asks for the all-fp32 gather over A
  if (umma_ok && order == 1 && p.dAh != nullptr && !(flags & 4))
    return run_mixed_f32_resid((const float*)A, (const float*)B, (int)n, k_svd, k_cyc, power_iterations,
                               (const float*)omega, force_sel_b, (float*)M, sel_b, scalars, p, S(stream));
  if (umma_ok)
    return run_mixed_f32_umma((const float*)A, (const float*)B, (int)n, k_svd, k_cyc, order, power_iterations,
                              (const float*)omega, force_sel_b, (float*)M, sel_b, scalars, p, S(stream));
  if (dtype == F32)
    return run_mixed<float>((const float*)A, (const float*)B, (int)n, k_svd, k_cyc, order, power_iterations,
                            (const float*)omega, force_sel_b, (float*)M, sel_b, scalars, p, split3, S(stream));
  return run_mixed<double>((const double*)A, (const double*)B, (int)n, k_svd, k_cyc, order, power_iterations,
                           (const double*)omega, force_sel_b, (double*)M, sel_b, scalars, p, split3, S(stream));
}

}  // extern "C"
