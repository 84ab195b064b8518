// Host-side launcher declarations shared by the C-ABI translation unit.
#pragma once
#include "common.cuh"

namespace apx {

// ---- cycle.cu ----
size_t cycle_energy_ws(int n);
size_t cycle_energy_ws_groups(int n, int groups);
int right_gather_rows(int n, size_t elem, int k);
// rows per block of a plain right gather (no ticket / ready flags / TF32 operands): the segmented
// kernel's R at large n, else right_gather_rows
int right_gather_rows_plain(int n, size_t elem, int k);
int right_gather_seg_rows(int n, size_t elem, int k);
template <typename T>
int launch_cycle_energies(const T* A, int n, double* energies, double* norms, double* fro2, double* partial,
                          cudaStream_t st, int ctas_per_sm = 8, int groups_override = 0, int rows4_ctas = 0);
// top-k selection (select.cuh); optionally fused: *kept = kept_scale * sum_t kept_w[sel[t]]^2 and
// *total = sum_i tot_w[i]
int qr_sm_footprint(int m, int l);  // linalg.cu: SMs of the fused CholeskyQR2
int launch_topk(const double* w, int n, int k, int* sel, cudaStream_t st, const double* kept_w = nullptr,
                double kept_scale = 1.0, double* kept = nullptr, const double* tot_w = nullptr,
                double* total = nullptr);
int launch_kept_energy(const double* norms, const int* sel, int k, double scale, double* out, cudaStream_t st);
template <typename T>
int launch_cycle_extract(const T* A, int n, const int* J, int k, T* lam, cudaStream_t st, bool aligned = false);
template <typename T>
int launch_cycle_materialize(const T* lam, const int* J, int k, int n, T* out, cudaStream_t st);
template <typename T>
int launch_cycle_left_gather(const T* X, const T* lam, const int* J, int k, int n, int accumulate, T* M,
                             cudaStream_t st);
template <typename T>
int launch_cycle_right_gather(const T* X, const int* JA, int ka, const T* lam, const int* J, int k, int n, int m_rows,
                              int accumulate, T* M, double* msq_partial, double* xsq_partial, cudaStream_t st,
                              bool lam_padded = false, int max_ctas = 0, int* ticket = nullptr, int col_chunks = 1,
                              int tf32_operands = 0, int* ready = nullptr, bool x_early = false,
                              int row_off = 0, const int* skip_if = nullptr);
// f16-staged segmented gather of a small masked residual (cycle.cu K11h; fp32, large n)
bool right_gather_seg_f16_ok(int n, size_t elem, int k);
size_t right_gather_seg_f16_ws(int n, int k);
int launch_cycle_right_gather_seg_f16(const float* X, const int* JA, int ka, const float* lam, const int* J, int k,
                                      int n, int m_rows, int accumulate, float* M, double* msq_partial,
                                      cudaStream_t st, int row_off, unsigned short* lamh, const double* fro2_x,
                                      const double* kept_x, const double* fro2_b);
// ---- row-sharded cycle product (local rows [0, m) of an n x n operand = global rows row_off + r)
template <typename T>
int launch_cycle_energies_rows(const T* A, int m, int row_off, int n, double* energies, double* partial,
                               cudaStream_t st);
template <typename T>
int launch_cycle_extract_rows(const T* A, int m, int row_off, int n, const int* J, int k, T* lam, cudaStream_t st);
template <typename T>
int launch_cycle_left_gather_rows(const T* X, const T* lam, const int* J, int k, int n, int r_lo, int r_hi, T* M_rows,
                                  cudaStream_t st);
template <typename T>
int launch_cycle_right_gather_cols(const T* X, const T* lam, const int* J, int k, int n, int m_rows, int c_lo,
                                   int c_hi, T* M, cudaStream_t st);
template <typename T>
int launch_sumsq(const T* x, size_t cnt, double* partial, int* nparts, cudaStream_t st);
int launch_sum_vector(const double* v, int n, double* out, cudaStream_t st);

}  // namespace apx

namespace apx {
// ---- gemm.cu ----
int gemm_splits(int M, int N, int K, int BM, int BN);
int launch_split_reduce_f32(const float* part, int splits, size_t count, float* out, cudaStream_t st);
template <typename T>
int gemm_skinny(int kind, const T* A, int64_t lda, const T* B, int64_t ldb, T* C, int64_t ldc, int M, int N, int K,
                int accumulate, const int* mJ, int mk, int mod_n, T* part, int splits, bool split3, cudaStream_t st);
// ---- linalg.cu ----
size_t qr_ws_bytes(int m, int l);
size_t cholqr_rows_ws(int m, int l);
int cholqr_rows_gram(const float* Y, int m, int l, double* G, void* ws, size_t bytes, cudaStream_t st);
int cholqr_rows_pass1(const float* Y, int m, int l, const double* G, float* Q, double* G2, void* ws, size_t bytes,
                      cudaStream_t st);
int cholqr_rows_pass2(int m, int l, const double* G2, float* Q, void* ws, size_t bytes, cudaStream_t st);
const int* cholqr_rows_flags(void* ws, size_t bytes, int m, int l);
int launch_flag_to_double(const int* flag, double* out, cudaStream_t st);
template <typename TI, typename TO>
int qr_orthonormalize(const TI* Y, int64_t rs, int64_t cs, int m, int l, TO* Q, int64_t qrs, int64_t qcs, TO* Q2,
                      int64_t q2rs, int64_t q2cs, void* wsp, size_t ws_bytes, int method, cudaStream_t st,
                      int tf32 = 0);
}  // namespace apx

namespace apx {
// ---- umma.cu (tcgen05 TF32) ----
int umma_set_variant(int v);
int umma_tma_gemm(int layout, int bn, const float* A, int64_t lda, const float* B, int64_t ldb, float* C,
                  int64_t ldc, int64_t c_split_stride, int M, int N, int K, int splits, int accumulate,
                  const int* mJ, int mk, int mod_n, cudaStream_t st, double* sq_partial = nullptr,
                  const int* ready = nullptr, int ready_rows = 0, const int* progress = nullptr,
                  int* defer = nullptr, uint16_t* hout = nullptr, const double* hscale = nullptr,
                  const int* f16_flag = nullptr, float* out32 = nullptr);
int umma_persist_gemm(const float* A, int64_t lda, const float* B, int64_t ldb, float* C, int64_t ldc, int M, int N,
                      int K, int accumulate, cudaStream_t st, double* sq_partial = nullptr, const int* ready = nullptr,
                      int ready_rows = 0, const int* progress = nullptr, int* defer = nullptr, int ctas = 0,
                      int bn = 128, int* ticket = nullptr);
// deferred Q.W tiles of a ready-flag GEMM, then the fixed-order ||C||^2 sum (umma_tma.cu)
int launch_qw_fixup_sum(const float* Q, int64_t ldq, const float* W, int64_t ldw, float* C, int64_t ldc, int M, int N,
                        int K, int bn, int* defer, double* sq_partial, int parts, double* out, cudaStream_t st);
// ---- capi.cu: the calling thread's side stream (fork from / join back into `st`) ----
int side_fork(cudaStream_t st, cudaStream_t* side);
int side_join(cudaStream_t st, cudaStream_t side);
// ---- mixed_f16.cu (residual plan of the C4 product) ----
int launch_split_tf32(const float* X, size_t count, float* X2, cudaStream_t st);
int launch_dup_cols(const float* Q, int rows, int l, float* Q2, cudaStream_t st);
int launch_round_tf32(float* X, size_t count, cudaStream_t st);
int launch_bm_finalize(const float* part, int splits, int l, int n, float* Bm, const float* Q, float* Q2,
                       double* bsq_part, const double* asq_part, int asq_parts, unsigned* counter, double* kept_out,
                       double* fro2_out, int* use_f16, int f16_mode, cudaStream_t st);
int launch_fallback_flags(const int* use_f16, int* ready, int blocks, cudaStream_t st);
int gather_f16_threads(int n);
size_t gather_f16_smem(int n, int kp);
int launch_lam_f16(const float* lam, int kp, int n, const double* fro2_b, uint16_t* out, cudaStream_t st);
int launch_gather_f16(const uint16_t* Xh, const uint16_t* lamh, const int* J, int k, int kp, int n, int m_rows, float* M,
                      const double* fro2_a, const double* fro2_b, int* ticket, int* ready, int ctas, cudaStream_t st,
                      double* msq_partial = nullptr, const int* gate = nullptr);
int umma_gemm(int layout, int bn, const float* A, int64_t lda, const float* B, int64_t ldb, float* C, int64_t ldc,
              int64_t c_split_stride, int M, int N, int K, int splits, int accumulate, const int* mJ, int mk,
              int mod_n, cudaStream_t st);
}  // namespace apx

namespace apx {
// ---- svd.cu ----
// l > 128 runs from a global scratch of small_svd_scratch_doubles(l) doubles
size_t small_svd_scratch_doubles(int l);
int launch_small_svd(const double* W, int l, double* U, double* S, double* V, double* VT, cudaStream_t st,
                     double* scratch = nullptr);
int launch_axpy2d(double* y, int64_t ldy, const double* x, int64_t ldx, int rows, int cols, double alpha,
                  const double* rowscale, int overwrite, cudaStream_t st);
int launch_sumsq_prefix(const double* s, int k, double* out, cudaStream_t st);
int launch_transpose_f64(const double* in, int64_t ldi, int rows, int cols, double* out, int64_t ldo, cudaStream_t st);
int launch_transpose_f32(const float* in, int64_t ldi, int rows, int cols, float* out, int64_t ldo, cudaStream_t st);
int launch_transpose_c128(const double2* in, int64_t ldi, int rows, int cols, double2* out, int64_t ldo,
                          cudaStream_t st);
inline int launch_transpose_any(const float* in, int64_t ldi, int rows, int cols, float* out, int64_t ldo,
                                cudaStream_t st) {
  return launch_transpose_f32(in, ldi, rows, cols, out, ldo, st);
}
inline int launch_transpose_any(const double* in, int64_t ldi, int rows, int cols, double* out, int64_t ldo,
                                cudaStream_t st) {
  return launch_transpose_f64(in, ldi, rows, cols, out, ldo, st);
}
// out[t] = (n - J[t]) mod n
int launch_negate_shifts(const int* J, int k, int n, int* out, cudaStream_t st);
// true when the left gather (column strips of width <= 2) is better replaced by the transposed
// right gather (A.X = (X^T A^T)^T) -- large n, where a column strip barely fits shared memory
bool left_via_transpose(int n, size_t elem, int k);
}  // namespace apx
