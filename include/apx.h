/*
 * apx.h -- C-ABI of the B200-native approximate dense product (arXiv 2504.19308).
 *
 * Drop-in boundary for the reference package `apxmm` (pkg/src/apxmm). The reference has no
 * plugin registry: its boundary is the set of module-level Python functions listed per entry
 * point below (file:line under /root/reference/pkg/src/apxmm/). The Python shim in
 * paper_2504_19308_b200/ keeps those exact signatures and calls these functions via ctypes.
 *
 * Conventions
 *   - Every matrix argument is a DEVICE pointer to a dense row-major array (leading dim = cols).
 *   - dtype: APX_F32 / APX_F64 real inputs; complex outputs use interleaved (re, im) pairs.
 *   - `stream` is a cudaStream_t passed as void*; all work is enqueued on it, nothing blocks,
 *     nothing is allocated: the caller owns `ws` (size from the matching *_workspace call).
 *   - Selected component indices are written to device int32 arrays, ascending.
 *   - `scalars` is a device array of APX_NSCALARS doubles (see APX_S_* slots); the shim turns
 *     them into the reference's ApproxReport (report.py:8-36) fields.
 *   - Return value 0 = success; nonzero = APX_E_* code, message via apx_last_error() (thread
 *     local). APX_E_ARG maps to the reference's ValueError.
 *   - Thread state: the error string, the optional stage events (apx_set_stage_events) and, for
 *     the multi-stream C4 plan, one pair of internal side streams per (host thread, device)
 *     pair -- created lazily on the device that is current at the call. The only process-wide
 *     state is the launch counter (an atomic). Calls from different threads never share streams;
 *     calls from one thread on one device serialise on that thread's side streams.
 */
#ifndef APX_H_
#define APX_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define APX_F32 0
#define APX_F64 1
#define APX_C64 2
#define APX_C128 3

#define APX_OK 0
#define APX_E_ARG 1
#define APX_E_CUDA 2
#define APX_E_WS 3
#define APX_E_NUMERIC 4
#define APX_E_UNSUPPORTED 5

/* scalar slots written by the product entry points */
#define APX_S_FRO2_A 0  /* ||A||_F^2 */
#define APX_S_FRO2_B 1  /* ||B||_F^2 */
#define APX_S_KEPT_A 2  /* energy captured by A's kept components */
#define APX_S_KEPT_B 3  /* energy captured by B's kept components */
#define APX_S_FRO2_M 4  /* ||M||_F^2 */
#define APX_S_RES2_A 5  /* ||dA||_F^2 measured directly (sfft only), else 0 */
#define APX_S_RES2_B 6  /* ||dB||_F^2 measured directly (sfft only), else 0 */
#define APX_NSCALARS 8

int apx_abi_version(void);
const char* apx_last_error(void);

/* diagnostics: number of kernels this library has launched since it was loaded, and
 * thread-local stage-boundary events (cudaEvent_t*, recorded on the call's stream at each
 * stage boundary of the product entry points; NULL disables). Used by bench.py. */
long long apx_launch_count(void);
int apx_set_stage_events(void** events, int count);

/* ---------------------------------------------------------------- selection primitives ---- */

/* top_indices (circulant.py:63-70): k largest of w[0..n) (non-negative doubles, device),
 * ties toward the lower index, written ascending to sel[0..k). */
int apx_top_indices(const double* w, int64_t n, int k, int32_t* sel, void* stream);

/* Cycle norms ||lambda_j||_2 of the left layout, i.e. the column norms of
 * cycle_reorder(A, "left") (core.py:106-125, left branch :123-124). norms: n doubles (device);
 * fro2 (device, may be NULL) receives ||A||_F^2. */
size_t apx_cycle_norms_workspace(int dtype, int64_t n);
int apx_cycle_norms(int dtype, const void* A, int64_t n, double* norms, double* fro2,
                    void* ws, size_t ws_bytes, void* stream);

/* -------------------------------------------------------------- cycle-truncated product ---- */
/* Restated (the reference ships only the primitives core.py:106-154):
 * A = sum_{j in J_A} Lambda_j C^j + dA, same for B with k_b cycles.
 * order 0: M = Ahat . Bhat;  order 1: M = Ahat . B + dA . Bhat  (first-order form of
 * svd.py:174-177 / circulant.py:193-198). force_sel_a/b (device, may be NULL) override the
 * selection (near-tie protocol, as test_circulant.py:108-110 does with spec.selected). */
size_t apx_cycle_first_order_workspace(int dtype, int64_t n, int k_a, int k_b, int order);
int apx_cycle_first_order(int dtype, const void* A, const void* B, int64_t n, int k_a, int k_b,
                          int order, const int32_t* force_sel_a, const int32_t* force_sel_b,
                          void* M, int32_t* sel_a, int32_t* sel_b, double* scalars,
                          void* ws, size_t ws_bytes, void* stream);

/* ---------------------------------------------------------------- mixed rSVD x cycles ---- */
/* Config C4 (restated): A by the randomized range finder of
 * randomized_partial_svd (svd.py:83-119) with l = k_svd sketch columns, q power iterations and
 * the caller's Gaussian sketch omega (n x l, device, drawn by the host exactly as svd.py:105-106
 * does, from default_rng([seed, 0]) -- svd.py:161); B by its k_cyc dominant cycles.
 * order 1: M = Ahat.B + dA.Bhat. fp32 with k_svd == 64, 1 <= k_cyc <= 128 and n a multiple of
 * 512 (up to ~13k) runs the residual plan M = Q.(Bm.B) + (A - Q.Bm).Bhat with dA and the kept
 * diagonals in scaled f16 (FHFMA gather, fp32 accumulation; csrc/mixed_f16.cu); otherwise, or with
 * flags bit 2, Q(Q^T A . dB) + A.Bhat with the gather over fp32 A. order 0: M = Ahat.Bhat.
 * flags bit 0: fp32 GEMMs as 3xTF32 on mma.sync; bit 1: force the mma.sync GEMMs (default: fp32
 * GEMMs on tcgen05 kind::tf32 when k_svd == 64); bit 2: the all-fp32 plan (no f16 residual).
 * APX_S_KEPT_A = sum sigma^2. */
size_t apx_mixed_first_order_workspace(int dtype, int64_t n, int k_svd, int k_cyc, int order);
int apx_mixed_first_order(int dtype, const void* A, const void* B, int64_t n, int k_svd, int k_cyc,
                          int order, int power_iterations, const void* omega,
                          const int32_t* force_sel_b, int flags, void* M, int32_t* sel_b,
                          double* scalars, void* ws, size_t ws_bytes, void* stream);

/* ---------------------------------------------------------------------- circulant path ---- */
/* circulant_first_order_multiply (circulant.py:164-218): A, B n x n fp64 or complex128 (dtype
 * APX_F64 / APX_C128), k components each, order 0 (Ahat B) / 1 (Ahat B + dA Bhat); M is n x n
 * complex128. Selections (ties -> lower index, ascending) land in sel_a / sel_b; force_sel_*
 * override them (near-tie protocol). scalars: FRO2_A/B, KEPT_A/B (= n sum mag^2), FRO2_M. */
size_t apx_circulant_first_order_workspace(int dtype, int64_t n, int k, int order);
int apx_circulant_first_order(int dtype, const void* A, const void* B, int64_t n, int k, int order,
                              const int32_t* force_sel_a, const int32_t* force_sel_b, void* M,
                              int32_t* sel_a, int32_t* sel_b, double* scalars, void* ws,
                              size_t ws_bytes, void* stream);

/* circulant_decompose (circulant.py:73-91): columns (n x n complex128, row k = first column of
 * R_k) and magnitudes (n doubles). */
size_t apx_circulant_decompose_workspace(int dtype, int64_t n);
int apx_circulant_decompose(int dtype, const void* A, int64_t n, void* columns, double* magnitudes,
                            void* ws, size_t ws_bytes, void* stream);

/* circulant_materialize (circulant.py:116-127) from the k selected first columns Ssel (k x n). */
size_t apx_circulant_materialize_workspace(int64_t n);
int apx_circulant_materialize(const void* Ssel, const int32_t* sel, int k, int64_t n, void* out,
                              void* ws, size_t ws_bytes, void* stream);

/* circulant_component (circulant.py:94-108): first column of R_kk by cycle averaging. Workspace:
 * apx_circulant_materialize_workspace(n). */
int apx_circulant_component(int dtype, const void* A, int64_t n, int kk, void* out, void* ws,
                            size_t ws_bytes, void* stream);

/* ----------------------------------------------------------- Fourier-sparsified path ---- */
/* fft_sparse_first_order_multiply (fsparse.py:168-240): A m x n, B n x p (APX_F64 / APX_C128),
 * At = A W*, Bt = W B, k largest |.| per row of At and per row (sparsify_cols = 0) or column
 * (1) of Bt, ties toward the lower index. order 0: SA dense(SB); order 1: SA Bt + (At-SA) SB.
 * M is m x p complex128. scalars: FRO2_A/B, RES2_A = ||At-SA||^2, RES2_B = ||Bt-SB||^2, FRO2_M.
 * sel_a (m x min(k,n)) / sel_b (n or p rows x kept) receive the kept columns (optional). */
size_t apx_sfft_first_order_workspace(int64_t m, int64_t n, int64_t p, int k);
int apx_sfft_first_order(int dtype, const void* A, const void* B, int64_t m, int64_t n, int64_t p,
                         int k, int order, int sparsify_cols, void* M, int32_t* sel_a,
                         int32_t* sel_b, double* scalars, void* ws, size_t ws_bytes, void* stream);

/* topk_sparsify (fsparse.py:121-139) on `rows` rows of complex128 M (rows x cols): budget[r]
 * (or k when budget is NULL) largest |M[r,:]|, ties to the lower column; sel is rows x k
 * (ascending, -1 padded), vals the kept entries. Workspace: rows*cols doubles. */
size_t apx_topk_rows_workspace(int64_t rows, int64_t cols);
int apx_topk_rows(const void* M, int64_t rows, int64_t cols, int k, const int32_t* budget,
                  int32_t* sel, void* vals, void* ws, size_t ws_bytes, void* stream);

/* sparse_dense_multiply (fsparse.py:142-165), S on the left: out (rows x p) = S X, S given as
 * rows x k (sel, vals complex128; -1 = unused slot), X complex128 with p columns, any k (the
 * entries are staged through shared memory in tiles of 256). */
int apx_sparse_rows_multiply(const int32_t* sel, const void* vals, int k, int64_t rows,
                             const void* X, int64_t p, void* out, void* stream);

/* fourier_row_decompose (fsparse.py:92-105): F = W(rows of A) / sqrt(n); weights[k] =
 * sqrt(n) ||F[:, k]||_2 (n fp64), directions = F[:, k] / ||F[:, k]|| (m x n complex128, zero
 * column where the weight vanishes). A is APX_F64 or APX_C128, m x n. */
size_t apx_fourier_row_decompose_workspace(int64_t m, int64_t n);
int apx_fourier_row_decompose(int dtype, const void* A, int64_t m, int64_t n, double* weights,
                              void* directions, void* ws, size_t ws_bytes, void* stream);

/* ------------------------------------------------------------------ core.py primitives ---- */
/* unitary_dft (core.py:82-97) on `batch` complex128 vectors (element i of vector b at
 * x[b*dist + i*stride]); inverse = 0 applies W, 1 applies W*. Lengths whose transform fits one
 * CTA's shared memory run there (a direct DFT for non-powers of two, up to ~7200); longer powers of
 * two (up to 2^18) use a four-step transform through global memory. */
size_t apx_unitary_dft_workspace(int64_t n, int64_t batch);
int apx_unitary_dft(const void* x, void* y, int64_t n, int64_t batch, int64_t stride, int64_t dist,
                    int inverse, void* ws, size_t ws_bytes, void* stream);

/* cycle_reorder (mode 0 right / 1 left) and cycle_reorder_inverse (2 right / 3 left),
 * core.py:106-137, elements of 8 (fp64) or 16 (complex128) bytes. */
int apx_cycle_layout(int elem_bytes, const void* in, int64_t n, int mode, void* out, void* stream);

/* apply_cycle_power (core.py:140-154): side 0 = C^k M (rows down), 1 = M C^k (columns left). */
int apx_apply_cycle_power(int elem_bytes, const void* in, int64_t rows, int64_t cols, int64_t k,
                          int side, void* out, void* stream);

/* frobenius (core.py:64-79) / relative_error (core.py:157-166) reductions: mode 0 writes
 * out[0..1] = <A,B>_F = sum conj(A) B (re, im); mode 1 writes (||B - A||_F^2, ||B||_F^2).
 * dtype_a / dtype_b: APX_F64 or APX_C128. */
size_t apx_pair_reduce_workspace(void);
int apx_pair_reduce(int dtype_a, const void* A, int dtype_b, const void* B, int64_t count, int mode,
                    double* out, void* ws, size_t ws_bytes, void* stream);

/* ------------------------------------------------------------------ randomized SVD path ---- */
/* randomized_partial_svd (svd.py:83-119), fp64: sketch width l (= k in the reference; l > k is
 * the oversampled variant of config C1), q power iterations, host-drawn Gaussian omega (n x l,
 * rng.standard_normal((n, l)) as svd.py:105-106). Outputs U (m x k), sigma (k, descending),
 * V (n x k); scalars: APX_S_FRO2_A = ||A||_F^2, APX_S_KEPT_A = sum sigma^2. */
size_t apx_rsvd_workspace(int dtype, int64_t m, int64_t n, int l);
int apx_rsvd(int dtype, const void* A, int64_t m, int64_t n, int l, int k, int power_iterations,
             const void* omega, void* U, double* sigma, void* V, double* scalars,
             void* ws, size_t ws_bytes, void* stream);

/* svd_first_order_multiply (svd.py:138-200), fp64, A m x n, B n x p, sketches l_a/l_b kept
 * k_a/k_b (k = l in the reference; k < l truncates an oversampled sketch), omega_a from
 * default_rng([seed,0]), omega_b from default_rng([seed,1]) (svd.py:161-162).
 * order 0: M = Ahat Bhat; order 1: M = Ahat B + dA Bhat. */
size_t apx_svd_first_order_workspace(int dtype, int64_t m, int64_t n, int64_t p, int l_a, int l_b);
int apx_svd_first_order(int dtype, const void* A, const void* B, int64_t m, int64_t n, int64_t p,
                        int l_a, int k_a, int l_b, int k_b, int power_iterations, int order,
                        const void* omega_a, const void* omega_b, void* M, double* scalars,
                        void* ws, size_t ws_bytes, void* stream);

/* qr_decompose (svd.py:63-69): thin QR of Y (m x k, m >= k), Householder with LAPACK's
 * reflector signs; R exactly upper triangular. */
size_t apx_qr_workspace(int dtype, int64_t m, int64_t k);
int apx_qr(int dtype, const void* Y, int64_t m, int64_t k, void* Q, void* R, void* ws,
           size_t ws_bytes, void* stream);

/* The C4 mixed product sharded by rows of A and M over ranks (the same math as
 * apx_mixed_first_order with kind::tf32 GEMMs, fp32, k_svd = 64). Rank g passes its row block A_rows
 * (m_rows x n), the whole B and the common sketch Omega (n x 64), and receives its rows of M. The call
 * is made four times, phase = 1..4, on the same workspace and stream; after each phase the caller
 * sums red_out over the ranks in place (NCCL all-reduce on `stream`) and passes it as the next
 * phase's red_in:
 *   phase 1: red_out = Gram(Y_g), 64 x 64 fp64          (red_in unused)
 *   phase 2: red_in = sum Gram; red_out = pass-2 Gram, 64 x 64 fp64
 *   phase 3: red_in = sum pass-2 Gram; red_out = Bm_g = Q_g^T A_g, 64 x n fp32
 *   phase 4: red_in = sum Bm; red_out = [||A_g||_F^2, ||M_g||_F^2, Cholesky breakdown (0/1)] fp64
 * flags bit 0: start M_g += Q_g W only after the whole gather (several shards driven on one device).
 * scalars (APX_NSCALARS) receive the rank-independent values (||B||^2, kept energies); the caller
 * fills FRO2_A / FRO2_M from the summed red_out of phase 4. Replaces nothing in the reference
 * (which has no multi-device path); the per-rank product is svd.py:174-177 restricted to rows. */
size_t apx_mixed_rows_workspace(int64_t n, int64_t m_rows, int k_svd, int k_cyc);
int apx_mixed_rows_phase(int phase, const float* A_rows, int64_t m_rows, const float* B, int64_t n, int k_svd,
                         int k_cyc, int order, int flags, const float* omega, float* M_rows, int32_t* sel_b,
                         const void* red_in, void* red_out, double* scalars, void* ws, size_t ws_bytes,
                         void* stream);

/* The cycle product (restated C2 / C5 path, apx_cycle_first_order) sharded by rows of A and M over
 * ranks. Rank g passes its row block A_rows = A[row0 : row0 + m_rows] and the whole
 * B, and receives M[row0 : row0 + m_rows]. Two calls on the same workspace and stream:
 *   phase 1: red_out = the energies of A's cycles over the rank's rows, n fp64 (red_in unused);
 *            the caller sums red_out over the ranks in place (NCCL all-reduce on `stream`);
 *   phase 2: red_in = the summed energies; selections, lambdas and the product rows; red_out[0] =
 *            ||M_g||_F^2, to be summed by the caller into scalars[APX_S_FRO2_M].
 * Every rank selects from the same summed energies, so sel_a agrees across ranks; B is replicated.
 * For the large-n left product (fp32 n > 5688, fp64 n > 2844) n must be a multiple of 512 and the
 * row block aligned to 128 (fp32) / 64 (fp64) rows. Replaces nothing in the reference (which has no
 * multi-device path); the per-rank product is the cycle product restricted to rows. */
size_t apx_cycle_rows_workspace(int dtype, int64_t n, int64_t m_rows, int k_a, int k_b, int order);
int apx_cycle_rows_phase(int phase, int dtype, const void* A_rows, int64_t m_rows, int64_t row0, const void* B,
                         int64_t n, int k_a, int k_b, int order, void* M_rows, int32_t* sel_a, int32_t* sel_b,
                         const double* red_in, double* red_out, double* scalars, void* ws, size_t ws_bytes,
                         void* stream);

/* The circulant product (circulant_first_order_multiply, circulant.py:164-218) sharded by rows of M
 * over ranks. A and B are replicated; rank g produces M[row0 : row0 + m_rows]
 * (complex128, m_rows x n) and computes term1 (circulant.py:136-147, column-local) for the columns
 * [col0, col0 + w_cols) and its decomposition share on the cycle blocks [blk0, blk1) of the grid
 * apx_circulant_rows_grid reports. Four calls on the same workspace and stream:
 *   phase 1: red_out = magnitude partials of A then B, 2 x parts x n fp64, zero outside this
 *            rank's blocks; the caller sums red_out over the ranks (an all-gather + rank-order sum);
 *   phase 2: red_in = the summed partials: magnitudes and selections (identical on every rank, and
 *            bitwise the single-device ones), kept energies; red_out = the selected spectrum rows
 *            of A then B from this rank's cycles, 2 x k x n complex128, zero elsewhere (summed by
 *            the caller = gathered);
 *   phase 3: red_in = the full selected spectra; T1 (n x w_cols complex128) = term1's columns; the
 *            caller moves T1[rows of rank h] to rank h (all-to-all) and assembles them into M_rows;
 *   phase 4: term2 (circulant.py:150-161) for the rank's rows added onto M_rows (order 1);
 *            red_out[0] = ||M_g||_F^2 (the caller sums it into scalars[APX_S_FRO2_M]).
 * row0 and col0 must be even; n within the fused shared-memory range (16 <= n <= 4096). Every
 * per-column and per-row computation is the single-device kernel, so the rows are bitwise the
 * single-device product's. Replaces nothing in the reference (which has no multi-device path). */
int apx_circulant_rows_grid(int64_t n, int64_t* parts, int64_t* cpc);
size_t apx_circulant_rows_workspace(int dtype, int64_t n, int k, int64_t m_rows, int64_t blk0, int64_t blk1);
int apx_circulant_rows_phase(int phase, int dtype, const void* A, const void* B, int64_t n, int k, int order,
                             int64_t row0, int64_t m_rows, int64_t col0, int64_t w_cols, int64_t blk0,
                             int64_t blk1, void* M_rows, void* T1, int32_t* sel_a, int32_t* sel_b,
                             const double* red_in, double* red_out, double* scalars, void* ws, size_t ws_bytes,
                             void* stream);

/* sketch_norm_estimate (errest.py:139-154): out[0] = ||A (B G)||_F^2 with A m x n, B n x p, G p x k
 * (all fp64 row-major; G drawn on the host with numpy exactly as the reference draws it). The
 * caller divides by k. Complex operands are passed as their real embeddings (see errest.py). */
size_t apx_sketch_norm_workspace(int64_t m, int64_t n, int64_t p, int k);
int apx_sketch_norm(const double* A, const double* B, int64_t m, int64_t n, int64_t p, const double* G, int k,
                    double* out, void* ws, size_t ws_bytes, void* stream);

/* Dense product C (+)= op(A) op(B) (matmul_naive core.py:48-61 / svd_reconstruct svd.py:133-135):
 * fp64 DMMA, fp32 3xTF32. trans_a: A stored K x M; trans_b: B stored N x K. */
size_t apx_gemm_workspace(int dtype, int64_t M, int64_t N, int64_t K, int trans_a, int trans_b);
int apx_gemm(int dtype, int trans_a, int trans_b, int64_t M, int64_t N, int64_t K, const void* A,
             int64_t lda, const void* B, int64_t ldb, void* C, int64_t ldc, int accumulate,
             void* ws, size_t ws_bytes, void* stream);

/* ------------------------------------------------------------------------- diagnostics ---- */
/* The tcgen05 TF32 GEMM used by the fp32 rSVD stages, exposed for kernel-level tests:
 * C (+)= opA . opB with layout bit 1 = A stored [k][m] (MN-major), bit 2 = B stored [k][n]
 * (MN-major; else [n][k]), bit 4 = store C transposed; bn in {64,128,256}; splits > 1 writes
 * `splits` partial slices of M*ldc floats. mask_j (optional) drops A-operand entries (m,k)
 * with (k - m) mod mod_n in mask_j (MN-major A only). */
int apx_debug_umma_gemm(int layout, int bn, const float* A, int64_t lda, const float* B, int64_t ldb,
                        float* C, int64_t ldc, int64_t M, int64_t N, int64_t K, int splits,
                        int accumulate, const int32_t* mask_j, int mask_k, int mod_n, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* APX_H_ */
