// Residual plan of the mixed rSVD x cycles product (config C4, fp32, order 1).
//
// The order-1 product is  M = Ahat.B + dA.Bhat  (Ahat = Q Q^T A, dA = A - Ahat, Bhat = the k_cyc
// kept cycles of B; the reference's svd_first_order_multiply structure, svd.py:174-177). With
// Bm = Q^T A (whatever the TF32 GEMM returns) it is evaluated as
//
//     M = Q . (Bm . B)  +  (A - Q . Bm) . Bhat                                   (1)
//
// which equals A.Bhat + Q Bm dB for ANY Bm -- so Bm's own rounding never enters M beyond the tiny
// Q Bm dB term -- provided both sides use the same Bm and each product is formed accurately:
//   * Q . (Bm . B): Bm . B = [TF32 GEMM Bm.B] - [TF32-truncated gather Bm.Bhat] + [fp32 gather
//     Bm.Bhat]; the first two cancel exactly on the kept cycles (the round-1 W trick), so the
//     result has TF32 error only relative to Bm.dB. The outer product by Q (TF32-exact from the QR)
//     runs on the tensor core as a K = 2l GEMM [Q | Q] . [hi(W); lo(W)] (hi/lo: TF32 split), i.e.
//     at fp32 accuracy.
//   * dA = A - Q . Bm: Bm is rounded to TF32 once it is formed (Bm := tf32(Bm) -- (1) holds for
//     any Bm), so with Q TF32-exact as well every tensor-core product is exact and the K = l GEMM
//     is fp32-accurate; the subtraction and the f16 store are fused into its epilogue
//     (gemm_tma_kernel FIX 4).
//   * dA . Bhat: dA carries ~1.8% of ||M|| at C4 (residual energy 3.4e-4 of ||A||^2), so it is
//     stored as scaled f16 (2^(15-e_A) dA, e_A from ||A||_F: no entry can overflow) and the
//     kept-cycle diagonals as scaled f16 too (2^(15-e_B) lambda', e_B from ||B||_F); the gather
//     multiplies them with FHFMA (fma.rn.f32.f16: f16 x f16 products, fp32 accumulation) and
//     rescales by 2^(e_A + e_B - 30) once per output. Each shared-memory operand is now 2 bytes
//     instead of 4, which halves the gather's shared-memory bytes per FMA -- the gather's
//     limiter. f16 rounding (2^-11 relative) on a term of 1.8% of M adds
//     ~4e-6 relative error (north_star allows reduced-precision operands where the fp32 1e-4
//     tolerance allows; measured parity in tests/test_gpu_mixed.py and bench.py).
//
// Kernels here: TF32 rounding and the hi/lo split, [Q | Q], the f16 lambda' table, the f16 gather.
#include <cuda_fp16.h>

#include "common.cuh"
#include "kernels.cuh"

namespace apx {

namespace {

__device__ __forceinline__ float tf32_rn(float x) {
  return __uint_as_float((__float_as_uint(x) + 0x1000u) & 0xffffe000u);
}

// X2[0:rows] = tf32(X), X2[rows:2 rows] = tf32(X - tf32(X)) (X - tf32(X) is exact in fp32)
__global__ void split_tf32_kernel(const float* __restrict__ X, size_t count, float* __restrict__ X2) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < count; i += (size_t)gridDim.x * blockDim.x) {
    const float x = X[i];
    const float hi = tf32_rn(x);
    X2[i] = hi;
    X2[count + i] = tf32_rn(x - hi);
  }
}

// X = tf32(X) in place (round to nearest, ties away)
__global__ void round_tf32_kernel(float* __restrict__ X, size_t count) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < count; i += (size_t)gridDim.x * blockDim.x)
    X[i] = tf32_rn(X[i]);
}

// Residual plan, after the Bm = Q^T A GEMM (one launch instead of seven): Bm = sum of the split-K
// partials (fixed order, fp64 -- split_reduce_kernel's arithmetic), ||Bm||^2 from Bm as formed,
// Bm := tf32(Bm), Q2 = [Q | Q]; per-CTA ||Bm||^2 partials, and the last CTA to finish (atomic
// counter, reset for the next product) sums them and the ||A||^2 partials of the GEMM in a fixed
// order into kept_out and fro2_out.
constexpr int kFinThreads = 256;
constexpr double kResidF16MaxEnergy = 0.01;  // residual energy fraction up to which dA goes f16
__global__ void __launch_bounds__(kFinThreads)
    bm_finalize_kernel(const float* __restrict__ part, int splits, int l, int n, float* __restrict__ Bm,
                       const float* __restrict__ Q, float* __restrict__ Q2, double* __restrict__ bsq_part,
                       const double* __restrict__ asq_part, int asq_parts, unsigned* __restrict__ counter,
                       double* __restrict__ kept_out, double* __restrict__ fro2_out, int* __restrict__ use_f16,
                       int f16_mode) {
  pdl_wait();
  __shared__ double red[32];
  __shared__ bool last;
  const size_t count = (size_t)l * n;
  double sq = 0.0;
  for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < count; e += (size_t)gridDim.x * blockDim.x) {
    double v = 0.0;
    for (int z = 0; z < splits; ++z) v += (double)part[(size_t)z * count + e];
    const float b = (float)v;
    sq = fma((double)b, (double)b, sq);
    Bm[e] = tf32_rn(b);
    const size_t r = e / l, c = e - r * l;  // Q is n x l: same element count
    const float q = Q[e];
    Q2[r * 2 * l + c] = q;
    Q2[r * 2 * l + l + c] = q;
  }
  sq = block_sum(sq, red);
  if (threadIdx.x == 0) {
    bsq_part[blockIdx.x] = sq;
    __threadfence();
    last = atomicAdd(counter, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  double k = 0.0, a = 0.0;
  for (int i = threadIdx.x; i < (int)gridDim.x; i += blockDim.x) k += bsq_part[i];
  for (int i = threadIdx.x; i < asq_parts; i += blockDim.x) a += asq_part[i];
  k = block_sum(k, red);
  __syncthreads();
  a = block_sum(a, red);
  if (threadIdx.x == 0) {
    *kept_out = k;
    *fro2_out = a;
    *counter = 0u;
    // the f16 residual is accurate enough only while dA stays a small part of the product: with
    // f16 rounding (2^-11) on a term carrying a fraction f of ||M|| the error is ~4e-4 f, so the
    // plan keeps it for a residual energy ||A||^2 - ||Bm||^2 <= 1% of ||A||^2 (f ~ 0.1) and falls
    // back to the fp32 gather over dA otherwise (f16_mode 1 / 2 force either, for tests)
    if (use_f16 != nullptr)
      *use_f16 = f16_mode == 1 ? 1 : f16_mode == 2 ? 0 : ((a - k) <= kResidF16MaxEnergy * a ? 1 : 0);
  }
}

// Q2 = [Q | Q] (rows x 2l)
__global__ void dup_cols_kernel(const float* __restrict__ Q, int rows, int l, float* __restrict__ Q2) {
  const size_t count = (size_t)rows * l;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < count; i += (size_t)gridDim.x * blockDim.x) {
    const size_t r = i / l, c = i - r * l;
    const float v = Q[i];
    Q2[r * 2 * l + c] = v;
    Q2[r * 2 * l + l + c] = v;
  }
}

constexpr int kHR = 8;  // rows per block: 8 halves = one 16-byte vector per column
constexpr int kHU = 4;  // shifts per lambda batch

// f16 lambda' table in the gather's thread order: the CPT columns g * CPT NT + q * NT + tid (q <
// CPT) of shift t are CPT/2 packed f16x2 words, scaled by 2^(15 - e_B), at word
//   ((g * kp / kHU + t / kHU) * NT + tid) * kHU * CPT/2 + (t % kHU) * CPT/2,
// so one thread's batch of kHU shifts is ONE contiguous 16- or 32-byte run (a warp's batch: 512 or
// 1024 contiguous bytes), fetched with one or two vector loads from one running pointer.
__global__ void lam_f16_kernel(const float* __restrict__ lam, int kp, int n, int nt, int cpt,
                               const double* __restrict__ fro2_b, uint32_t* __restrict__ out) {
  const float s = ldexpf(1.f, 15 - f16_scale_exp(*fro2_b));
  const int per_row = n / cpt, lw = cpt / 2;
  const size_t count = (size_t)kp * per_row;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < count; i += (size_t)gridDim.x * blockDim.x) {
    const int t = (int)(i / per_row), e = (int)(i - (size_t)t * per_row);
    const int g = e / nt, tid = e - g * nt;
    const float* row = lam + (size_t)t * n + (size_t)g * cpt * nt + tid;
    const size_t o = (((size_t)g * (kp / kHU) + t / kHU) * nt + tid) * kHU * lw + (size_t)(t % kHU) * lw;
    for (int w = 0; w < lw; ++w) out[o + w] = pack_half2(s * row[(2 * w) * nt], s * row[(2 * w + 1) * nt]);
  }
}

__device__ __forceinline__ float fhfma(unsigned short a, unsigned short b, float c) {
  float d;
  asm("fma.rn.f32.f16 %0, %1, %2, %3;" : "=f"(d) : "h"(a), "h"(b), "f"(c));
  return d;
}
__device__ __forceinline__ unsigned short lo16(uint32_t v) { return (unsigned short)(v & 0xffffu); }
__device__ __forceinline__ unsigned short hi16(uint32_t v) { return (unsigned short)(v >> 16); }

// one thread's lambda' batch: kHU shifts x W words, contiguous (lam_f16_kernel's layout)
template <int W>
__device__ __forceinline__ void ldg_nc_batch(const uint32_t* p, uint32_t (&v)[kHU][W]) {
  static_assert(kHU == 4 && (W == 1 || W == 2), "batch = 16 or 32 bytes");
  asm volatile("ld.global.nc.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v[0][0]), "=r"(v[W == 1 ? 1 : 0][W - 1]), "=r"(v[W == 1 ? 2 : 1][0]), "=r"(v[W == 1 ? 3 : 1][W - 1])
               : "l"(p));
  if constexpr (W == 2)
    asm volatile("ld.global.nc.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(v[2][0]), "=r"(v[2][1]), "=r"(v[3][0]), "=r"(v[3][1])
                 : "l"(p + 4));
}

__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(b)), "r"(c));
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t phase) {
  asm volatile(
      "{\n.reg .pred p;\nW_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra W_%=;\n}\n" ::"r"((uint32_t)__cvta_generic_to_shared(b)),
      "r"(phase)
      : "memory");
}


// M[r0 + i, c] = 2^(e_A + e_B - 30) sum_t dAh[r0 + i, (c + J_t) mod n] * lamh_t[c], i < 8.
// Xh: ceil(m_rows / 8) blocks of n uint4 (block b, column m = rows 8b..8b+7 of column m as f16);
// one block is one contiguous 16 n-byte run, staged into shared memory by ONE bulk async copy.
// Thread tid owns columns g * CPT NT + q * NT + tid of each column group g; per shift it loads
// one CPT-half vector of lambda' (its CPT columns) and, per column, one 16-byte shared vector (8
// rows) feeding 8 FHFMAs: per warp CPT x 4 shared wavefronts + CPT/2 lambda' wavefronts per
// 256 CPT FMAs (the fp32 gather: 7 per 192). Persistent CTAs pull row blocks from `ticket`,
// prefetch the next block into L2 during the last column group, and publish each finished
// block in `ready` (consumed by M += Q.W, see run_mixed_f32_resid).
// RMW: M += (instead of =) the gather -- each column group's old M values are loaded at the
// group's start (their latency hides under the shift loop) -- and the per-block ||M||^2 partials
// of the final values go to msq_partial[blk] (fixed-order block sum).
// PAD: the first (CPT - 1) NT columns of the block are staged a second time behind its end (a
// second bulk copy on the same barrier), so a thread's CPT columns for one shift are ONE wrapped base
// plus the constant offsets q NT -- one index wrap per shift instead of one per column, and the
// loads take their offsets as immediates.
template <int NT, int CPT, bool RMW, bool PAD>
__global__ void __launch_bounds__(NT, 1)
    cycle_gather_f16_kernel(const uint4* __restrict__ Xh, const uint32_t* __restrict__ lamh,
                            const int* __restrict__ J, int k, int kp, int n, int m_rows, float* __restrict__ M,
                            const double* __restrict__ fro2_a, const double* __restrict__ fro2_b,
                            int* __restrict__ ticket, int* __restrict__ ready, double* __restrict__ msq_partial,
                            const int* __restrict__ gate) {
  if (gate != nullptr && *gate == 0) return;  // the plan fell back to the fp32 gather (bm_finalize)
  constexpr int LW = CPT / 2;  // lambda' words per thread per shift
  extern __shared__ __align__(16) unsigned char smem_raw[];
  constexpr int PADC = PAD ? (CPT - 1) * NT : 0;  // replicated columns behind the block
  uint4* Xs = reinterpret_cast<uint4*>(smem_raw);
  int* sJ = reinterpret_cast<int*>(Xs + n + PADC);
  __shared__ __align__(8) uint64_t bar;
  __shared__ int s_blk, s_nxt;
  __shared__ double red[32];
  const int tid = threadIdx.x;
  const int nblk = (int)ceil_div(m_rows, kHR);
  pdl_wait();  // programmatic dependent launch: the previous kernel's outputs (dA) are read below
  const float inv = ldexpf(1.f, f16_scale_exp(*fro2_a) + f16_scale_exp(*fro2_b) - 30);
  for (int t = tid; t < kp; t += NT) sJ[t] = t < k ? J[t] : 0;  // padded shifts: zero lambda' rows
  if (tid == 0) {
    mbar_init(&bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    s_nxt = -1;
  }
  const uint32_t bytes = (uint32_t)n * 16u, pbytes = (uint32_t)PADC * 16u;
  const int groups = n / (CPT * NT);
  for (int it = 0;; ++it) {
    if (tid == 0) {
      s_blk = (s_nxt < 0) ? atomicAdd(ticket, 1) : s_nxt;
      s_nxt = -1;
      if (s_blk < nblk) {
        // the previous block's generic-proxy reads of Xs are ordered before this async write by
        // the barrier that ended it; the proxy fence makes that ordering hold across proxies
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
                         (uint32_t)__cvta_generic_to_shared(&bar)),
                     "r"(bytes + pbytes)
                     : "memory");
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                (uint32_t)__cvta_generic_to_shared(Xs)),
            "l"(Xh + (size_t)s_blk * n), "r"(bytes), "r"((uint32_t)__cvta_generic_to_shared(&bar))
            : "memory");
        if constexpr (PAD)
          asm volatile(
              "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                  (uint32_t)__cvta_generic_to_shared(Xs + n)),
              "l"(Xh + (size_t)s_blk * n), "r"(pbytes), "r"((uint32_t)__cvta_generic_to_shared(&bar))
              : "memory");
      }
    }
    __syncthreads();
    const int blk = s_blk;
    if (blk >= nblk) break;
    const int r0 = blk * kHR;
    const int rows = min(kHR, m_rows - r0);
    mbar_wait(&bar, (uint32_t)(it & 1));
    double msq = 0.0;
    for (int g = 0; g < groups; ++g) {
      if (g == groups - 1 && tid == 0) {
        const int nx = atomicAdd(ticket, 1);
        s_nxt = nx;
        if (nx < nblk)
          asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(Xh + (size_t)nx * n), "r"(bytes) : "memory");
      }
      const int cbase = g * CPT * NT + tid;
      float mold[RMW ? CPT : 1][RMW ? kHR : 1];
      if constexpr (RMW) {
#pragma unroll
        for (int r = 0; r < kHR; ++r)
#pragma unroll
          for (int q = 0; q < CPT; ++q)
            mold[q][r] = r < rows ? __ldcg(M + (size_t)(r0 + r) * n + cbase + q * NT) : 0.f;
      }
      // this thread's lambda' batches for group g: one running pointer, NT kHU LW words per batch
      const uint32_t* lp = lamh + ((size_t)g * (kp / kHU) * NT + tid) * (kHU * LW);
      constexpr int kLStep = NT * kHU * LW;
      float acc[CPT][kHR];
#pragma unroll
      for (int q = 0; q < CPT; ++q)
#pragma unroll
        for (int r = 0; r < kHR; ++r) acc[q][r] = 0.f;
      // batch b + 1's lambda' loads are in flight while batch b is consumed
      // (the batch's shifts ride along: their shared loads head each column's index chain)
      uint32_t lvA[kHU][LW], lvB[kHU][LW];
      int jA[kHU], jB[kHU];
      ldg_nc_batch<LW>(lp, lvA);
#pragma unroll
      for (int u = 0; u < kHU; ++u) jA[u] = sJ[u];
      auto compute = [&](const int (&jv)[kHU], const uint32_t (&lv)[kHU][LW]) {
#pragma unroll
        for (int u = 0; u < kHU; ++u) {
          const int jt = jv[u];
          unsigned m0 = (unsigned)(cbase + jt);
          if constexpr (PAD) m0 = min(m0, m0 - (unsigned)n);
#pragma unroll
          for (int q = 0; q < CPT; ++q) {
            unsigned m;
            if constexpr (PAD) {
              m = m0 + q * NT;
              APX_DCHECK(m < (unsigned)(n + PADC));
            } else {
              m = m0 + q * NT;
              m = min(m, m - (unsigned)n);
              APX_DCHECK(m < (unsigned)n);
            }
            const uint4 x = Xs[m];
            const unsigned short l = (q & 1) ? hi16(lv[u][q >> 1]) : lo16(lv[u][q >> 1]);
            acc[q][0] = fhfma(lo16(x.x), l, acc[q][0]);
            acc[q][1] = fhfma(hi16(x.x), l, acc[q][1]);
            acc[q][2] = fhfma(lo16(x.y), l, acc[q][2]);
            acc[q][3] = fhfma(hi16(x.y), l, acc[q][3]);
            acc[q][4] = fhfma(lo16(x.z), l, acc[q][4]);
            acc[q][5] = fhfma(hi16(x.z), l, acc[q][5]);
            acc[q][6] = fhfma(lo16(x.w), l, acc[q][6]);
            acc[q][7] = fhfma(hi16(x.w), l, acc[q][7]);
          }
        }
      };
      for (int t0 = 0; t0 < kp; t0 += 2 * kHU) {
        if (t0 + kHU < kp) {
          lp += kLStep;
          ldg_nc_batch<LW>(lp, lvB);
#pragma unroll
          for (int u = 0; u < kHU; ++u) jB[u] = sJ[t0 + kHU + u];
        }
        compute(jA, lvA);
        if (t0 + kHU >= kp) break;
        if (t0 + 2 * kHU < kp) {
          lp += kLStep;
          ldg_nc_batch<LW>(lp, lvA);
#pragma unroll
          for (int u = 0; u < kHU; ++u) jA[u] = sJ[t0 + 2 * kHU + u];
        }
        compute(jB, lvB);
      }
#pragma unroll
      for (int r = 0; r < kHR; ++r)
        if (r < rows) {
          float* mp = M + (size_t)(r0 + r) * n + cbase;
#pragma unroll
          for (int q = 0; q < CPT; ++q) {
            if constexpr (RMW) {
              const float v = fmaf(acc[q][r], inv, mold[q][r]);
              mp[q * NT] = v;
              msq = fma((double)v, (double)v, msq);
            } else {
              mp[q * NT] = acc[q][r] * inv;
            }
          }
        }
    }
    if constexpr (RMW) {
      msq = block_sum(msq, red);
      if (tid == 0) msq_partial[blk] = msq;
    }
    __syncthreads();  // every M store of the block, and every read of Xs, precede what follows
    if (tid == 0 && ready) {
      __threadfence();
      atomicExch(ready + blk, 1);
    }
  }
}

// gather shape (threads per CTA = column stride, columns per thread): APX_F16_CFG="NTxCPT"
// overrides (tuning); the default is the largest NT of the preferred CPT that tiles n
struct F16Cfg {
  int nt, cpt;
};
F16Cfg f16_cfg(int n) {
  static const F16Cfg env = [] {
    F16Cfg c{0, 0};
    if (const char* e = getenv("APX_F16_CFG")) sscanf(e, "%dx%d", &c.nt, &c.cpt);
    return c;
  }();
  if (env.nt > 0 && (env.cpt == 2 || env.cpt == 4) && n % (env.nt * env.cpt) == 0) return env;
  // four columns per thread at 512 threads (measured: 512x4 0.457 ms, 1024x2 0.461, 512x2 0.497 at
  // C4 on 132 SMs); the read-modify-write variant keeps its old values in registers (128 at 512x4)
  for (int nt : {512, 256, 128})
    if (n % (4 * nt) == 0) return {nt, 4};
  return {0, 0};
}

}  // namespace

int launch_split_tf32(const float* X, size_t count, float* X2, cudaStream_t st) {
  const unsigned blocks = (unsigned)std::min<size_t>(ceil_div(count, (size_t)256), (size_t)kNumSMs * 8);
  split_tf32_kernel<<<blocks, 256, 0, st>>>(X, count, X2);
  APX_LAUNCH_CHECK();
  return OK;
}

int launch_bm_finalize(const float* part, int splits, int l, int n, float* Bm, const float* Q, float* Q2,
                       double* bsq_part, const double* asq_part, int asq_parts, unsigned* counter, double* kept_out,
                       double* fro2_out, int* use_f16, int f16_mode, cudaStream_t st) {
  const unsigned blocks = (unsigned)std::min<size_t>(ceil_div((size_t)l * n, (size_t)kFinThreads), (size_t)kNumSMs * 4);
  APX_CUDA(launch_pdl(bm_finalize_kernel, dim3(blocks), dim3(kFinThreads), 0, st, part, splits, l, n, Bm, Q, Q2,
                      bsq_part, asq_part, asq_parts, counter, kept_out, fro2_out, use_f16, f16_mode));
  APX_LAUNCH_CHECK();
  return OK;
}

// fallback of the residual plan: once the fp32 gather (which publishes no flags) is done, mark every
// row block ready for M += Q.W; a no-op when the f16 gather ran (it published them itself)
__global__ void fallback_flags_kernel(const int* __restrict__ use_f16, int* __restrict__ ready, int blocks) {
  if (*use_f16 != 0) return;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < blocks; i += gridDim.x * blockDim.x) ready[i] = 1;
}

int launch_fallback_flags(const int* use_f16, int* ready, int blocks, cudaStream_t st) {
  fallback_flags_kernel<<<(unsigned)std::min(64, (int)ceil_div(blocks, 256)), 256, 0, st>>>(use_f16, ready, blocks);
  APX_LAUNCH_CHECK();
  return OK;
}

int launch_round_tf32(float* X, size_t count, cudaStream_t st) {
  const unsigned blocks = (unsigned)std::min<size_t>(ceil_div(count, (size_t)256), (size_t)kNumSMs * 8);
  round_tf32_kernel<<<blocks, 256, 0, st>>>(X, count);
  APX_LAUNCH_CHECK();
  return OK;
}

int launch_dup_cols(const float* Q, int rows, int l, float* Q2, cudaStream_t st) {
  const unsigned blocks = (unsigned)std::min<size_t>(ceil_div((size_t)rows * l, (size_t)256), (size_t)kNumSMs * 8);
  dup_cols_kernel<<<blocks, 256, 0, st>>>(Q, rows, l, Q2);
  APX_LAUNCH_CHECK();
  return OK;
}

// threads per CTA (= column stride) of the f16 gather for n, or 0 when n does not fit its layout
int gather_f16_threads(int n) { return f16_cfg(n).nt; }

// the padded layout when it fits (APX_F16_PAD=0 disables it)
static bool f16_pad(int n, int kp) {
  static const bool off = getenv("APX_F16_PAD") != nullptr && atoi(getenv("APX_F16_PAD")) == 0;
  const F16Cfg c = f16_cfg(n);
  return !off && c.nt > 0 && (size_t)(n + (c.cpt - 1) * c.nt) * 16 + (size_t)kp * sizeof(int) <= 220 * 1024;
}

size_t gather_f16_smem(int n, int kp) {
  const F16Cfg c = f16_cfg(n);
  return (size_t)(n + (f16_pad(n, kp) ? (c.cpt - 1) * c.nt : 0)) * 16 + (size_t)kp * sizeof(int);
}

int launch_lam_f16(const float* lam, int kp, int n, const double* fro2_b, uint16_t* out, cudaStream_t st) {
  const F16Cfg c = f16_cfg(n);
  APX_REQUIRE(c.nt > 0, "f16 gather: n=%d must be a multiple of 512", n);
  const size_t count = (size_t)kp * (n / c.cpt);
  const unsigned blocks = (unsigned)std::min<size_t>(ceil_div(count, (size_t)256), (size_t)kNumSMs * 8);
  lam_f16_kernel<<<blocks, 256, 0, st>>>(lam, kp, n, c.nt, c.cpt, fro2_b, reinterpret_cast<uint32_t*>(out));
  APX_LAUNCH_CHECK();
  return OK;
}

int launch_gather_f16(const uint16_t* Xh, const uint16_t* lamh, const int* J, int k, int kp, int n, int m_rows, float* M,
                      const double* fro2_a, const double* fro2_b, int* ticket, int* ready, int ctas, cudaStream_t st,
                      double* msq_partial, const int* gate) {
  const F16Cfg c = f16_cfg(n);
  APX_REQUIRE(c.nt > 0, "f16 gather: n=%d must be a multiple of 512", n);
  APX_REQUIRE(kp % (2 * kHU) == 0 && kp > 0, "f16 gather: shift count %d must be a positive multiple of 8", kp);
  const size_t smem = gather_f16_smem(n, kp);
  APX_REQUIRE(smem <= 220 * 1024, "f16 gather: n=%d needs %zu bytes of shared memory", n, smem);
  const int nblk = (int)ceil_div(m_rows, kHR);
  const unsigned grid = (unsigned)std::max(1, std::min(nblk, ctas));
  APX_CUDA(cudaMemsetAsync(ticket, 0, sizeof(int), st));
  auto go = [&](auto kern) -> int {
    APX_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    APX_CUDA(launch_pdl(kern, dim3(grid), dim3(c.nt), smem, st, reinterpret_cast<const uint4*>(Xh),
                        reinterpret_cast<const uint32_t*>(lamh), J, k, kp, n, m_rows, M, fro2_a, fro2_b, ticket, ready,
                        msq_partial, gate));
    APX_LAUNCH_CHECK();
    return OK;
  };
  const bool pad = f16_pad(n, kp);
#define APX_F16(NTV, CPTV)                                                                                   \
  if (c.nt == NTV && c.cpt == CPTV) {                                                                         \
    if (pad)                                                                                                  \
      return msq_partial ? go(cycle_gather_f16_kernel<NTV, CPTV, true, true>)                                 \
                         : go(cycle_gather_f16_kernel<NTV, CPTV, false, true>);                               \
    return msq_partial ? go(cycle_gather_f16_kernel<NTV, CPTV, true, false>)                                  \
                       : go(cycle_gather_f16_kernel<NTV, CPTV, false, false>);                                \
  }
  APX_F16(512, 4) APX_F16(256, 4) APX_F16(128, 4) APX_F16(1024, 2) APX_F16(512, 2) APX_F16(256, 2)
#undef APX_F16
  set_error("f16 gather: unsupported shape %dx%d", c.nt, c.cpt);
  return E_ARG;
}

}  // namespace apx
