// tcgen05 (5th-gen tensor core) TF32 GEMMs for the fp32 randomized-SVD contractions.
//
//   C[M x N] (=|+=) opA[M x K] . opB[K x N],  fp32 in, fp32 accumulate in TMEM.
//   opA: K-major (A[m][k], k contiguous)  or MN-major (stored [k][m], m contiguous)
//   opB: K-major (stored [n][k])          or MN-major (stored [k][n], n contiguous)
//   Optional cycle mask on the MN-major A operand (dB^T: element (m,k) dropped when
//   (k - m) mod mod_n is a kept shift), optional transposed store C^T, optional split-K.
//
// One CTA = 128 x BN output tile; 4 warps. All threads stream operand tiles with cp.async into a
// STAGES-deep ring laid out in the UMMA "interleaved" (no-swizzle) canonical form: 8-row x 16-byte
// core matrices, so every 16-byte global chunk lands in one cp.async. Thread 0 issues
// tcgen05.mma.cta_group::1.kind::tf32 (M=128, N=BN, K=8) from shared-memory descriptors and
// commits each stage to an mbarrier that gates the reuse of that stage. The accumulator lives in
// TMEM (BN columns); the epilogue drains it with tcgen05.ld.32x32b.x32 (warp w owns lanes
// 32w..32w+31 = tile rows).
#include "common.cuh"
#include "kernels.cuh"

namespace apx {
namespace umma {

__device__ __forceinline__ uint32_t smem_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void cp16(uint32_t dst, const void* src, bool pred) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(src), "r"(pred ? 16 : 0));
}
__device__ __forceinline__ void cp4(uint32_t dst, const void* src, bool pred) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(dst), "l"(src), "r"(pred ? 4 : 0));
}
__device__ __forceinline__ void commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void wait_group() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_addr(bar)),
      "r"(phase));
}

// UMMA shared-memory descriptor (Blackwell version field = 1). layout: 0 = SWIZZLE_NONE
// ("interleave", used for K-major tiles), 1 = SWIZZLE_128B_BASE32B (MN-major TF32 tiles).
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo_bytes, uint32_t sbo_bytes,
                                              uint32_t layout = 0) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo_bytes >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo_bytes >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // version
  d |= (uint64_t)(layout & 7) << 61;
  // base_offset = 0, lbo_mode = 0
  return d;
}

// Instruction descriptor: D=F32, A=B=TF32, majors, N>>3, M>>4.
__host__ __device__ constexpr uint32_t make_idesc(int M, int N, bool a_mn, bool b_mn) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((a_mn ? 1u : 0u) << 15) | ((b_mn ? 1u : 0u) << 16) |
         ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_addr(bar))
               : "memory");
}
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float* v) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%"
      "19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

constexpr int BM = 128, BK = 32, kThreads = 128;
__device__ int g_desc_variant = 0;

template <int BN, int STAGES>
struct Cfg {
  static constexpr int kTileA = BM * BK * 4;  // bytes
  static constexpr int kTileB = BN * BK * 4;
  static constexpr int kStage = kTileA + kTileB;
  static constexpr size_t kSmem = (size_t)STAGES * kStage + 1024;  // + barriers / tmem slot
  static constexpr int kTmemCols = BN < 32 ? 32 : BN;
};

// Byte offset of element (row, k) inside a K-major operand tile with R rows (core matrices of
// 8 rows x 16 B; SBO = 128 B between 8-row groups, LBO = R*16 B between 16-byte K chunks).
__device__ __forceinline__ uint32_t off_kmajor(int row, int k, int R) {
  return (uint32_t)((row & 7) * 16 + (row >> 3) * 128 + (k >> 2) * (R * 16) + (k & 3) * 4);
}
// Byte offset of element (mn, k) inside an MN-major operand tile with R MN-entries. TF32
// MN-major operands must use the SWIZZLE_128B_BASE32B canonical layout (layout type 1): atoms of
// 4 k-rows x 128 B (32 mn), the 32-byte granules of row k XOR-swizzled by (k & 3). Atoms along MN
// are LBO = 512 B apart, 4-row k-groups SBO = (R/32)*512 B apart; tiles are 512 B aligned.
__device__ __forceinline__ uint32_t off_mnmajor(int mn, int k, int R) {
  const int e = mn & 31;
  return (uint32_t)((mn >> 5) * 512 + (k >> 2) * ((R / 32) * 512) + (k & 3) * 128 +
                    ((((e >> 3) ^ (k & 3)) & 3) << 5) + (e & 7) * 4);
}

template <int BN, int STAGES, bool A_MN, bool B_MN, bool TRANS_OUT>
__global__ void __launch_bounds__(kThreads, 1)
    umma_gemm_kernel(const float* __restrict__ A, int64_t lda, const float* __restrict__ B, int64_t ldb,
                     float* __restrict__ C, int64_t ldc, int64_t c_split_stride, int M, int N, int K, int k_per_split,
                     int accumulate, const int* __restrict__ mJ, int mk, int mod_n, int vec_ok) {
  using CF = Cfg<BN, STAGES>;
  extern __shared__ __align__(1024) unsigned char smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + (size_t)STAGES * CF::kStage);
  uint64_t* done_bar = bars + STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done_bar + 1);
  __shared__ int sJ[128];

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  const int kz = blockIdx.z;
  const int kbeg = kz * k_per_split, kend = min(K, kbeg + k_per_split);
  const int ktiles = (int)ceil_div(max(0, kend - kbeg), BK);

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_addr(tmem_slot)),
                 "r"(CF::kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) mbar_init(&bars[s], 1);
    mbar_init(done_bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int t = tid; t < mk && t < 128; t += kThreads) sJ[t] = mJ[t];
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t sbase = smem_addr(smem);

  auto load_tile = [&](int stage, int kt) {
    const int k0 = kbeg + kt * BK;
    const uint32_t a_s = sbase + stage * CF::kStage;
    const uint32_t b_s = a_s + CF::kTileA;
    if (vec_ok) {
      // A operand: BM x BK
      if (!A_MN) {  // A[m][k]: 16B chunks along k
        for (int c = tid; c < BM * (BK / 4); c += kThreads) {
          const int r = c / (BK / 4), kk = (c % (BK / 4)) * 4;
          const int gm = m0 + r, gk = k0 + kk;
          const bool ok = gm < M && gk < kend;
          cp16(a_s + off_kmajor(r, kk, BM), ok ? A + (size_t)gm * lda + gk : A, ok);
        }
      } else {  // stored [k][m]: 16B chunks along m
        for (int c = tid; c < BK * (BM / 4); c += kThreads) {
          const int kk = c / (BM / 4), r = (c % (BM / 4)) * 4;
          const int gm = m0 + r, gk = k0 + kk;
          const bool ok = gm < M && gk < kend;
          cp16(a_s + off_mnmajor(r, kk, BM), ok ? A + (size_t)gk * lda + gm : A, ok);
        }
      }
      if (!B_MN) {  // stored [n][k]
        for (int c = tid; c < BN * (BK / 4); c += kThreads) {
          const int r = c / (BK / 4), kk = (c % (BK / 4)) * 4;
          const int gn = n0 + r, gk = k0 + kk;
          const bool ok = gn < N && gk < kend;
          cp16(b_s + off_kmajor(r, kk, BN), ok ? B + (size_t)gn * ldb + gk : B, ok);
        }
      } else {  // stored [k][n]
        for (int c = tid; c < BK * (BN / 4); c += kThreads) {
          const int kk = c / (BN / 4), r = (c % (BN / 4)) * 4;
          const int gn = n0 + r, gk = k0 + kk;
          const bool ok = gn < N && gk < kend;
          cp16(b_s + off_mnmajor(r, kk, BN), ok ? B + (size_t)gk * ldb + gn : B, ok);
        }
      }
    } else {
      for (int c = tid; c < BM * BK; c += kThreads) {
        int r, kk;
        if (!A_MN) { r = c / BK; kk = c % BK; } else { kk = c / BM; r = c % BM; }
        const int gm = m0 + r, gk = k0 + kk;
        const bool ok = gm < M && gk < kend;
        const float* src = ok ? (A_MN ? A + (size_t)gk * lda + gm : A + (size_t)gm * lda + gk) : A;
        cp4(a_s + (A_MN ? off_mnmajor(r, kk, BM) : off_kmajor(r, kk, BM)), src, ok);
      }
      for (int c = tid; c < BN * BK; c += kThreads) {
        int r, kk;
        if (!B_MN) { r = c / BK; kk = c % BK; } else { kk = c / BN; r = c % BN; }
        const int gn = n0 + r, gk = k0 + kk;
        const bool ok = gn < N && gk < kend;
        const float* src = ok ? (B_MN ? B + (size_t)gk * ldb + gn : B + (size_t)gn * ldb + gk) : B;
        cp4(b_s + (B_MN ? off_mnmajor(r, kk, BN) : off_kmajor(r, kk, BN)), src, ok);
      }
    }
  };

  constexpr uint32_t idesc = make_idesc(BM, BN, A_MN, B_MN);
  // per-MMA (K=8) descriptor strides
  constexpr uint32_t a_lbo = A_MN ? 512 : BM * 16, a_sbo = A_MN ? (BM / 32) * 512 : 128;
  constexpr uint32_t b_lbo = B_MN ? 512 : BN * 16, b_sbo = B_MN ? (BN / 32) * 512 : 128;
  constexpr uint32_t a_lay = A_MN ? 1 : 0, b_lay = B_MN ? 1 : 0;
  constexpr uint32_t a_kstep = A_MN ? 2 * a_sbo : 2 * BM * 16;  // bytes per K=8
  constexpr uint32_t b_kstep = B_MN ? 2 * b_sbo : 2 * BN * 16;

#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < ktiles) load_tile(s, s);
    commit();
  }
  for (int kt = 0; kt < ktiles; ++kt) {
    const int stage = kt % STAGES;
    wait_group<STAGES - 2>();
    if (mJ != nullptr) {
      // mask kept cycles of the MN-major A operand (dB^T): element (m, k) <- dB[k][m]
      __syncthreads();
      const int k0 = kbeg + kt * BK;
      unsigned char* a_p = smem + stage * CF::kStage;
      for (int e = tid; e < BK * mk; e += kThreads) {
        const int kk = e / mk, t = e - kk * mk;
        int m = k0 + kk - sJ[t];
        if (m < 0) m += mod_n;
        if (m >= m0 && m < m0 + BM)
          *reinterpret_cast<float*>(a_p + off_mnmajor(m - m0, kk, BM)) = 0.f;
      }
    }
    fence_proxy_async();
    __syncthreads();
    if (tid == 0) {
      fence_after();
      const uint32_t a_s = sbase + stage * CF::kStage;
      const uint32_t b_s = a_s + CF::kTileA;
#pragma unroll
      for (int kk = 0; kk < BK / 8; ++kk) {
        const uint64_t da = make_desc(a_s + kk * a_kstep, a_lbo, a_sbo, a_lay);
        const uint64_t db = make_desc(b_s + kk * b_kstep, b_lbo, b_sbo, b_lay);
        mma_tf32(tmem, da, db, idesc, (kt > 0 || kk > 0) ? 1u : 0u);
      }
      mma_commit(&bars[stage]);
    }
    // refill the stage consumed in iteration kt-1 once its MMAs have drained it
    const int nk = kt + STAGES - 1;
    if (nk < ktiles) {
      if (kt >= 1) mbar_wait(&bars[(kt - 1) % STAGES], (uint32_t)(((kt - 1) / STAGES) & 1));
      load_tile(nk % STAGES, nk);
    }
    commit();
  }
  wait_group<0>();
  if (tid == 0) {
    if (ktiles > 0) mma_commit(done_bar);
    else asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(done_bar)));
  }
  mbar_wait(done_bar, 0);
  fence_after();

  // epilogue: warp w <-> tile rows 32w..32w+31 (TMEM lanes)
  const int row = m0 + warp * 32 + lane;
  float* Cz = C + (size_t)kz * c_split_stride;
#pragma unroll 1
  for (int j0 = 0; j0 < BN; j0 += 32) {
    float v[32];
    if (ktiles > 0) {
      tmem_ld32(tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)j0, v);
    } else {
#pragma unroll
      for (int i = 0; i < 32; ++i) v[i] = 0.f;
    }
    if (row < M) {
      if (!TRANS_OUT) {
        float* p = Cz + (size_t)row * ldc + n0 + j0;
        const bool full = (n0 + j0 + 32 <= N) && ((((uintptr_t)p) & 15) == 0);
        if (full) {
#pragma unroll
          for (int i = 0; i < 32; i += 4) {
            float4 o = make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
            if (accumulate) {
              const float4 q = *reinterpret_cast<const float4*>(p + i);
              o.x += q.x; o.y += q.y; o.z += q.z; o.w += q.w;
            }
            *reinterpret_cast<float4*>(p + i) = o;
          }
        } else {
          for (int i = 0; i < 32; ++i)
            if (n0 + j0 + i < N) p[i] = accumulate ? p[i] + v[i] : v[i];
        }
      } else {
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          const int col = n0 + j0 + i;
          if (col < N) {
            float* p = Cz + (size_t)col * ldc + row;
            *p = accumulate ? *p + v[i] : v[i];
          }
        }
      }
    }
  }
  fence_before();
  __syncthreads();
  if (warp == 0) {
    fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(CF::kTmemCols));
  }
}

}  // namespace umma

// C (ldc) = opA . opB ; see the header comment. Returns E_ARG for unsupported shapes.
template <int BN, bool A_MN, bool B_MN, bool TRANS_OUT>
static int umma_launch(const float* A, int64_t lda, const float* B, int64_t ldb, float* C, int64_t ldc,
                       int64_t c_split_stride, int M, int N, int K, int splits, int accumulate, const int* mJ, int mk,
                       int mod_n, cudaStream_t st) {
  constexpr int STAGES = 4;
  using CF = umma::Cfg<BN, STAGES>;
  const int kps = (int)(ceil_div(ceil_div(K, splits), umma::BK) * umma::BK);
  dim3 grid((unsigned)ceil_div(N, BN), (unsigned)ceil_div(M, umma::BM), (unsigned)splits);
  const int vec = ((lda % 4) == 0 && (ldb % 4) == 0 && ((uintptr_t)A % 16) == 0 && ((uintptr_t)B % 16) == 0) ? 1 : 0;
  auto fn = umma::umma_gemm_kernel<BN, STAGES, A_MN, B_MN, TRANS_OUT>;
  APX_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)CF::kSmem));
  fn<<<grid, umma::kThreads, CF::kSmem, st>>>(A, lda, B, ldb, C, ldc, c_split_stride, M, N, K, kps, accumulate, mJ,
                                              mk, mod_n, vec);
  APX_LAUNCH_CHECK();
  return OK;
}

// Dispatcher over the layouts the mixed product uses. layout bits: 1 = A MN-major,
// 2 = B MN-major, 4 = transposed store. bn in {64, 128, 256}.
int umma_set_variant(int v) {
  APX_CUDA(cudaMemcpyToSymbol(umma::g_desc_variant, &v, sizeof(int)));
  return OK;
}

int umma_gemm(int layout, int bn, const float* A, int64_t lda, const float* B, int64_t ldb, float* C, int64_t ldc,
              int64_t c_split_stride, int M, int N, int K, int splits, int accumulate, const int* mJ, int mk,
              int mod_n, cudaStream_t st) {
  APX_REQUIRE(mk <= 128, "umma_gemm: at most 128 masked shifts");
#define APX_UL(BNV, L)                                                                                        \
  if (bn == BNV && layout == L)                                                                             \
    return umma_launch<BNV, (L & 1) != 0, (L & 2) != 0, (L & 4) != 0>(A, lda, B, ldb, C, ldc, c_split_stride, M, N, \
                                                                      K, splits, accumulate, mJ, mk, mod_n, st);
  APX_UL(64, 0) APX_UL(64, 1) APX_UL(64, 2) APX_UL(64, 3) APX_UL(64, 4) APX_UL(64, 5) APX_UL(64, 6) APX_UL(64, 7)
  APX_UL(128, 0) APX_UL(128, 2) APX_UL(256, 0) APX_UL(256, 2)
#undef APX_UL
  set_error("umma_gemm: unsupported layout %d / BN %d", layout, bn);
  return E_ARG;
}

}  // namespace apx
