// Warp-specialized tcgen05 TF32 GEMM with TMA operand loads (the fp32 rSVD contractions).
//
//   C[M x N] (=|+=) opA[M x K] . opB[K x N]   (same operand conventions as umma.cu)
//
// 192 threads per CTA, one 128 x BN output tile (split-K slice):
//   warp 0      TMA producer: one elected lane streams A/B K-tiles (BK = 32) into a STAGES-deep
//               shared-memory ring, arming each stage's `full` mbarrier with the byte count.
//   warp 1      TMEM allocator + MMA issuer: one lane issues tcgen05.mma.cta_group::1.kind::tf32
//               (M=128, N=BN, K=8) x4 per stage and commits to the stage's `empty` mbarrier.
//   warps 2..5  (FIX 1) zero the kept-cycle entries of each landed A tile (dB^T), or (FIX 2) round
//               the landed A tile to TF32 nearest (the tensor core itself truncates: a
//               systematic -2^-11.5 relative bias per operand, which a sum of squares of the
//               result -- ||Q^T A||^2 for the residual energy -- accumulates), then
//               epilogue: tcgen05.ld.32x32b.x32 from TMEM (warp%4 selects the lane quarter).
// Layouts: K-major tiles use TMA SWIZZLE_128B <-> UMMA SWIZZLE_128B (rows of 128 B, 8-row atoms,
// SBO = 1024 B, K advanced by 32 B per MMA); MN-major tiles (TF32 requires it) use TMA
// SWIZZLE_128B_ATOM_32B <-> UMMA SWIZZLE_128B_BASE32B (boxes of 32 mn x 32 k = 4 KB; 4-row atoms,
// SBO = 512 B between k-groups, LBO = 4 KB between 32-mn boxes).
#include <cuda.h>

#include <mutex>

#include "common.cuh"
#include "kernels.cuh"

namespace apx {
namespace tma {

constexpr int BM = 128, BK = 32, kThreads = 192;

__device__ __forceinline__ uint32_t saddr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(saddr(b)), "r"(c));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(saddr(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(saddr(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t phase) {
  asm volatile(
      "{\n.reg .pred p;\nW_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra W_%=;\n}\n" ::"r"(saddr(b)),
      "r"(phase)
      : "memory");
}
__device__ __forceinline__ int ld_relaxed_gpu(const int* p) {
  int v;
  asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::
          "r"(dst),
      "l"(map), "r"(c0), "r"(c1), "r"(saddr(bar))
      : "memory");
}
__device__ __forceinline__ uint64_t desc(uint32_t addr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46) | ((uint64_t)(layout & 7) << 61);
}
__host__ __device__ constexpr uint32_t idesc(int M, int N, bool a_mn, bool b_mn) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((a_mn ? 1u : 0u) << 15) | ((b_mn ? 1u : 0u) << 16) |
         ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void mma(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
      "l"(a), "l"(b), "r"(id), "r"(acc));
}
__device__ __forceinline__ void commit(uint64_t* b) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(saddr(b))
               : "memory");
}
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }

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

// byte offset of element (mn, k) in an MN-major tile built from 32x32 TMA boxes (ATOM_32B swizzle)
__device__ __forceinline__ uint32_t mn_off(int mn, int k) {
  const int e = mn & 31;
  return (uint32_t)((mn >> 5) * 4096 + k * 128 + ((((e >> 3) ^ (k & 3)) & 3) << 5) + (e & 7) * 4);
}

template <int BN, int STAGES>
struct Cfg {
  static constexpr int kTileA = BM * BK * 4;
  static constexpr int kTileB = BN * BK * 4;
  static constexpr int kStage = kTileA + kTileB;
  static constexpr size_t kSmem = (size_t)STAGES * kStage + 1024 /*align slack*/ + 256 /*barriers*/;
  static constexpr int kTmemCols = BN;
};

template <int BN, int STAGES, bool A_MN, bool B_MN, bool TRANS_OUT, int FIX>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_tma_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                    float* __restrict__ C, int64_t ldc, int64_t c_split_stride, int M, int N, int K,
                    int k_per_split, int accumulate, const int* __restrict__ mJ, int mk, int mod_n,
                    double* __restrict__ sq_partial, int c_async, const int* __restrict__ ready, int ready_rows,
                    const int* __restrict__ progress, int* __restrict__ defer, unsigned long long stall_ns,
                    uint16_t* __restrict__ hout, const double* __restrict__ hscale,
                    const int* __restrict__ f16_flag, float* __restrict__ out32) {
  using CF = Cfg<BN, STAGES>;
  // FIX 3: FIX 2 plus the sum of squares of the A operand (before rounding) into sq_partial.
  // FIX 4: residual epilogue -- C is an fp32 INPUT X; the CTA writes f16(2^(15-e) (X - acc)) to
  // hout in the row-block-interleaved layout of the f16 gather (8 rows x 2 bytes per column),
  // e = f16_scale_exp(*hscale) (hscale = ||X||_F^2, so no value can overflow f16).
  constexpr bool MASK = FIX == 1, ROUND = FIX == 2 || FIX == 3, FIXUP = FIX >= 1 && FIX <= 3;
  constexpr bool OPSQ = FIX == 3, DELTA = FIX == 4;
  extern __shared__ unsigned char smem_raw[];
  // 1024-byte alignment for the swizzled tiles
  // 1024-byte alignment by pointer arithmetic on the shared array (an integer round trip would
  // lose the address space and turn every epilogue shared access into a generic one)
  unsigned char* smem = smem_raw + ((1024u - (saddr(smem_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)STAGES * CF::kStage);
  uint64_t* empty = full + STAGES;
  uint64_t* masked = empty + STAGES;
  uint64_t* done = masked + STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 1);
  __shared__ int sJ[128];
  __shared__ double sq_red[4];
  __shared__ int s_deferred;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  APX_DCHECK(m0 < M && n0 < N);
  const int kz = blockIdx.z;
  const int kbeg = kz * k_per_split, kend = min(K, kbeg + k_per_split);
  const int ktiles = (int)ceil_div(max(0, kend - kbeg), BK);

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
      mbar_init(&masked[s], 4);  // one arrival per mask warp
    }
    mbar_init(done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmA) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmB) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(saddr(tmem_slot)),
                 "r"(CF::kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  // programmatic dependent launch: the prologue above (barriers, TMEM, tensor-map prefetch) ran
  // while the previous kernel drained; its outputs are read only after this wait
  pdl_wait();
  for (int t = threadIdx.x; t < mk && t < 128; t += kThreads) sJ[t] = mJ[t];
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t sbase = saddr(smem);

  if (warp == 0) {
    // ---------------- TMA producer ----------------
    if (lane == 0) {
      for (int kt = 0; kt < ktiles; ++kt) {
        const int s = kt % STAGES;
        if (kt >= STAGES) mbar_wait(&empty[s], (uint32_t)(((kt / STAGES) - 1) & 1));
        mbar_expect_tx(&full[s], (uint32_t)CF::kStage);
        const uint32_t a_s = sbase + s * CF::kStage, b_s = a_s + CF::kTileA;
        const int k0 = kbeg + kt * BK;
        if (!A_MN) {
          tma_load_2d(a_s, &tmA, k0, m0, &full[s]);
        } else {
#pragma unroll
          for (int a = 0; a < BM / 32; ++a) tma_load_2d(a_s + a * 4096, &tmA, m0 + 32 * a, k0, &full[s]);
        }
        if (!B_MN) {
          tma_load_2d(b_s, &tmB, k0, n0, &full[s]);
        } else {
#pragma unroll
          for (int a = 0; a < BN / 32; ++a) tma_load_2d(b_s + a * 4096, &tmB, n0 + 32 * a, k0, &full[s]);
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer ----------------
    constexpr uint32_t id = idesc(BM, BN, A_MN, B_MN);
    if (lane == 0) {
      for (int kt = 0; kt < ktiles; ++kt) {
        const int s = kt % STAGES;
        const uint32_t ph = (uint32_t)((kt / STAGES) & 1);
        if (FIXUP) mbar_wait(&masked[s], ph);
        else mbar_wait(&full[s], ph);
        fence_after();
        const uint32_t a_s = sbase + s * CF::kStage, b_s = a_s + CF::kTileA;
#pragma unroll
        for (int kk = 0; kk < BK / 8; ++kk) {
          const uint64_t da = A_MN ? desc(a_s + kk * 1024, 4096, 512, 1) : desc(a_s + kk * 32, 16, 1024, 2);
          const uint64_t db = B_MN ? desc(b_s + kk * 1024, 4096, 512, 1) : desc(b_s + kk * 32, 16, 1024, 2);
          mma(tmem, da, db, id, (kt > 0 || kk > 0) ? 1u : 0u);
        }
        commit(&empty[s]);
      }
      if (ktiles > 0) commit(done);
      else mbar_arrive(done);
    }
  } else {
    // ---------------- mask fix-up (dB^T) + epilogue ----------------
    const int et = threadIdx.x - 64;  // 0..127
    double osq = 0.0;                  // FIX 3: this thread's share of the A operand's squares
    if (MASK) {
      for (int kt = 0; kt < ktiles; ++kt) {
        const int s = kt % STAGES;
        mbar_wait(&full[s], (uint32_t)((kt / STAGES) & 1));
        unsigned char* a_p = smem + (size_t)s * CF::kStage;
        const int k0 = kbeg + kt * BK;
        // shift t masks the diagonal m = (k0 + kk - J_t) mod n of the tile: test the whole
        // 32-row segment once, then zero the (rare) in-tile entries
        bool wrote = false;
        for (int t = et; t < mk; t += 128) {
          int off = k0 - sJ[t] - m0;  // m - m0 at kk = 0, taken mod n below
          off %= mod_n;
          if (off < 0) off += mod_n;
          if (off < BM || off + BK - 1 >= mod_n) {
            wrote = true;
#pragma unroll 4
            for (int kk = 0; kk < BK; ++kk) {
              int q = off + kk;
              if (q >= mod_n) q -= mod_n;
              if (q < BM) *reinterpret_cast<float*>(a_p + mn_off(q, kk)) = 0.f;
            }
          }
        }
        // generic-proxy writes must be made visible to the tensor core (async proxy) before the
        // MMA issuer is released; warps that wrote nothing skip the proxy fence
        if (__any_sync(0xffffffffu, wrote)) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive(&masked[s]);
      }
    }
    if (ROUND) {
      for (int kt = 0; kt < ktiles; ++kt) {
        const int s = kt % STAGES;
        mbar_wait(&full[s], (uint32_t)((kt / STAGES) & 1));
        // every 4-byte word of the A tile is an operand value: round in place (the B operand,
        // Q, is produced already rounded: qr_orthonormalize(..., tf32 = 1))
        uint4* w = reinterpret_cast<uint4*>(smem + (size_t)s * CF::kStage);
        float osq32 = 0.f;
#pragma unroll 4
        for (int v = et; v < CF::kTileA / 16; v += 128) {
          // round the magnitude half-up at bit 13 (sign-magnitude: an integer add on the bits;
          // a carry into the exponent is the correct rounding): two integer ops per value
          uint4 x = w[v];
          if constexpr (OPSQ) {
            osq32 = fmaf(__uint_as_float(x.x), __uint_as_float(x.x), osq32);
            osq32 = fmaf(__uint_as_float(x.y), __uint_as_float(x.y), osq32);
            osq32 = fmaf(__uint_as_float(x.z), __uint_as_float(x.z), osq32);
            osq32 = fmaf(__uint_as_float(x.w), __uint_as_float(x.w), osq32);
          }
          x.x = (x.x + 0x1000u) & 0xffffe000u;
          x.y = (x.y + 0x1000u) & 0xffffe000u;
          x.z = (x.z + 0x1000u) & 0xffffe000u;
          x.w = (x.w + 0x1000u) & 0xffffe000u;
          w[v] = x;
        }
        osq += (double)osq32;  // one short fp32 partial per K-tile, folded in fp64
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive(&masked[s]);
      }
    }
    // C tile staged through the (drained) operand ring for a read-modify-write epilogue
    constexpr bool kStageC = !TRANS_OUT && (size_t)STAGES * CF::kStage >= (size_t)BM * BN * 4;
    bool stage_c = kStageC && accumulate && c_async;
    if (DELTA) {
      // the residual epilogue stages this CTA's X tile (an HBM read): pull it into L2 during the
      // main loop, one 128-byte line per thread per step
      for (int e = et; e < BM * (BN / 32); e += 128) {
        const int r = m0 + e / (BN / 32), c = n0 + (e % (BN / 32)) * 32;
        if (r < M && c < N) asm volatile("prefetch.global.L2 [%0];" ::"l"(C + (size_t)r * ldc + c));
      }
    }
    if (accumulate && !TRANS_OUT && !stage_c) {
      // the read-modify-write epilogue reads this CTA's C tile: start pulling it toward L2 now
      // (overlaps the main loop); 128 threads x BN/32 lines per row group
      for (int rr = et; rr < BM; rr += 128) {
        const int r = m0 + rr;
        if (r < M)
          for (int cc = 0; cc < BN; cc += 32)
            if (n0 + cc < N) asm volatile("prefetch.global.L2 [%0];" ::"l"(C + (size_t)kz * c_split_stride + (size_t)r * ldc + n0 + cc));
      }
    }
    mbar_wait(done, 0);
    fence_after();
    if constexpr (DELTA) {
      // X tile staged through the drained ring (cp.async, XOR-swizzled granules as in the
      // read-modify-write path below), v = s (X - acc) in place, then 8-row groups stored as one
      // 16-byte f16 vector per column: a warp writes 32 consecutive columns = 512 contiguous bytes
      static_assert((size_t)STAGES * CF::kStage >= (size_t)BM * BN * 4, "residual epilogue needs the staged tile");
      const int quarter = warp & 3;
      constexpr int GPR = BN / 4;
      float* creg = reinterpret_cast<float*>(smem) + (size_t)quarter * 32 * BN;
      const int rbase = m0 + quarter * 32;
      const float* X = C;
#pragma unroll 4
      for (int g = lane; g < 32 * GPR; g += 32) {
        const int r = g / GPR, gc = g - r * GPR;
        const int rg = rbase + r, cg = n0 + gc * 4;
        const bool ok = rg < M && cg < N;
        const float* src = ok ? X + (size_t)rg * ldc + cg : X;
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(saddr(creg + r * BN + ((gc ^ (r & 7)) << 2))),
                     "l"(src), "r"(ok ? 16 : 0)
                     : "memory");
      }
      asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
      __syncwarp();
      // f16_flag == 0 (the residual plan's fallback): X - acc in fp32, row-major into out32
      const bool to_f16 = f16_flag == nullptr || *f16_flag != 0;
      const float sc = to_f16 ? ldexpf(1.f, 15 - f16_scale_exp(*hscale)) : 1.f;
#pragma unroll 1
      for (int j0 = 0; j0 < BN; j0 += 32) {
        float v[32];
        if (ktiles > 0) {
          tmem_ld32(tmem + ((uint32_t)(quarter * 32) << 16) + (uint32_t)j0, v);
        } else {
#pragma unroll
          for (int i = 0; i < 32; ++i) v[i] = 0.f;
        }
        float* rowp = creg + lane * BN;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          float4* p4 = reinterpret_cast<float4*>(rowp + ((((j0 >> 2) + i) ^ (lane & 7)) << 2));
          float4 o = *p4;
          o.x = sc * (o.x - v[4 * i]);
          o.y = sc * (o.y - v[4 * i + 1]);
          o.z = sc * (o.z - v[4 * i + 2]);
          o.w = sc * (o.w - v[4 * i + 3]);
          *p4 = o;
        }
      }
      __syncwarp();
      if (!to_f16) {
#pragma unroll 4
        for (int r = 0; r < 32; ++r) {
          const int rg = rbase + r;
          if (rg >= M) break;
#pragma unroll
          for (int j0 = 0; j0 < BN; j0 += 32) {
            const int c = j0 + lane;
            if (n0 + c < N) out32[(size_t)rg * N + n0 + c] = creg[r * BN + ((((c >> 2) ^ (r & 7))) << 2) + (c & 3)];
          }
        }
      }
#pragma unroll 1
      for (int g8 = 0; g8 < 4 && to_f16; ++g8) {
        const int r8 = rbase + 8 * g8;
        if (r8 >= M) break;
        uint4* dst = reinterpret_cast<uint4*>(hout) + (size_t)(r8 >> 3) * N + n0;
#pragma unroll
        for (int j0 = 0; j0 < BN; j0 += 32) {
          const int c = j0 + lane;
          uint32_t w[4];
#pragma unroll
          for (int h = 0; h < 4; ++h) {
            const int ra = 8 * g8 + 2 * h, rb = ra + 1;
            const float a = creg[ra * BN + ((((c >> 2) ^ (ra & 7))) << 2) + (c & 3)];
            const float b = creg[rb * BN + ((((c >> 2) ^ (rb & 7))) << 2) + (c & 3)];
            w[h] = pack_half2(a, b);
          }
          if (n0 + c < N) dst[c] = make_uint4(w[0], w[1], w[2], w[3]);
        }
      }
    } else {
    bool deferred = false;
    if (ready != nullptr && accumulate) {
      // C rows are produced by a concurrent kernel (the persistent gather) that publishes one flag
      // per block of ready_rows rows: wait (acquire) for the blocks under this tile before reading
      // C. The operand pipeline above has already run, so only the read-modify-write waits.
      // The first epilogue warp polls one flag per lane (relaxed loads, all in flight at once),
      // then one fence turns the observed flags into an acquire for the whole CTA.
      // Bounded wait: if the producer makes no progress at all (its `progress` counter -- the
      // gather's row-block ticket -- stands still for stall_ns (20 ms), e.g. because none of its CTAs is
      // resident under an MPS SM limit or a co-tenant), the tile is deferred instead: it leaves
      // C untouched, records itself in `defer`, and qw_fixup_sum_kernel adds its Q.W after the
      // producer finished (stream-ordered), so the SMs held here are released.
      if (warp == 2) {
        const int b0 = m0 / ready_rows, b1 = (min(M, m0 + BM) - 1) / ready_rows;
        bool stalled = false;
        unsigned long long t0 = 0;
        int last = 0;
        if (defer && lane == 0) {
          asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
          last = ld_relaxed_gpu(progress);
        }
        if (defer && stall_ns == 0) stalled = true;  // test mode: defer every tile
        for (int bb = b0; bb <= b1 && !stalled; bb += 32) {
          const int b = bb + lane;
          while (!__all_sync(0xffffffffu, b > b1 || ld_relaxed_gpu(ready + b) != 0)) {
            __nanosleep(128);
            if (defer) {
              int st = 0;
              if (lane == 0) {
                unsigned long long now;
                asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
                const int cur = ld_relaxed_gpu(progress);
                if (cur != last) {
                  last = cur;
                  t0 = now;
                } else if (now - t0 > stall_ns) {
                  st = 1;
                }
              }
              if (__shfl_sync(0xffffffffu, st, 0)) {
                stalled = true;
                break;
              }
            }
          }
        }
        if (lane == 0) s_deferred = stalled ? 1 : 0;
        __threadfence();
      }
      asm volatile("bar.sync 2, 128;" ::: "memory");  // the four epilogue warps only
      deferred = s_deferred != 0;
    }
    if (deferred && et == 0) {
      const int slot = atomicAdd(defer, 1);
      APX_DCHECK(slot < (int)(gridDim.x * gridDim.y * gridDim.z));
      defer[1 + slot] = ((int)blockIdx.z * (int)gridDim.y + (int)blockIdx.y) * (int)gridDim.x + (int)blockIdx.x;
    }
    const int quarter = warp & 3;
    const int row = m0 + quarter * 32 + lane;
    float* Cz = C + (size_t)kz * c_split_stride;
    double sq = 0.0;  // sum of squares of the values this thread stores (sq_partial)
    if (deferred) stage_c = false;
    if (stage_c) {
      // Each warp copies its 32 x BN slab of C into the ring with cp.async (every 16-byte granule
      // in flight at once), adds the accumulator in place, then streams the rows back out.
      // Granule gc of row r sits at (gc ^ (r & 7)): row-wise float4 access (lane = row) and
      // column-wise reads (lane = column) are both bank-conflict free.
      constexpr int GPR = BN / 4;
      float* creg = reinterpret_cast<float*>(smem) + (size_t)quarter * 32 * BN;
      const int rbase = m0 + quarter * 32;
#pragma unroll 4
      for (int g = lane; g < 32 * GPR; g += 32) {
        const int r = g / GPR, gc = g - r * GPR;
        const int rg = rbase + r, cg = n0 + gc * 4;
        const bool ok = rg < M && cg < N;
        const float* src = ok ? Cz + (size_t)rg * ldc + cg : Cz;
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(saddr(creg + r * BN + ((gc ^ (r & 7)) << 2))),
                     "l"(src), "r"(ok ? 16 : 0)
                     : "memory");
      }
      asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
      __syncwarp();
#pragma unroll 1
      for (int j0 = 0; j0 < BN; j0 += 32) {
        float v[32];
        if (ktiles > 0) {
          tmem_ld32(tmem + ((uint32_t)(quarter * 32) << 16) + (uint32_t)j0, v);
        } else {
#pragma unroll
          for (int i = 0; i < 32; ++i) v[i] = 0.f;
        }
        float* rowp = creg + lane * BN;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          float4* p4 = reinterpret_cast<float4*>(rowp + ((((j0 >> 2) + i) ^ (lane & 7)) << 2));
          float4 o = *p4;
          o.x += v[4 * i];
          o.y += v[4 * i + 1];
          o.z += v[4 * i + 2];
          o.w += v[4 * i + 3];
          *p4 = o;
        }
      }
      __syncwarp();
      float sq32[2] = {0.f, 0.f};  // short fp32 partial sums, folded into the fp64 total
#pragma unroll 4
      for (int r = 0; r < 32; ++r) {
        const int rg = rbase + r;
        if (rg >= M) break;
        const float* rowp = creg + r * BN;
#pragma unroll
        for (int j0 = 0; j0 < BN; j0 += 32) {
          const int c = j0 + lane;
          const float val = rowp[((((c >> 2) ^ (r & 7))) << 2) | (c & 3)];
          if (n0 + c < N) {
            Cz[(size_t)rg * ldc + n0 + c] = val;
            sq32[r & 1] = fmaf(val, val, sq32[r & 1]);
          }
        }
      }
      sq += (double)sq32[0] + (double)sq32[1];
    }
#pragma unroll 1
    for (int j0 = 0; j0 < BN && !stage_c && !deferred; j0 += 32) {
      float v[32];
      if (ktiles > 0) {
        tmem_ld32(tmem + ((uint32_t)(quarter * 32) << 16) + (uint32_t)j0, v);
      } else {
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] = 0.f;
      }
      if (!TRANS_OUT) {
        // transpose the warp's 32 x 32 chunk through shared memory (the drained stage ring) so
        // every store instruction writes 128 contiguous bytes of one output row
        float* tw = reinterpret_cast<float*>(smem) + (warp - 2) * (32 * 33);
        __syncwarp();
#pragma unroll
        for (int i = 0; i < 32; ++i) tw[lane * 33 + i] = v[i];
        __syncwarp();
        const int col = n0 + j0 + lane;
#pragma unroll 1
        for (int r8 = 0; r8 < 32; r8 += 16) {
          // accumulate: the 16 old values are loaded before the first store (one latency, not 16)
          float old[16];
#pragma unroll
          for (int r = 0; r < 16; ++r) {
            const int rr = m0 + quarter * 32 + r8 + r;
            old[r] = (accumulate && rr < M && col < N) ? Cz[(size_t)rr * ldc + col] : 0.f;
          }
#pragma unroll
          for (int r = 0; r < 16; ++r) {
            const int rr = m0 + quarter * 32 + r8 + r;
            if (rr < M && col < N) {
              const float val = old[r] + tw[(r8 + r) * 33 + lane];
              Cz[(size_t)rr * ldc + col] = val;
              sq = fma((double)val, (double)val, sq);
            }
          }
        }
      } else if (row < M) {
        {
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            const int col = n0 + j0 + i;
            if (col < N) {
              float* p = Cz + (size_t)col * ldc + row;
              const float val = accumulate ? *p + v[i] : v[i];
              *p = val;
              sq = fma((double)val, (double)val, sq);
            }
          }
        }
      }
    }
    if (sq_partial) {
      if constexpr (OPSQ) sq = osq;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, o);
      if (lane == 0) sq_red[quarter] = sq;
      asm volatile("bar.sync 1, 128;" ::: "memory");  // the four epilogue warps only
      if (et == 0)
        sq_partial[((size_t)blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x] =
            (sq_red[0] + sq_red[1]) + (sq_red[2] + sq_red[3]);
    }
    }  // !DELTA
  }
  fence_before();
  __syncthreads();
  if (warp == 1) {
    fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(CF::kTmemCols));
  }
}

// ---- host: tensor maps through the driver entry point (no libcuda link dependency) ----------
using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeFn encode_fn() {
  static EncodeFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeFn>(p);
  });
  return fn;
}

// 2-D fp32 tensor map over a row-major [rows][cols] array with leading dimension ld (elements).
// kmajor: box = 32 cols x box_rows, 128B swizzle. mnmajor: box = 32 x 32, 128B/32B-atom swizzle.
static int make_map(CUtensorMap* map, const float* base, int64_t rows, int64_t cols, int64_t ld, int box_rows,
                    bool mn_major) {
  EncodeFn fn = encode_fn();
  if (!fn) {
    set_error("cuTensorMapEncodeTiled unavailable");
    return E_CUDA;
  }
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)(ld * 4)};
  cuuint32_t box[2] = {32u, (cuuint32_t)(mn_major ? 32 : box_rows)};
  cuuint32_t estr[2] = {1u, 1u};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, (void*)base, dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE,
                  mn_major ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled failed (%d): rows=%lld cols=%lld ld=%lld", (int)r, (long long)rows,
              (long long)cols, (long long)ld);
    return E_CUDA;
  }
  return OK;
}

// Stall threshold of the bounded ready-flag wait; APX_QW_STALL_NS overrides it (0 = test mode:
// every tile defers, exercising the fixup path end to end).
static unsigned long long stall_ns() {
  static const unsigned long long v = [] {
    const char* e = getenv("APX_QW_STALL_NS");
    return e ? strtoull(e, nullptr, 10) : 20ull * 1000 * 1000;
  }();
  return v;
}

template <int BN, int STAGES, bool A_MN, bool B_MN, bool TRANS_OUT, int FIX>
static int launch(const float* A, int64_t lda, const float* B, int64_t ldb, float* C, int64_t ldc,
                  int64_t c_split_stride, int M, int N, int K, int splits, int accumulate, const int* mJ, int mk,
                  int mod_n, double* sq_partial, const int* ready, int ready_rows, const int* progress,
                  int* defer, uint16_t* hout, const double* hscale, const int* f16_flag, float* out32,
                  cudaStream_t st) {
  using CF = Cfg<BN, STAGES>;
  CUtensorMap ta, tb;
  // A operand: K-major stored [M][K]; MN-major stored [K][M]
  APX_TRY(make_map(&ta, A, A_MN ? K : M, A_MN ? M : K, lda, BM, A_MN));
  APX_TRY(make_map(&tb, B, B_MN ? K : N, B_MN ? N : K, ldb, BN, B_MN));
  const int kps = (int)(ceil_div(ceil_div(K, splits), BK) * BK);
  dim3 grid((unsigned)ceil_div(N, BN), (unsigned)ceil_div(M, BM), (unsigned)splits);
  auto fn = gemm_tma_kernel<BN, STAGES, A_MN, B_MN, TRANS_OUT, FIX>;
  APX_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)CF::kSmem));
  const int c_async = ((uintptr_t)C % 16) == 0 && (ldc % 4) == 0 && (N % 4) == 0 && (c_split_stride % 4) == 0;
  APX_CUDA(launch_pdl(fn, grid, dim3(kThreads), CF::kSmem, st, ta, tb, C, ldc, c_split_stride, M, N, K, kps,
                      accumulate, mJ, mk, mod_n, sq_partial, c_async, ready, ready_rows, progress, defer, stall_ns(),
                      hout, hscale, f16_flag, out32));
  APX_LAUNCH_CHECK();
  return OK;
}


// ---- persistent n x n tile loop: C[M x N] (=|+=) A[M x K] . B[K x N] ------------------------------
// A K-major (row-major [M][K]), B MN-major (row-major [K][N]); the C4 product's M (+)= Q.W with a
// short K (2l = 128). One CTA per SM walks tiles t = blockIdx.x + i * gridDim.x (row-band-major:
// t = band * ceil(N/BN) + column tile), with the accumulator double-buffered in TMEM
// (2 x BN columns): the MMA warp fills buffer (i+1)&1 while the epilogue warps drain buffer i&1,
// and the TMA producer streams the K-chunks of the next tiles through a 4-stage ring. So the
// HBM-bound epilogue (the C tile's read-modify-write) overlaps the next tile's operand loads,
// which the one-tile-per-CTA kernel above serialises (~48% of the HBM bandwidth at 3 CTAs per SM).
// Epilogue: 32 x 32 chunks transposed through shared memory (row-contiguous 128-byte stores),
// ACC: all 16 old values of a half-chunk loaded before the first store; ready flags, bounded wait,
// deferral and per-tile ||C||^2 partials exactly as gemm_tma_kernel (same tile numbering, so
// qw_fixup_sum_kernel completes deferred tiles unchanged).
constexpr int kPStages = 3;
constexpr int kPQueue = 4;  // tile-id queue depth (dynamic scheduling)
template <int BN>
struct PCfg {
  static constexpr int kTileA = BM * BK * 4;
  static constexpr int kTileB = BN * BK * 4;
  static constexpr int kStage = kTileA + kTileB;
  static constexpr int kSlab = 32 * BN * 4;                // one epilogue warp's 32 x BN slab of C
  static constexpr int kStaging = 4 * 2 * kSlab;           // double-buffered per warp
  static constexpr size_t kSmem = (size_t)kPStages * kStage + kStaging + 1024 + 512;
  static constexpr int kTmemCols = 2 * BN;
};

__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, int c0, int c1, uint32_t src) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(map), "r"(c0),
               "r"(c1), "r"(src)
               : "memory");
}

// Tile order: with `ticket` (dynamic), the producer claims tiles in ascending order from a global
// counter and passes each id to the MMA warp and the epilogue through a kPQueue-deep shared queue
// (tile_ready: producer -> consumers, release/acquire; tile_free: 1 MMA + 4 epilogue arrivals), so
// whichever CTAs are resident work the lowest open tiles -- required when the CTAs only get SMs as a
// concurrent kernel releases them and the epilogues wait on that kernel's row flags. Without a
// ticket the tiles are strided statically (t = blockIdx.x + i * gridDim.x).
// Epilogue: TMA in and out. Each epilogue warp owns a double-buffered 32 x BN slab of C laid out
// as BN/32 boxes of 32 x 32 fp32 in the 128-byte swizzle (granule g of row r at g ^ (r & 7)): the
// old C slab (ACC) arrives by TMA (issued before the accumulator wait, so it overlaps the MMAs),
// the lane owning row r adds its TMEM row into its granules (conflict-free 16-byte accesses), and
// one TMA store per box writes the slab back; the slab is reused two tiles later, after the
// store has finished reading it (bulk wait_group.read).
template <int BN, bool ACC>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_persist_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                        const __grid_constant__ CUtensorMap tmC, int M, int N, int K, double* __restrict__ sq_partial,
                        const int* __restrict__ ready, int ready_rows, const int* __restrict__ progress,
                        int* __restrict__ defer, unsigned long long stall_ns, int* __restrict__ ticket) {
  using CF = PCfg<BN>;
  extern __shared__ unsigned char smem_raw[];
  unsigned char* smem = smem_raw + ((1024u - (saddr(smem_raw) & 1023u)) & 1023u);
  unsigned char* stg = smem + (size_t)kPStages * CF::kStage;
  uint64_t* full = reinterpret_cast<uint64_t*>(stg + CF::kStaging);
  uint64_t* empty = full + kPStages;
  uint64_t* acc_full = empty + kPStages;
  uint64_t* acc_empty = acc_full + 2;
  uint64_t* tile_ready = acc_empty + 2;
  uint64_t* tile_free = tile_ready + kPQueue;
  uint64_t* cbar = tile_free + kPQueue;  // [warp 0..3][slab 0..1]: the old C slab landed
  int* tile_id = reinterpret_cast<int*>(cbar + 8);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tile_id + kPQueue);
  __shared__ double sq_red[4];
  __shared__ int s_deferred[4];

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nct = (int)ceil_div(N, BN);
  const int tiles = (int)ceil_div(M, BM) * nct;
  const int kchunks = (int)ceil_div(K, BK);
  if (warp == 0 && lane == 0) {
    for (int s = 0; s < kPStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&acc_full[b], 1);
      mbar_init(&acc_empty[b], 4);  // one arrival per epilogue warp
    }
    for (int q = 0; q < kPQueue; ++q) {
      mbar_init(&tile_ready[q], 1);
      mbar_init(&tile_free[q], 5);  // the MMA lane + one lane per epilogue warp
    }
    for (int q = 0; q < 8; ++q) mbar_init(&cbar[q], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmA) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmB) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmC) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(saddr(tmem_slot)),
                 "r"(CF::kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  pdl_wait();  // programmatic dependent launch (see gemm_tma_kernel)
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t sbase = saddr(smem);
  // consumer side of the tile queue: the i-th tile id (>= tiles: done)
  auto next_tile = [&](int i, int t_static) -> int {
    if (!ticket) return t_static;
    const int q = i % kPQueue;
    mbar_wait(&tile_ready[q], (uint32_t)((i / kPQueue) & 1));
    return tile_id[q];
  };
  auto release_tile = [&](int i) {
    if (ticket) mbar_arrive(&tile_free[i % kPQueue]);
  };

  if (warp == 0) {
    if (lane == 0) {
      int g = 0;  // global K-chunk counter over this CTA's tiles
      for (int i = 0;; ++i) {
        int t;
        if (ticket) {
          const int q = i % kPQueue;
          if (i >= kPQueue) mbar_wait(&tile_free[q], (uint32_t)(((i / kPQueue) - 1) & 1));
          t = atomicAdd(ticket, 1);
          tile_id[q] = t;
          mbar_arrive(&tile_ready[q]);
        } else {
          t = blockIdx.x + i * gridDim.x;
        }
        if (t >= tiles) break;
        const int m0 = (t / nct) * BM, n0 = (t % nct) * BN;
        for (int kc = 0; kc < kchunks; ++kc, ++g) {
          const int s = g % kPStages;
          if (g >= kPStages) mbar_wait(&empty[s], (uint32_t)(((g / kPStages) - 1) & 1));
          mbar_expect_tx(&full[s], (uint32_t)CF::kStage);
          const uint32_t a_s = sbase + s * CF::kStage, b_s = a_s + CF::kTileA;
          const int k0 = kc * BK;
          tma_load_2d(a_s, &tmA, k0, m0, &full[s]);
#pragma unroll
          for (int a = 0; a < BN / 32; ++a) tma_load_2d(b_s + a * 4096, &tmB, n0 + 32 * a, k0, &full[s]);
        }
      }
    }
  } else if (warp == 1) {
    constexpr uint32_t id = idesc(BM, BN, false, true);
    if (lane == 0) {
      int g = 0;
      for (int i = 0;; ++i) {
        const int t = next_tile(i, blockIdx.x + i * gridDim.x);
        release_tile(i);
        if (t >= tiles) break;
        const int b = i & 1;
        if (i >= 2) mbar_wait(&acc_empty[b], (uint32_t)(((i >> 1) - 1) & 1));
        fence_after();
        const uint32_t d = tmem + (uint32_t)(b * BN);
        for (int kc = 0; kc < kchunks; ++kc, ++g) {
          const int s = g % kPStages;
          mbar_wait(&full[s], (uint32_t)((g / kPStages) & 1));
          fence_after();
          const uint32_t a_s = sbase + s * CF::kStage, b_s = a_s + CF::kTileA;
#pragma unroll
          for (int kk = 0; kk < BK / 8; ++kk)
            mma(d, desc(a_s + kk * 32, 16, 1024, 2), desc(b_s + kk * 1024, 4096, 512, 1), id,
                (kc > 0 || kk > 0) ? 1u : 0u);
          commit(&empty[s]);
        }
        commit(&acc_full[b]);
      }
    }
  } else {
    const int quarter = warp & 3, ew = warp - 2;
    int loads = 0;  // per slab: C loads issued so far (mbarrier phase)
    int lslab0 = 0, lslab1 = 0;
    for (int i = 0;; ++i) {
      int t = 0;
      if (lane == 0) t = next_tile(i, blockIdx.x + i * gridDim.x);
      t = __shfl_sync(0xffffffffu, t, 0);
      __syncwarp();
      if (lane == 0) release_tile(i);
      if (t >= tiles) break;
      const int b = i & 1;  // TMEM buffer and slab
      const int m0 = (t / nct) * BM, n0 = (t % nct) * BN;
      const int rbase = m0 + quarter * 32;
      unsigned char* slab = stg + (size_t)(ew * 2 + b) * CF::kSlab;
      const uint32_t slab_s = saddr(slab);
      uint64_t* cb = &cbar[ew * 2 + b];
      bool deferred = false;
      if (ACC && ready != nullptr) {
        // wait (acquire) for the producer's row blocks under this warp's 32 rows; bounded as in
        // gemm_tma_kernel: a producer without progress for stall_ns defers the tile
        const int b0 = rbase / ready_rows, b1 = (min(M, rbase + 32) - 1) / ready_rows;
        bool stalled = defer != nullptr && stall_ns == 0;
        unsigned long long t0 = 0;
        int last = 0;
        if (defer && lane == 0) {
          asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
          last = ld_relaxed_gpu(progress);
        }
        for (int bb = b0; bb <= b1 && !stalled && rbase < M; bb += 32) {
          const int fb = bb + lane;
          while (!__all_sync(0xffffffffu, fb > b1 || ld_relaxed_gpu(ready + fb) != 0)) {
            __nanosleep(128);
            if (defer) {
              int st = 0;
              if (lane == 0) {
                unsigned long long now;
                asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
                const int cur = ld_relaxed_gpu(progress);
                if (cur != last) {
                  last = cur;
                  t0 = now;
                } else if (now - t0 > stall_ns) {
                  st = 1;
                }
              }
              if (__shfl_sync(0xffffffffu, st, 0)) {
                stalled = true;
                break;
              }
            }
          }
        }
        __threadfence();
        // the tile is deferred (whole: the fixup kernel redoes all 128 rows) if any warp stalled
        if (lane == 0) s_deferred[quarter] = stalled ? 1 : 0;
        asm volatile("bar.sync 1, 128;" ::: "memory");
        deferred = (s_deferred[0] | s_deferred[1] | s_deferred[2] | s_deferred[3]) != 0;
        asm volatile("bar.sync 1, 128;" ::: "memory");  // s_deferred is rewritten by the next tile
        if (deferred && threadIdx.x == 64) {
          const int slot = atomicAdd(defer, 1);
          defer[1 + slot] = t;
        }
      }
      // this slab's previous TMA store (tile i - 2) must have finished reading it
      if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
      __syncwarp();
      uint32_t cphase = 0;
      const bool load_c = ACC && !deferred && rbase < M;
      if (load_c) {
        int& nl = b ? lslab1 : lslab0;
        cphase = (uint32_t)(nl & 1);
        ++nl;
        if (lane == 0) {
          mbar_expect_tx(cb, (uint32_t)CF::kSlab);
#pragma unroll
          for (int j = 0; j < BN / 32; ++j) tma_load_2d(slab_s + j * 4096, &tmC, n0 + 32 * j, rbase, cb);
        }
      }
      (void)loads;
      mbar_wait(&acc_full[b], (uint32_t)((i >> 1) & 1));
      fence_after();
      double sq = 0.0;
      float v[BN / 32][32];
#pragma unroll
      for (int j = 0; j < BN / 32; ++j)
        tmem_ld32(tmem + ((uint32_t)(quarter * 32) << 16) + (uint32_t)(b * BN + j * 32), v[j]);
      fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&acc_empty[b]);  // the MMA warp may refill this buffer
      if (!deferred && rbase < M) {
        if (load_c) mbar_wait(cb, cphase);
        float sq32 = 0.f;
#pragma unroll
        for (int j = 0; j < BN / 32; ++j)
#pragma unroll
          for (int i4 = 0; i4 < 8; ++i4) {
            float4* p4 = reinterpret_cast<float4*>(slab + j * 4096 + lane * 128 + ((i4 ^ (lane & 7)) << 4));
            float4 o = ACC ? *p4 : make_float4(0.f, 0.f, 0.f, 0.f);
            o.x += v[j][4 * i4];
            o.y += v[j][4 * i4 + 1];
            o.z += v[j][4 * i4 + 2];
            o.w += v[j][4 * i4 + 3];
            *p4 = o;
            sq32 = fmaf(o.x, o.x, fmaf(o.y, o.y, fmaf(o.z, o.z, fmaf(o.w, o.w, sq32))));
          }
        sq = (double)sq32;  // rows / columns past the edge hold zeros (TMA zero fill, zero operands)
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) {
#pragma unroll
          for (int j = 0; j < BN / 32; ++j) tma_store_2d(&tmC, n0 + 32 * j, rbase, slab_s + j * 4096);
          asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
      }
      if (sq_partial) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, o);
        if (lane == 0) sq_red[quarter] = sq;
        asm volatile("bar.sync 1, 128;" ::: "memory");
        if (threadIdx.x == 64) sq_partial[t] = deferred ? 0.0 : (sq_red[0] + sq_red[1]) + (sq_red[2] + sq_red[3]);
        asm volatile("bar.sync 1, 128;" ::: "memory");
      }
    }
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");  // stores complete
  }
  fence_before();
  __syncthreads();
  if (warp == 1) {
    fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(CF::kTmemCols));
  }
}

template <int BN, bool ACC>
static int launch_persist(const float* A, int64_t lda, const float* B, int64_t ldb, float* C, int64_t ldc, int M,
                          int N, int K, double* sq_partial, const int* ready, int ready_rows, const int* progress,
                          int* defer, int ctas, int* ticket, cudaStream_t st) {
  using CF = PCfg<BN>;
  CUtensorMap ta, tb, tc;
  APX_TRY(make_map(&ta, A, M, K, lda, BM, false));
  APX_TRY(make_map(&tb, B, K, N, ldb, BN, true));
  APX_TRY(make_map(&tc, C, M, N, ldc, 32, false));  // 32 x 32 boxes, 128-byte swizzle
  const int tiles = (int)(ceil_div(M, BM) * ceil_div(N, BN));
  auto fn = gemm_persist_kernel<BN, ACC>;
  APX_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)CF::kSmem));
  if (ticket) APX_CUDA(cudaMemsetAsync(ticket, 0, sizeof(int), st));
  APX_CUDA(launch_pdl(fn, dim3((unsigned)std::max(1, std::min(tiles, ctas))), dim3(kThreads), CF::kSmem, st, ta, tb,
                      tc, M, N, K, sq_partial, ready, ready_rows, progress, defer, stall_ns(), ticket));
  APX_LAUNCH_CHECK();
  return OK;
}

}  // namespace tma

// Completes the tiles gemm_tma_kernel deferred (bounded wait: its producer made no progress)
// and then sums the per-tile ||C||^2 partials exactly like sum_vector_kernel (1024 threads,
// strided per-thread sums, fixed block tree), so the normal path's bits are unchanged. One CTA:
// this only runs real work in the pathological no-co-residency case; normally defer[0] == 0.
// The deferred tiles use fp32 FMAs on TF32-truncated operands (the tensor core's inputs).
__global__ void __launch_bounds__(1024)
    qw_fixup_sum_kernel(const float* __restrict__ Q, int64_t ldq, const float* __restrict__ W, int64_t ldw,
                        float* __restrict__ C, int64_t ldc, int M, int N, int K, int bn, int* __restrict__ defer,
                        double* __restrict__ sq_partial, int parts, double* __restrict__ out) {
  __shared__ double sh[32];
  const int cnt = defer[0];
  const int gx = (int)ceil_div(N, bn);
  for (int d = 0; d < cnt; ++d) {
    const int tile = defer[1 + d];
    const int m0 = (tile / gx) * tma::BM, n0 = (tile % gx) * bn;
    double sq = 0.0;
    for (int e = threadIdx.x; e < tma::BM * bn; e += blockDim.x) {
      const int r = m0 + e / bn, c = n0 + e % bn;
      if (r >= M || c >= N) continue;
      float acc = 0.f;
      for (int k = 0; k < K; ++k)
        acc = fmaf(__uint_as_float(__float_as_uint(Q[(size_t)r * ldq + k]) & 0xffffe000u),
                   __uint_as_float(__float_as_uint(W[(size_t)k * ldw + c]) & 0xffffe000u), acc);
      const float val = C[(size_t)r * ldc + c] + acc;
      C[(size_t)r * ldc + c] = val;
      sq = fma((double)val, (double)val, sq);
    }
    sq = block_sum(sq, sh);
    if (threadIdx.x == 0) sq_partial[tile] = sq;
    __syncthreads();
  }
  if (threadIdx.x == 0) defer[0] = 0;  // ready for the next product
  double s = 0.0;
  for (int i = threadIdx.x; i < parts; i += blockDim.x) s += sq_partial[i];
  s = block_sum(s, sh);
  if (threadIdx.x == 0) *out = s;
}

int launch_qw_fixup_sum(const float* Q, int64_t ldq, const float* W, int64_t ldw, float* C, int64_t ldc, int M, int N,
                        int K, int bn, int* defer, double* sq_partial, int parts, double* out, cudaStream_t st) {
  qw_fixup_sum_kernel<<<1, 1024, 0, st>>>(Q, ldq, W, ldw, C, ldc, M, N, K, bn, defer, sq_partial, parts, out);
  APX_LAUNCH_CHECK();
  return OK;
}

// Same contract as umma_gemm (umma.cu); requires 16-byte aligned bases and leading dimensions,
// M, N multiples of 32 for MN-major operands. layout bits: 1 A MN-major, 2 B MN-major, 4 C^T.
// sq_partial (optional): one fp64 sum of squares of the stored values per CTA, indexed
// (z * grid.y + y) * grid.x + x -- ||C||_F^2 partials for a split-free launch.
int umma_tma_gemm(int layout, int bn, const float* A, int64_t lda, const float* B, int64_t ldb, float* C,
                  int64_t ldc, int64_t c_split_stride, int M, int N, int K, int splits, int accumulate,
                  const int* mJ, int mk, int mod_n, cudaStream_t st, double* sq_partial, const int* ready,
                  int ready_rows, const int* progress, int* defer, uint16_t* hout, const double* hscale,
                  const int* f16_flag, float* out32) {
  APX_REQUIRE(ready == nullptr || (accumulate && ready_rows > 0 && splits == 1 && !(layout & 4)),
              "umma_tma_gemm: ready flags need an accumulating, split-free, row-major C");
  APX_REQUIRE(defer == nullptr || (ready != nullptr && progress != nullptr && sq_partial != nullptr),
              "umma_tma_gemm: deferral needs ready flags, a progress counter and sq partials");
  APX_REQUIRE(mk <= 128, "umma_tma_gemm: at most 128 masked shifts");
  APX_REQUIRE(((uintptr_t)A % 16) == 0 && ((uintptr_t)B % 16) == 0 && (lda % 4) == 0 && (ldb % 4) == 0,
              "umma_tma_gemm: 16-byte aligned operands required");
  const bool mask = mJ != nullptr && mk > 0;
  // layout bit 8: round the A operand to TF32 nearest (+ bit 16: its sum of squares into
  // sq_partial); bit 32: residual epilogue (C is the fp32 input X, the f16 result goes to hout)
  const int fix = mask ? 1 : (layout & 32) ? 4 : (layout & 8) ? ((layout & 16) ? 3 : 2) : 0;
  APX_REQUIRE(fix != 4 || (hout != nullptr && hscale != nullptr && splits == 1 && (layout & 7) == 2 && bn == 128 &&
                           ((uintptr_t)hout % 16) == 0 && (N % 4) == 0 && ((uintptr_t)C % 16) == 0 && (ldc % 4) == 0),
              "umma_tma_gemm: residual epilogue needs hout, hscale, layout 2, BN 128, no split, aligned X");
  layout &= 7;
  // ring depth: BN 128 with K <= 4 K-tiles runs 2 stages (64 KB: three CTAs per SM, and the
  // drained ring holds a staged C tile)
  const int stages = bn == 256 ? 2 : (bn == 128 && K <= 4 * tma::BK) ? 2 : 4;
#define APX_TL(BNV, ST, L, FX)                                                                               \
  if (bn == BNV && stages == ST && layout == L && fix == FX)                                                 \
    return tma::launch<BNV, ST, (L & 1) != 0, (L & 2) != 0, (L & 4) != 0, FX>(A, lda, B, ldb, C, ldc,         \
                                                                              c_split_stride, M, N, K, splits, \
                                                                              accumulate, mJ, mk, mod_n,       \
                                                                              sq_partial, ready, ready_rows,   \
                                                                              progress, defer, hout, hscale,   \
                                                                              f16_flag, out32, st);
  APX_TL(64, 4, 0, 0) APX_TL(64, 4, 1, 0) APX_TL(64, 4, 2, 0) APX_TL(64, 4, 3, 0)
  APX_TL(64, 4, 4, 0) APX_TL(64, 4, 5, 0) APX_TL(64, 4, 6, 0) APX_TL(64, 4, 7, 0)
  APX_TL(64, 4, 1, 1) APX_TL(64, 4, 5, 1) APX_TL(64, 4, 7, 2) APX_TL(64, 4, 7, 3) APX_TL(128, 2, 2, 4)
  APX_TL(128, 4, 0, 0) APX_TL(128, 4, 2, 0) APX_TL(256, 2, 0, 0) APX_TL(256, 2, 2, 0)
  APX_TL(128, 2, 0, 0) APX_TL(128, 2, 2, 0)
#undef APX_TL
  set_error("umma_tma_gemm: unsupported layout %d / BN %d / fix-up %d", layout, bn, fix);
  return E_ARG;
}

// Persistent C[M x N] (=|+=) A[M x K] . B[K x N] (A row-major [M][K], B row-major [K][N], 16-byte
// aligned, N a multiple of 32): the tile loop of gemm_persist_kernel on `ctas` CTAs (default: one
// per SM). Same ready / defer / sq_partial contract as umma_tma_gemm (one partial per 128 x BN tile,
// tile = row band * ceil(N / BN) + column tile).
int umma_persist_gemm(const float* A, int64_t lda, const float* B, int64_t ldb, float* C, int64_t ldc, int M, int N,
                      int K, int accumulate, cudaStream_t st, double* sq_partial, const int* ready, int ready_rows,
                      const int* progress, int* defer, int ctas, int bn, int* ticket) {
  APX_REQUIRE(ready == nullptr || (accumulate && ready_rows > 0), "umma_persist_gemm: ready flags need accumulate");
  APX_REQUIRE(defer == nullptr || (ready != nullptr && progress != nullptr && sq_partial != nullptr),
              "umma_persist_gemm: deferral needs ready flags, a progress counter and sq partials");
  APX_REQUIRE(((uintptr_t)A % 16) == 0 && ((uintptr_t)B % 16) == 0 && ((uintptr_t)C % 16) == 0 && (lda % 4) == 0 &&
                  (ldb % 4) == 0 && (ldc % 4) == 0 && (N % 32) == 0 && K >= 1,
              "umma_persist_gemm: 16-byte aligned operands and N %% 32 == 0 required");
  if (ctas <= 0) ctas = device_sms();
  if (bn == 64)
    return accumulate ? tma::launch_persist<64, true>(A, lda, B, ldb, C, ldc, M, N, K, sq_partial, ready, ready_rows,
                                                      progress, defer, ctas, ticket, st)
                      : tma::launch_persist<64, false>(A, lda, B, ldb, C, ldc, M, N, K, sq_partial, ready,
                                                       ready_rows, progress, defer, ctas, ticket, st);
  return accumulate ? tma::launch_persist<128, true>(A, lda, B, ldb, C, ldc, M, N, K, sq_partial, ready, ready_rows,
                                                     progress, defer, ctas, ticket, st)
                    : tma::launch_persist<128, false>(A, lda, B, ldb, C, ldc, M, N, K, sq_partial, ready, ready_rows,
                                                      progress, defer, ctas, ticket, st);
}

}  // namespace apx
