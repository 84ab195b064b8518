// Tensor-core GEMMs for the randomized-SVD contractions (K12/K15 of SURVEY.md §2.3):
//   Y  = A . Omega        (n x n  .  n x l)      -- sketch, big operand streamed once
//   Bm = Q^T . A          (l x n  .  n x n)      -- projection (Q^T given as l x n, K-contiguous)
//   W  = Bm . dB          (l x n  .  n x n)      -- dB = B with the kept cycles masked on load
//   M  = Q . W            (n x l  .  l x n)      -- low-rank part of the mixed product
// All four are C[M x N] = A[M x K] . B[K x N] with A K-contiguous and B N-contiguous.
//
// fp32 path: mma.sync m16n8k8 TF32 with fp32 accumulation (optionally 3xTF32 split for
// fp32-level accuracy); fp64 path: DMMA mma.sync m8n8k4. Operand tiles are staged through a
// 3-stage cp.async ring; split-K writes per-slice partials that a fixed-order reduction sums
// (deterministic, no atomics).
#include "common.cuh"
#include "kernels.cuh"

namespace apx {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

template <int BYTES>
__device__ __forceinline__ void cp_async(void* dst, const void* src, bool pred) {
  const int sz = pred ? BYTES : 0;
  if constexpr (BYTES == 16)
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(smem_u32(dst)), "l"(src), "r"(sz));
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], %2, %3;\n" ::"r"(smem_u32(dst)), "l"(src), "n"(BYTES),
                 "r"(sz));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

__device__ __forceinline__ uint32_t to_tf32(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;\n" : "=r"(r) : "f"(x));
  return r;
}

__device__ __forceinline__ void mma_tf32(float* c, const uint32_t* a, const uint32_t* b) {
  asm volatile(
      "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};\n"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}

__device__ __forceinline__ void mma_f64(double* c, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

// ------------------------------------------------------------------------------------------
// Generic tiled kernel. Template: element type T (float -> TF32 mma, double -> DMMA),
// tile BM x BN x BK, warp grid WM x WN (8 warps), SPLIT3 (3xTF32 for fp32).
// Masking (cycle residual of the B operand): if mJ != nullptr, B[k][c] is treated as 0 when
// (k - c) mod mod_n is one of mJ[0..mk) -- applied to the staged tile before the MMAs.
// ------------------------------------------------------------------------------------------
template <typename T, int BM, int BN, int BK, int WM, int WN, bool SPLIT3>
struct GemmCfg {
  static constexpr int kThreads = WM * WN * 32;
  static constexpr int kStages = 3;
  static constexpr int kPadA = 4;   // row stride BK+pad: 16B-aligned rows, conflict-free fragments
  static constexpr int kPadB = (sizeof(T) == 4) ? 8 : 4;  // (BN+pad) spreads the k rows over banks
  static constexpr int kSA = BK + kPadA;
  static constexpr int kSB = BN + kPadB;
  static constexpr int kTileA = BM * kSA;
  static constexpr int kTileB = BK * kSB;
  static constexpr size_t kSmem = (size_t)kStages * (kTileA + kTileB) * sizeof(T);
  static constexpr int kWarpM = BM / WM, kWarpN = BN / WN;
  static constexpr int kMmaM = sizeof(T) == 4 ? 16 : 8;
  static constexpr int kMmaN = 8;
  static constexpr int kMmaK = sizeof(T) == 4 ? 8 : 4;
  static constexpr int MI = kWarpM / kMmaM, NI = kWarpN / kMmaN;
};

template <typename T, int BM, int BN, int BK, int WM, int WN, bool SPLIT3, bool VEC>
__global__ void __launch_bounds__(WM* WN * 32) gemm_kernel(const T* __restrict__ A, int64_t lda,
                                                           const T* __restrict__ B, int64_t ldb, T* __restrict__ C,
                                                           int64_t ldc, int64_t c_split_stride, int M, int N, int K,
                                                           int k_per_split, int accumulate,
                                                           const int* __restrict__ mJ, int mk, int mod_n) {
  using Cfg = GemmCfg<T, BM, BN, BK, WM, WN, SPLIT3>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* sA = reinterpret_cast<T*>(smem_raw);
  T* sB = sA + Cfg::kStages * Cfg::kTileA;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp / WN, wn = warp % WN;
  const int gid = lane >> 2, tig = lane & 3;
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  const int kz = blockIdx.z;
  const int kbeg = kz * k_per_split, kend = min(K, kbeg + k_per_split);
  const int ktiles = (int)ceil_div(max(0, kend - kbeg), BK);

  constexpr int EV = VEC ? 16 / sizeof(T) : 1;  // elements per async copy
  auto load_tile = [&](int stage, int kt) {
    const int k0 = kbeg + kt * BK;
    T* a = sA + stage * Cfg::kTileA;
    T* b = sB + stage * Cfg::kTileB;
    constexpr int ACH = BM * BK / EV;
    for (int c = tid; c < ACH; c += Cfg::kThreads) {
      const int r = c / (BK / EV), kk = (c % (BK / EV)) * EV;
      const int gm = m0 + r, gk = k0 + kk;
      const bool ok = gm < M && gk < kend;
      const T* src = ok ? A + (size_t)gm * lda + gk : A;
      cp_async<EV * sizeof(T)>(a + r * Cfg::kSA + kk, src, ok);
    }
    constexpr int BCH = BK * BN / EV;
    for (int c = tid; c < BCH; c += Cfg::kThreads) {
      const int r = c / (BN / EV), nn = (c % (BN / EV)) * EV;
      const int gk = k0 + r, gn = n0 + nn;
      const bool ok = gk < kend && gn < N;
      const T* src = ok ? B + (size_t)gk * ldb + gn : B;
      cp_async<EV * sizeof(T)>(b + r * Cfg::kSB + nn, src, ok);
    }
  };

  float accf[Cfg::MI][Cfg::NI][4];
  double accd[Cfg::MI][Cfg::NI][2];
  if constexpr (sizeof(T) == 4) {
#pragma unroll
    for (int i = 0; i < Cfg::MI; ++i)
#pragma unroll
      for (int j = 0; j < Cfg::NI; ++j)
#pragma unroll
        for (int q = 0; q < 4; ++q) accf[i][j][q] = 0.f;
  } else {
#pragma unroll
    for (int i = 0; i < Cfg::MI; ++i)
#pragma unroll
      for (int j = 0; j < Cfg::NI; ++j) accd[i][j][0] = accd[i][j][1] = 0.0;
  }

#pragma unroll
  for (int s = 0; s < Cfg::kStages - 1; ++s) {
    if (s < ktiles) load_tile(s, s);
    cp_async_commit();
  }

  for (int kt = 0; kt < ktiles; ++kt) {
    cp_async_wait<Cfg::kStages - 2>();
    __syncthreads();
    const int stage = kt % Cfg::kStages;
    T* a = sA + stage * Cfg::kTileA;
    T* b = sB + stage * Cfg::kTileB;
    if (mJ != nullptr) {
      const int k0 = kbeg + kt * BK;
      for (int e = tid; e < BK * mk; e += Cfg::kThreads) {
        const int r = e / mk, t = e - r * mk;
        int c = k0 + r - mJ[t];  // k0 + r < mod_n and 0 <= mJ[t] < mod_n
        if (c < 0) c += mod_n;
        if (c >= n0 && c < n0 + BN) b[r * Cfg::kSB + (c - n0)] = T(0);
      }
      __syncthreads();
    }
    // prefetch the tile STAGES-1 ahead (its slot was consumed in iteration kt-1)
    {
      const int nk = kt + Cfg::kStages - 1;
      if (nk < ktiles) load_tile(nk % Cfg::kStages, nk);
      cp_async_commit();
    }
#pragma unroll
    for (int kk = 0; kk < BK; kk += Cfg::kMmaK) {
      if constexpr (sizeof(T) == 4) {
        uint32_t af[Cfg::MI][4], bf[Cfg::NI][2];
        uint32_t al[Cfg::MI][4], bl[Cfg::NI][2];
#pragma unroll
        for (int i = 0; i < Cfg::MI; ++i) {
          const int r = wm * Cfg::kWarpM + i * 16 + gid;
          const float x0 = a[r * Cfg::kSA + kk + tig], x1 = a[(r + 8) * Cfg::kSA + kk + tig];
          const float x2 = a[r * Cfg::kSA + kk + tig + 4], x3 = a[(r + 8) * Cfg::kSA + kk + tig + 4];
          af[i][0] = to_tf32(x0); af[i][1] = to_tf32(x1); af[i][2] = to_tf32(x2); af[i][3] = to_tf32(x3);
          if constexpr (SPLIT3) {
            al[i][0] = to_tf32(x0 - __uint_as_float(af[i][0]));
            al[i][1] = to_tf32(x1 - __uint_as_float(af[i][1]));
            al[i][2] = to_tf32(x2 - __uint_as_float(af[i][2]));
            al[i][3] = to_tf32(x3 - __uint_as_float(af[i][3]));
          }
        }
#pragma unroll
        for (int j = 0; j < Cfg::NI; ++j) {
          const int c = wn * Cfg::kWarpN + j * 8 + gid;
          const float y0 = b[(kk + tig) * Cfg::kSB + c], y1 = b[(kk + tig + 4) * Cfg::kSB + c];
          bf[j][0] = to_tf32(y0); bf[j][1] = to_tf32(y1);
          if constexpr (SPLIT3) {
            bl[j][0] = to_tf32(y0 - __uint_as_float(bf[j][0]));
            bl[j][1] = to_tf32(y1 - __uint_as_float(bf[j][1]));
          }
        }
#pragma unroll
        for (int i = 0; i < Cfg::MI; ++i)
#pragma unroll
          for (int j = 0; j < Cfg::NI; ++j) {
            if constexpr (SPLIT3) {
              mma_tf32(accf[i][j], al[i], bf[j]);
              mma_tf32(accf[i][j], af[i], bl[j]);
            }
            mma_tf32(accf[i][j], af[i], bf[j]);
          }
      } else {
        double af[Cfg::MI], bfv[Cfg::NI];
#pragma unroll
        for (int i = 0; i < Cfg::MI; ++i) {
          const int r = wm * Cfg::kWarpM + i * 8 + gid;
          af[i] = a[r * Cfg::kSA + kk + tig];
        }
#pragma unroll
        for (int j = 0; j < Cfg::NI; ++j) {
          const int c = wn * Cfg::kWarpN + j * 8 + gid;
          bfv[j] = b[(kk + tig) * Cfg::kSB + c];
        }
#pragma unroll
        for (int i = 0; i < Cfg::MI; ++i)
#pragma unroll
          for (int j = 0; j < Cfg::NI; ++j) mma_f64(accd[i][j], af[i], bfv[j]);
      }
    }
  }
  cp_async_wait<0>();

  // epilogue
  T* Cz = C + (size_t)kz * c_split_stride;
#pragma unroll
  for (int i = 0; i < Cfg::MI; ++i)
#pragma unroll
    for (int j = 0; j < Cfg::NI; ++j) {
      const int cb = n0 + wn * Cfg::kWarpN + j * 8 + 2 * tig;
      if constexpr (sizeof(T) == 4) {
        const int rb = m0 + wm * Cfg::kWarpM + i * 16 + gid;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int r = rb + 8 * h;
          if (r >= M) continue;
          T* p = Cz + (size_t)r * ldc + cb;
          float v0 = accf[i][j][2 * h], v1 = accf[i][j][2 * h + 1];
          if (accumulate) {
            if (cb < N) v0 += p[0];
            if (cb + 1 < N) v1 += p[1];
          }
          if (cb + 1 < N && ((((uintptr_t)p) & 7) == 0)) {
            *reinterpret_cast<float2*>(p) = make_float2(v0, v1);
          } else {
            if (cb < N) p[0] = v0;
            if (cb + 1 < N) p[1] = v1;
          }
        }
      } else {
        const int r = m0 + wm * Cfg::kWarpM + i * 8 + gid;
        if (r >= M) continue;
        T* p = Cz + (size_t)r * ldc + cb;
        double v0 = accd[i][j][0], v1 = accd[i][j][1];
        if (accumulate) {
          if (cb < N) v0 += p[0];
          if (cb + 1 < N) v1 += p[1];
        }
        if (cb < N) p[0] = v0;
        if (cb + 1 < N) p[1] = v1;
      }
    }
}

// out[e] = sum_z part[z][e] (fixed order), e < count; optionally converts to double.
template <typename T, typename O>
__global__ void split_reduce_kernel(const T* __restrict__ part, int splits, size_t count, O* __restrict__ out) {
  for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < count; e += (size_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int z = 0; z < splits; ++z) s += (double)part[(size_t)z * count + e];
    out[e] = (O)s;
  }
}

template <typename T, int BM, int BN, int BK, int WM, int WN, bool SPLIT3>
static int gemm_launch(const T* A, int64_t lda, const T* B, int64_t ldb, T* C, int64_t ldc, int M, int N, int K,
                       int splits, int accumulate, const int* mJ, int mk, int mod_n, cudaStream_t st) {
  using Cfg = GemmCfg<T, BM, BN, BK, WM, WN, SPLIT3>;
  const bool vec = (lda * sizeof(T)) % 16 == 0 && (ldb * sizeof(T)) % 16 == 0 && ((uintptr_t)A % 16) == 0 &&
                   ((uintptr_t)B % 16) == 0;
  const int kps = (int)(ceil_div(ceil_div(K, splits), BK) * BK);
  dim3 grid((unsigned)ceil_div(N, BN), (unsigned)ceil_div(M, BM), (unsigned)splits);
  const size_t cstride = (size_t)M * ldc;
  if (vec) {
    auto fn = gemm_kernel<T, BM, BN, BK, WM, WN, SPLIT3, true>;
    APX_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Cfg::kSmem));
    fn<<<grid, Cfg::kThreads, Cfg::kSmem, st>>>(A, lda, B, ldb, C, ldc, cstride, M, N, K, kps, accumulate, mJ, mk,
                                                mod_n);
  } else {
    auto fn = gemm_kernel<T, BM, BN, BK, WM, WN, SPLIT3, false>;
    APX_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Cfg::kSmem));
    fn<<<grid, Cfg::kThreads, Cfg::kSmem, st>>>(A, lda, B, ldb, C, ldc, cstride, M, N, K, kps, accumulate, mJ, mk,
                                                mod_n);
  }
  APX_LAUNCH_CHECK();
  return OK;
}

// Number of K-splits so that tall/wide skinny GEMMs put >= ~2 CTAs on every SM.
int gemm_splits(int M, int N, int K, int BM, int BN) {
  const int64_t tiles = ceil_div(M, BM) * ceil_div(N, BN);
  int s = (int)std::max<int64_t>(1, ceil_div(2 * kNumSMs, tiles));
  s = std::min<int>(s, std::max<int>(1, (int)(K / 256)));
  return s;
}

// C = A . B for the skinny rSVD shapes. kind: 0 = tall output (N small, e.g. A.Omega),
// 1 = wide output (M small, e.g. Q^T.A / Bm.dB), 2 = outer (K small, e.g. Q.W).
// part: split-K scratch (splits * M * N elements) or nullptr when splits == 1.
template <typename T>
int gemm_skinny(int kind, const T* A, int64_t lda, const T* B, int64_t ldb, T* C, int64_t ldc, int M, int N, int K,
                int accumulate, const int* mJ, int mk, int mod_n, T* part, int splits, bool split3, cudaStream_t st) {
  if (M <= 0 || N <= 0) return OK;
  T* dst = splits > 1 ? part : C;
  const int64_t ld = splits > 1 ? N : ldc;
  const int acc = splits > 1 ? 0 : accumulate;
  int rc;
  if constexpr (sizeof(T) == 4) {
    if (kind == 0)
      rc = split3 ? gemm_launch<T, 128, 64, 32, 4, 2, true>(A, lda, B, ldb, dst, ld, M, N, K, splits, acc, mJ, mk, mod_n, st)
                  : gemm_launch<T, 128, 64, 32, 4, 2, false>(A, lda, B, ldb, dst, ld, M, N, K, splits, acc, mJ, mk, mod_n, st);
    else if (kind == 1)
      rc = split3 ? gemm_launch<T, 64, 128, 32, 2, 4, true>(A, lda, B, ldb, dst, ld, M, N, K, splits, acc, mJ, mk, mod_n, st)
                  : gemm_launch<T, 64, 128, 32, 2, 4, false>(A, lda, B, ldb, dst, ld, M, N, K, splits, acc, mJ, mk, mod_n, st);
    else
      rc = split3 ? gemm_launch<T, 128, 128, 32, 4, 2, true>(A, lda, B, ldb, dst, ld, M, N, K, splits, acc, mJ, mk, mod_n, st)
                  : gemm_launch<T, 128, 128, 32, 4, 2, false>(A, lda, B, ldb, dst, ld, M, N, K, splits, acc, mJ, mk, mod_n, st);
  } else {
    if (kind == 0)
      rc = gemm_launch<T, 64, 64, 16, 4, 2, false>(A, lda, B, ldb, dst, ld, M, N, K, splits, acc, mJ, mk, mod_n, st);
    else if (kind == 1)
      rc = gemm_launch<T, 64, 64, 16, 2, 4, false>(A, lda, B, ldb, dst, ld, M, N, K, splits, acc, mJ, mk, mod_n, st);
    else
      rc = gemm_launch<T, 64, 64, 16, 4, 2, false>(A, lda, B, ldb, dst, ld, M, N, K, splits, acc, mJ, mk, mod_n, st);
  }
  if (rc != OK) return rc;
  if (splits > 1) {
    // fixed-order reduction of the partial slices into C (row-major, ldc == N required here)
    if (accumulate || ldc != N) {
      set_error("gemm_skinny: split-K needs a dense, non-accumulating destination");
      return E_ARG;
    }
    const size_t cnt = (size_t)M * N;
    split_reduce_kernel<T, T><<<(unsigned)std::min<int64_t>(ceil_div(cnt, 256), kNumSMs * 8), 256, 0, st>>>(
        part, splits, cnt, C);
    APX_LAUNCH_CHECK();
  }
  return OK;
}

int launch_split_reduce_f32(const float* part, int splits, size_t count, float* out, cudaStream_t st) {
  split_reduce_kernel<float, float><<<(unsigned)std::min<int64_t>(ceil_div(count, 256), kNumSMs * 8), 256, 0, st>>>(
      part, splits, count, out);
  APX_LAUNCH_CHECK();
  return OK;
}

template int gemm_skinny<float>(int, const float*, int64_t, const float*, int64_t, float*, int64_t, int, int, int,
                                int, const int*, int, int, float*, int, bool, cudaStream_t);
template int gemm_skinny<double>(int, const double*, int64_t, const double*, int64_t, double*, int64_t, int, int,
                                 int, int, const int*, int, int, double*, int, bool, cudaStream_t);

}  // namespace apx
