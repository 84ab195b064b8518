// Small dense SVD for the randomized SVD (K14; reference svd.py:113 -> LAPACK gesdd).
//
// One CTA runs one-sided (Hestenes) Jacobi on a square l x l matrix W held column-major in
// shared memory (l <= 128) or, for wider sketches, in a global (L2-resident) scratch buffer:
// W V' = U' S. Rounds of the circle tournament rotate l/2
// disjoint column pairs in parallel (one half-warp per pair, lanes over rows, fp64), sweeps repeat
// until no pair is rotated. Singular values come out as column norms, sorted descending (stable
// on ties); columns with zero norm are completed to an orthonormal basis by Gram-Schmidt on unit
// vectors, so U' is orthonormal even for rank-deficient inputs (zero / rank-1 test matrices,
// test_svd.py:56-77), where a Gram-matrix eigensolver would lose the tiny singular values.
#include "common.cuh"
#include "kernels.cuh"

namespace apx {

constexpr int kSvdMax = 128;
#ifdef APX_CHECKED
constexpr bool getenv_sweeps_debug = true;  // the checked build reports the sweep count
#endif

// fp64 reciprocal / reciprocal square root for positive normal x (MUFU seed + two Newton steps,
// no special-case branches): the rotation angle is on every round's critical path
__device__ __forceinline__ double svd_rcp(double x) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  double e = fma(-x, y, 1.0);
  y = fma(y, e, y);
  e = fma(-x, y, 1.0);
  return fma(y, e, y);
}
__device__ __forceinline__ double svd_rsqrt(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double h = 0.5 * x;
  double e = fma(-h * y, y, 0.5);
  y = fma(y, e, y);
  e = fma(-h * y, y, 0.5);
  return fma(y, e, y);
}

// KR: rows per lane of a pair's half-warp (ceil(l / 16)); the shared-memory kernel is
// instantiated for l <= 32, 48, 64, 128 so a small sketch does not carry zero-padded registers
template <bool GLOBAL, int KR = (kSvdMax + 15) / 16>
__global__ void __launch_bounds__(GLOBAL ? 1024 : 512)
    hestenes_svd_kernel(const double* __restrict__ Win, int l, double* __restrict__ Uout, double* __restrict__ Sout,
                        double* __restrict__ Vout, double* __restrict__ VoutT, double* __restrict__ scratch) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int le = l + (l & 1);  // even number of columns (pad with a zero column)
  // GLOBAL: W, V, the norms, the permutation and the completion vector live in `scratch`
  double* Wc = GLOBAL ? scratch : reinterpret_cast<double*>(smem_raw);  // le columns x l rows, column-major
  double* Vc = Wc + (size_t)le * l;                                      // le x le
  __shared__ int s_rot;
  __shared__ int perm_s[GLOBAL ? 1 : kSvdMax + 2];
  __shared__ double norms_s[GLOBAL ? 1 : kSvdMax + 2];
  int* perm = GLOBAL ? reinterpret_cast<int*>(Vc + (size_t)le * le + le) : perm_s;
  double* norms = GLOBAL ? Vc + (size_t)le * le : norms_s;
  __shared__ double nrm2_s[GLOBAL ? 1 : kSvdMax + 2];
  double* nrm2 = GLOBAL ? norms + 3 * le + 2 + l : nrm2_s;  // GLOBAL: after the completion vector
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  for (int e = tid; e < le * l; e += blockDim.x) {
    const int j = e / l, i = e - j * l;
    Wc[e] = j < l ? Win[i * l + j] : 0.0;
  }
  for (int e = tid; e < le * le; e += blockDim.x) {
    const int j = e / le, i = e - j * le;
    Vc[e] = (i == j) ? 1.0 : 0.0;
  }
  __syncthreads();
  const double eps = 2.220446049250313e-16;
  const double tol2 = (eps * l) * (eps * l);
  for (int sweep = 0; sweep < 60; ++sweep) {
    // squared column norms, exact at the start of every sweep, then carried through the sweep's
    // rotations (||a'||^2 = al - t ga, ||b'||^2 = be + t ga): one dot product per pair instead of three
    for (int j = warp; j < le; j += nw) {
      double q = 0.0;
      if (j < l)
        for (int i = lane; i < l; i += 32) q = fma(Wc[(size_t)j * l + i], Wc[(size_t)j * l + i], q);
      q = warp_sum(q);
      if (lane == 0) nrm2[j] = q;
    }
    if (tid == 0) s_rot = 0;
    __syncthreads();
    for (int round = 0; round < le - 1; ++round) {
      // half-warp per column pair (16 lanes over the rows): up to 2 * nw pairs per pass
      const int half = lane >> 4, hl = lane & 15;
      for (int p0 = 2 * warp; p0 < le / 2; p0 += 2 * nw) {
        const int pr = p0 + half;
        const bool active = pr < le / 2;
        // circle method: position 0 fixed, others rotate
        int a = 0, b = 1;
        if (active) {
          // (x) mod (le - 1) for 0 <= x < 2 (le - 1): one conditional subtract instead of a division
          int xa = pr - 1 + round, xb = le - 2 - pr + round;
          if (xa >= le - 1) xa -= le - 1;
          if (xb >= le - 1) xb -= le - 1;
          a = (pr == 0) ? 0 : 1 + xa;
          b = 1 + xb;
          if (a > b) { const int t = a; a = b; b = t; }
        }
        double* wa = Wc + (size_t)a * l;
        double* wb = Wc + (size_t)b * l;
        double* va = Vc + (size_t)a * le;
        double* vb = Vc + (size_t)b * le;
        // shared-memory kernel (l <= 128): the pair's W and V entries in registers, all loads
        // issued before the reduction; the global-scratch kernel (wide sketches) re-reads them
        constexpr int kR = GLOBAL ? 1 : KR;
        double xw[kR], yw[kR], xv[kR], yv[kR];
        double ga = 0.0;
        // the pair's carried squared norms: loaded ahead of the dot product's reduction
        const double al = active ? nrm2[a] : 0.0, be = active ? nrm2[b] : 0.0;
        if (GLOBAL) {
          if (active)
            for (int i = hl; i < l; i += 16) ga = fma(wa[i], wb[i], ga);
        } else {
#pragma unroll
          for (int u = 0; u < kR; ++u) {
            const int i = hl + 16 * u;
            xw[u] = (active && i < l) ? wa[i] : 0.0;
            yw[u] = (active && i < l) ? wb[i] : 0.0;
            xv[u] = (active && i < le) ? va[i] : 0.0;
            yv[u] = (active && i < le) ? vb[i] : 0.0;
            ga = fma(xw[u], yw[u], ga);
          }
        }
#pragma unroll
        for (int o = 8; o > 0; o >>= 1) ga += __shfl_xor_sync(0xffffffffu, ga, o);
        if (active && ga != 0.0 && ga * ga > tol2 * al * be) {
          // t = tan(theta) = sign(zeta) / (|zeta| + sqrt(1 + zeta^2)), zeta = (be - al) / (2 ga),
          // written as sign(d) g2 / (|d| + hypot(d, g2)) with d = be - al, g2 = 2 ga: three
          // dependent rcp/rsqrt chains instead of four (the rotation is every round's critical path)
          const double d = be - al, g2 = 2.0 * ga;
          const double h2 = fma(d, d, g2 * g2);
          const double hyp = h2 > 1e-290 ? h2 * svd_rsqrt(h2) : hypot(d, g2);  // (squares underflow)
          const double t = (d >= 0.0 ? g2 : -g2) * svd_rcp(fabs(d) + hyp);
          const double c = svd_rsqrt(fma(t, t, 1.0)), sn = c * t;
          if (GLOBAL) {
            for (int i = hl; i < l; i += 16) {
              const double x = wa[i], y = wb[i];
              wa[i] = c * x - sn * y;
              wb[i] = sn * x + c * y;
            }
            for (int i = hl; i < le; i += 16) {
              const double x = va[i], y = vb[i];
              va[i] = c * x - sn * y;
              vb[i] = sn * x + c * y;
            }
          } else {
#pragma unroll
            for (int u = 0; u < kR; ++u) {
              const int i = hl + 16 * u;
              if (i < l) {
                wa[i] = c * xw[u] - sn * yw[u];
                wb[i] = sn * xw[u] + c * yw[u];
              }
              if (i < le) {
                va[i] = c * xv[u] - sn * yv[u];
                vb[i] = sn * xv[u] + c * yv[u];
              }
            }
          }
          if (hl == 0) {
            nrm2[a] = al - t * ga;
            nrm2[b] = be + t * ga;
            s_rot = 1;
          }
        }
      }
      __syncthreads();
    }
#ifdef APX_CHECKED
    if (!s_rot && tid == 0 && getenv_sweeps_debug) printf("hestenes l=%d converged after %d sweeps\n", l, sweep + 1);
#endif
    if (!s_rot) break;
    __syncthreads();
  }
  // column norms, stable descending order
  for (int j = tid; j < l; j += blockDim.x) {
    double s = 0.0;
    for (int i = 0; i < l; ++i) s = fma(Wc[(size_t)j * l + i], Wc[(size_t)j * l + i], s);
    norms[j] = sqrt(s);
  }
  __syncthreads();
  for (int j = tid; j < l; j += blockDim.x) {
    int rank = 0;
    for (int q = 0; q < l; ++q) rank += (norms[q] > norms[j]) || (norms[q] == norms[j] && q < j);
    perm[rank] = j;
  }
  __syncthreads();
  // U' columns = W columns / sigma (zero columns completed below); outputs row-major l x l
  for (int e = tid; e < l * l; e += blockDim.x) {
    const int i = e / l, r = e - i * l;  // row i, output column r
    const int j = perm[r];
    const double sg = norms[j];
    Uout[e] = sg > 0.0 ? Wc[(size_t)j * l + i] / sg : 0.0;
    Vout[e] = Vc[(size_t)j * le + i];
  }
  for (int r = tid; r < l; r += blockDim.x) Sout[r] = norms[perm[r]];
  if (VoutT != nullptr)
    for (int e = tid; e < l * l; e += blockDim.x) {
      const int r = e / l, i = e - r * l;  // V'^T[r][i] = V'[i][r]
      VoutT[e] = Vc[(size_t)perm[r] * le + i];
    }
  __threadfence_block();
  __syncthreads();
  if (tid == 0) {
    // Gram-Schmidt completion of zero columns (rank-deficient input)
    for (int r = 0; r < l; ++r) {
      if (norms[perm[r]] > 0.0) continue;
      for (int cand = 0; cand < l; ++cand) {
        double v_s[GLOBAL ? 1 : kSvdMax];
        double* v = GLOBAL ? norms + 2 * le + 2 : v_s;
        for (int i = 0; i < l; ++i) v[i] = (i == cand) ? 1.0 : 0.0;
        for (int pass = 0; pass < 2; ++pass)
          for (int q = 0; q < l; ++q) {
            if (q == r) continue;
            double d = 0.0;
            for (int i = 0; i < l; ++i) d += Uout[i * l + q] * v[i];
            for (int i = 0; i < l; ++i) v[i] -= d * Uout[i * l + q];
          }
        double nv = 0.0;
        for (int i = 0; i < l; ++i) nv += v[i] * v[i];
        nv = sqrt(nv);
        if (nv > 0.5) {
          for (int i = 0; i < l; ++i) Uout[i * l + r] = v[i] / nv;
          break;
        }
      }
    }
  }
}

size_t small_svd_scratch_doubles(int l) {
  if (l <= kSvdMax) return 0;
  const size_t le = (size_t)l + (l & 1);
  return le * l + le * le + 2 * le + 2 + le + 8 + le + 2;  // W, V, norms, perm, completion vector, nrm2
}

int launch_small_svd(const double* W, int l, double* U, double* S, double* V, double* VT, cudaStream_t st,
                     double* scratch) {
  APX_REQUIRE(l >= 1, "small SVD size %d", l);
  if (l > kSvdMax) {
    APX_REQUIRE(scratch != nullptr, "small SVD of size %d needs a scratch buffer", l);
    hestenes_svd_kernel<true><<<1, 1024, 0, st>>>(W, l, U, S, V, VT, scratch);
    APX_LAUNCH_CHECK();
    return OK;
  }
  const int le = l + (l & 1);
  const size_t smem = ((size_t)le * l + (size_t)le * le) * sizeof(double);
  auto go = [&](auto kern) -> int {
    APX_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    // one half-warp per column pair of a round: ceil(le / 4) warps (a 40-wide sketch: 10 warps, no
    // idle warps in the per-round barrier)
    const int threads = std::min(512, std::max(64, 32 * ((le / 2 + 1) / 2)));
    kern<<<1, threads, smem, st>>>(W, l, U, S, V, VT, nullptr);
    APX_LAUNCH_CHECK();
    return OK;
  };
  if (le <= 32) return go(hestenes_svd_kernel<false, 2>);
  if (le <= 48) return go(hestenes_svd_kernel<false, 3>);
  if (le <= 64) return go(hestenes_svd_kernel<false, 4>);
  return go(hestenes_svd_kernel<false, 8>);
}

// y[i*ldy + j] (+)= alpha * x[i*ldx + j] * (rowscale ? rowscale[i] : 1), i < rows, j < cols
__global__ void axpy2d_kernel(double* __restrict__ y, int64_t ldy, const double* __restrict__ x, int64_t ldx,
                              int rows, int cols, double alpha, const double* __restrict__ rowscale, int overwrite) {
  const size_t total = (size_t)rows * cols;
  for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < total; e += (size_t)gridDim.x * blockDim.x) {
    const int i = (int)(e / cols), j = (int)(e % cols);
    double v = alpha * x[(size_t)i * ldx + j];
    if (rowscale) v *= rowscale[i];
    double* py = y + (size_t)i * ldy + j;
    *py = overwrite ? v : *py + v;
  }
}

int launch_axpy2d(double* y, int64_t ldy, const double* x, int64_t ldx, int rows, int cols, double alpha,
                  const double* rowscale, int overwrite, cudaStream_t st) {
  if (rows <= 0 || cols <= 0) return OK;
  const int blocks = (int)std::min<int64_t>(ceil_div((int64_t)rows * cols, 256), kNumSMs * 8);
  axpy2d_kernel<<<blocks, 256, 0, st>>>(y, ldy, x, ldx, rows, cols, alpha, rowscale, overwrite);
  APX_LAUNCH_CHECK();
  return OK;
}

// out = sum_{i<k} s[i]^2 (single thread, fixed order)
__global__ void sumsq_prefix_kernel(const double* __restrict__ s, int k, double* __restrict__ out) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    double a = 0.0;
    for (int i = 0; i < k; ++i) a += s[i] * s[i];
    *out = a;
  }
}

int launch_sumsq_prefix(const double* s, int k, double* out, cudaStream_t st) {
  sumsq_prefix_kernel<<<1, 32, 0, st>>>(s, k, out);
  APX_LAUNCH_CHECK();
  return OK;
}

}  // namespace apx
