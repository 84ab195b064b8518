// Per-pivot cycles of the one-warp 16 x 16 elimination in cholinv_blk (linalg.cu) and stripped
// variants (VAR 0 full, 1 no reciprocal, 2 no FMA update, 3 no shared publish: shuffles instead,
// 4 dependent DFMA chain of 64, 5 rcp.approx.f64 + 2 Newton steps chained 16 times).
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ double fast_rcp(double x) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  double e = fma(-x, y, 1.0);
  y = fma(y, e, y);
  e = fma(-x, y, 1.0);
  return fma(y, e, y);
}
template <int VAR>
__global__ void probe(const double* A, double* out, long long* cyc) {
  __shared__ __align__(16) double rowbuf[16][32];
  const int lane = threadIdx.x, li = lane & 15, half = lane >> 4;
  double v[16];
#pragma unroll
  for (int c = 0; c < 16; ++c) v[c] = half == 0 ? A[li * 16 + c] : (c == li ? 1.0 : 0.0);
  __syncwarp();
  long long t0 = clock64();
  if (VAR == 4) {
    double x = v[0];
#pragma unroll
    for (int i = 0; i < 64; ++i) x = fma(x, v[1], v[2]);
    v[0] = x;
  } else if (VAR == 5) {
    double x = v[0] + 1.0;
#pragma unroll
    for (int i = 0; i < 16; ++i) x = fast_rcp(x) + 1.0;
    v[0] = x;
  } else {
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      double piv, f = 0.0;
      if (VAR == 3) {
        piv = __shfl_sync(0xffffffffu, v[j], j);
        const double aji = __shfl_sync(0xffffffffu, v[li], j);  // a_j[li] from lane j (half 0)
        const double inv = fast_rcp(piv);
        f = aji * inv;
        if (li > j) {
#pragma unroll
          for (int c = 0; c < 16; ++c) {
            const double w = __shfl_sync(0xffffffffu, v[c], j + 16 * half);
            v[c] = fma(-f, w, v[c]);
          }
        } else {
#pragma unroll
          for (int c = 0; c < 16; ++c) (void)__shfl_sync(0xffffffffu, v[c], j + 16 * half);
        }
      } else {
        if (li == j) {
#pragma unroll
          for (int c = 0; c < 16; c += 2)
            *reinterpret_cast<double2*>(&rowbuf[j][half * 16 + c]) = make_double2(v[c], v[c + 1]);
        }
        __syncwarp();
        piv = rowbuf[j][j];
        const double inv = VAR == 1 ? piv : fast_rcp(piv);
        if (li > j && VAR != 2) {
          f = rowbuf[j][li] * inv;
          const double* pr = &rowbuf[j][half * 16];
#pragma unroll
          for (int c = 0; c < 16; c += 2) {
            const double2 w = *reinterpret_cast<const double2*>(pr + c);
            v[c] = fma(-f, w.x, v[c]);
            v[c + 1] = fma(-f, w.y, v[c + 1]);
          }
        } else if (VAR == 2 && li > j) {
          v[j + 1 < 16 ? j + 1 : 0] *= inv;
        }
      }
    }
  }
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int c = 0; c < 16; ++c) s += v[c];
  out[lane] = s;
  if (lane == 0) cyc[VAR] = t1 - t0;
}
int main() {
  double h[256];
  for (int i = 0; i < 16; ++i)
    for (int j = 0; j < 16; ++j) h[i * 16 + j] = (i == j ? 20.0 : 0.0) + 1.0 / (1 + i + j);
  double *A, *o;
  long long* c;
  cudaMalloc(&A, sizeof(h));
  cudaMalloc(&o, 32 * 8);
  cudaMalloc(&c, 8 * 8);
  cudaMemcpy(A, h, sizeof(h), cudaMemcpyHostToDevice);
  for (int rep = 0; rep < 2; ++rep) {
    probe<0><<<1, 32>>>(A, o, c);
    probe<1><<<1, 32>>>(A, o, c);
    probe<2><<<1, 32>>>(A, o, c);
    probe<3><<<1, 32>>>(A, o, c);
    probe<4><<<1, 32>>>(A, o, c);
    probe<5><<<1, 32>>>(A, o, c);
  }
  long long hc[8];
  cudaMemcpy(hc, c, sizeof(hc), cudaMemcpyDeviceToHost);
  printf("16 pivots: full %lld, no rcp %lld, no update %lld, shuffles %lld cycles; 64 dependent DFMA %lld; 16 chained rcp %lld\n",
         hc[0], hc[1], hc[2], hc[3], hc[4], hc[5]);
  return 0;
}
