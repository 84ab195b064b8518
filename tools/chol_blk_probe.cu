// Per-phase cycles of cholinv_blk (linalg.cu) and the launch times of the Cholesky-inverse kernels
// on a random SPD 64 x 64 matrix. Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3
// -std=c++17 -Ipaper_2504_19308_b200/csrc tools/chol_blk_probe.cu -o tools/chol_blk_probe
// -Lpaper_2504_19308_b200 -l:_apx.so -Xlinker -rpath=$PWD/paper_2504_19308_b200
#include <cstdio>
__device__ long long g_stamp[16];
#define APX_CHOL_STAMP(i) \
  if (threadIdx.x == 0 && blockIdx.x == 0) g_stamp[i] = clock64();
__device__ unsigned long long g_qstamp[8];
#define APX_CQR_STAMP(i)                                  \
  if (threadIdx.x == 0 && blockIdx.x == 0) {               \
    unsigned long long t_;                                 \
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_)); \
    g_qstamp[i] = t_;                                      \
  }
#include "linalg.cu"
using namespace apx;

int main() {
  const int l = 64;
  double hG[64 * 64], hA[64 * 200];
  srand(7);
  for (int i = 0; i < 64 * 200; ++i) hA[i] = rand() / (double)RAND_MAX - 0.5;
  for (int i = 0; i < l; ++i)
    for (int j = 0; j < l; ++j) {
      double s = 0;
      for (int k = 0; k < 200; ++k) s += hA[i * 200 + k] * hA[j * 200 + k];
      hG[i * l + j] = s;
    }
  double *G, *X;
  int* flags;
  cudaMalloc(&G, sizeof(hG));
  cudaMalloc(&X, sizeof(hG));
  cudaMalloc(&flags, 16);
  cudaMemcpy(G, hG, sizeof(hG), cudaMemcpyHostToDevice);
  cudaMemset(flags, 0, 16);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaFuncSetAttribute(cholinv_blk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kCholBlkSmem);
  const size_t fsm = (size_t)64 * 128 * sizeof(double);
  cudaFuncSetAttribute(cholinv64f_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fsm);
  for (int v = 0; v < 2; ++v) {
    for (int w = 0; w < 3; ++w) {
      if (v == 0) cholinv_blk_kernel<<<1, 256, kCholBlkSmem>>>(G, l, X, flags, flags + 1, flags + 2, 3e4);
      else cholinv64f_kernel<<<1, 256, fsm>>>(G, l, X, flags, flags + 1, flags + 2, 3e4);
    }
    cudaEventRecord(a);
    for (int w = 0; w < 20; ++w) {
      if (v == 0) cholinv_blk_kernel<<<1, 256, kCholBlkSmem>>>(G, l, X, flags, flags + 1, flags + 2, 3e4);
      else cholinv64f_kernel<<<1, 256, fsm>>>(G, l, X, flags, flags + 1, flags + 2, 3e4);
    }
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    double hX[64 * 64];
    cudaMemcpy(hX, X, sizeof(hX), cudaMemcpyDeviceToHost);
    // check X^T G X = I (X = R^{-1}, G = R^T R)
    double err = 0;
    for (int i = 0; i < l; ++i)
      for (int j = 0; j < l; ++j) {
        double s = 0;
        for (int p = 0; p < l; ++p)
          for (int q = 0; q < l; ++q) s += hX[p * l + i] * hG[p * l + q] * hX[q * l + j];
        err = fmax(err, fabs(s - (i == j)));
      }
    printf("%s: %.2f us per launch, max |X^T G X - I| = %.3e\n", v == 0 ? "cholinv_blk" : "cholinv64f", ms * 1000 / 20,
           err);
  }
  long long st[16];
  cudaMemcpyFromSymbol(st, g_stamp, sizeof(st));
  printf("cholinv_blk phase cycles (load, then per block: diag, T/Mb, update):");
  for (int i = 1; i < 13; ++i) printf(" %lld", st[i] - st[i - 1]);
  printf("\n");
  // the fused CholeskyQR2 on a random 8192 x 64 fp32 sketch (pass 2 skipped: well conditioned)
  {
    const int m = 8192, ll = 64, parts = m / 64;
    float* hY = (float*)malloc(sizeof(float) * m * ll);
    for (int i = 0; i < m * ll; ++i) hY[i] = rand() / (float)RAND_MAX - 0.5f;
    float *Yd, *Qd;
    double *p1, *p2, *g1, *g2;
    int* fl;
    cudaMalloc(&Yd, sizeof(float) * m * ll);
    cudaMalloc(&Qd, sizeof(float) * m * ll);
    cudaMalloc(&p1, sizeof(double) * parts * ll * ll);
    cudaMalloc(&p2, sizeof(double) * parts * ll * ll);
    cudaMalloc(&g1, sizeof(double) * ll * ll);
    cudaMalloc(&g2, sizeof(double) * ll * ll);
    cudaMalloc(&fl, 16);
    cudaMemcpy(Yd, hY, sizeof(float) * m * ll, cudaMemcpyHostToDevice);
    cudaFuncSetAttribute(cqr2_fused_kernel<float, float, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(CqrSmem<1>));
    float best = 1e9;
    for (int it = 0; it < 10; ++it) {
      cudaMemset(fl, 0, 16);
      cudaEventRecord(a);
      cqr2_fused_kernel<float, float, 1><<<parts, 256, sizeof(CqrSmem<1>)>>>(Yd, ll, 1, m, ll, p1, p2, g1, g2, fl, Qd, ll, 1,
                                                                (float*)nullptr, 0, 0, 1, 3e4);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      best = fminf(best, ms);
    }
    unsigned long long qs[8];
    cudaMemcpyFromSymbol(qs, g_qstamp, sizeof(qs));
    int hq[4];
    cudaMemcpy(hq, fl, 16, cudaMemcpyDeviceToHost);
    printf("fused QR 8192x64: %.2f us (best of 10), flags %d %d; CTA 0 phases (ns): load %llu gram %llu barrier %llu "
           "reduce %llu barrier %llu cholinv %llu apply %llu (%s)\n",
           best * 1000, hq[0], hq[1], qs[1] - qs[0], qs[2] - qs[1], qs[3] - qs[2], qs[4] - qs[3], qs[5] - qs[4],
           qs[6] - qs[5], qs[7] - qs[6], cudaGetErrorString(cudaGetLastError()));
  }
  int hf[4];
  cudaMemcpy(hf, flags, 16, cudaMemcpyDeviceToHost);
  printf("flags %d %d %d\n", hf[0], hf[1], hf[2]);
  return 0;
}
