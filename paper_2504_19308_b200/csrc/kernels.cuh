// Host-side launcher declarations shared by the C-ABI translation unit.
#pragma once
#include "common.cuh"

namespace apx {

// ---- cycle.cu ----
size_t cycle_energy_ws(int n);
int right_gather_rows(int n, size_t elem);
template <typename T>
int launch_cycle_energies(const T* A, int n, double* energies, double* norms, double* fro2, double* partial,
                          cudaStream_t st);
int launch_topk(const double* w, int n, int k, int* sel, cudaStream_t st);
int launch_kept_energy(const double* norms, const int* sel, int k, double scale, double* out, cudaStream_t st);
template <typename T>
int launch_cycle_extract(const T* A, int n, const int* J, int k, T* lam, cudaStream_t st);
template <typename T>
int launch_cycle_materialize(const T* lam, const int* J, int k, int n, T* out, cudaStream_t st);
template <typename T>
int launch_cycle_left_gather(const T* X, const T* lam, const int* J, int k, int n, int accumulate, T* M,
                             cudaStream_t st);
template <typename T>
int launch_cycle_right_gather(const T* X, const int* JA, int ka, const T* lam, const int* J, int k, int n,
                              int accumulate, T* M, double* msq_partial, cudaStream_t st);
template <typename T>
int launch_sumsq(const T* x, size_t cnt, double* partial, int* nparts, cudaStream_t st);
int launch_sum_vector(const double* v, int n, double* out, cudaStream_t st);

}  // namespace apx
