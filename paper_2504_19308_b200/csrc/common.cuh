// Shared helpers for the apx (approximate-product) sm_100a kernels.
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdlib>
#include <utility>
#include <cstdio>
#include <cstring>
#include <string>
#include <algorithm>
#include <type_traits>

#include <nvtx3/nvToolsExt.h>

namespace apx {

// NVTX range over a C-ABI call (SURVEY.md §5 tracing): host-side push/pop around the enqueue of a
// product's kernels, visible in Nsight Systems / ncu --nvtx timelines; header-only NVTX3, a no-op
// unless a tool injects itself.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};
#define APX_NVTX(name) ::apx::NvtxRange apx_nvtx_range_(name)

// Grid-shape constant: the B200's SM count, used to size reduction grids, split-K factors and
// partial-sum buffers. Results (fixed-order sums) depend on these shapes, so they are a constant,
// not a device query: the same inputs give the same bits on any device. Grids whose correctness
// or progress depends on how many CTAs are co-resident (the persistent gather) use
// device_sms() instead.
constexpr int kNumSMs = 148;

// Multiprocessor count of the current device (queried once per device).
inline int device_sms() {
  static int cache[64] = {0};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return kNumSMs;
  if (cache[dev] == 0) {
    int v = 0;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0) v = kNumSMs;
    cache[dev] = v;
  }
  return cache[dev];
}

// Device-side bounds checks of the checked build (APX_CHECKED=1 python -m
// paper_2504_19308_b200.build -> _apx_checked.so, selected with APX_LIB): a failed check prints the
// condition and location and traps, so the calling test fails loudly. compute-sanitizer is closed
// on this pool; these checks on the index computations of the main kernels, run over small cases
// of every path (tools/sanitize_cases.py) and the parity tests, stand in for memcheck.
#ifdef APX_CHECKED
#define APX_DCHECK(cond)                                                                            \
  do {                                                                                              \
    if (!(cond)) {                                                                                  \
      printf("APX_DCHECK failed: %s at %s:%d (block %d,%d thread %d)\n", #cond, __FILE__, __LINE__, \
             (int)blockIdx.x, (int)blockIdx.y, (int)threadIdx.x);                                  \
      __trap();                                                                                     \
    }                                                                                               \
  } while (0)
#else
#define APX_DCHECK(cond) \
  do {                   \
  } while (0)
#endif

// dtype codes used across the C-ABI (include/apx.h)
enum DType : int { F32 = 0, F64 = 1, C64 = 2, C128 = 3 };

// error codes returned by every C-ABI entry point
enum Err : int {
  OK = 0,
  E_ARG = 1,       // precondition violated (maps to ValueError in the Python shim)
  E_CUDA = 2,      // CUDA runtime error
  E_WS = 3,        // workspace too small
  E_NUMERIC = 4,   // numerical breakdown the caller must handle
  E_UNSUPPORTED = 5
};

void set_error(const char* fmt, ...);
void count_launch();
// Records the i-th stage-boundary event on `st` when the caller armed them (apx_set_stage_events).
void stage_mark(int i, cudaStream_t st);

#define APX_CUDA(expr)                                                                 \
  do {                                                                                  \
    cudaError_t _e = (expr);                                                            \
    if (_e != cudaSuccess) {                                                            \
      ::apx::set_error("%s:%d %s: %s", __FILE__, __LINE__, #expr, cudaGetErrorString(_e)); \
      return ::apx::E_CUDA;                                                             \
    }                                                                                   \
  } while (0)

#define APX_LAUNCH_CHECK()                                                               \
  do {                                                                                  \
    ::apx::count_launch();                                                              \
    cudaError_t _e = cudaGetLastError();                                                \
    if (_e != cudaSuccess) {                                                            \
      ::apx::set_error("%s:%d launch: %s", __FILE__, __LINE__, cudaGetErrorString(_e)); \
      return ::apx::E_CUDA;                                                             \
    }                                                                                   \
  } while (0)

// Programmatic dependent launch: a kernel launched with launch_pdl may start while the previous
// kernel of its stream is still running; it must call pdl_wait() before touching anything that
// kernel writes (griddepcontrol.wait returns once the previous grid has completed and its memory
// is visible; it is a no-op for a normal launch). pdl_trigger() in the previous kernel lets the
// dependent grid launch early. APX_NO_PDL=1 falls back to ordinary launches (A/B measurements).
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

inline bool pdl_enabled() {
  static const bool on = [] {
    const char* e = getenv("APX_NO_PDL");
    return !(e && atoi(e) != 0);
  }();
  return on;
}

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  // inside a CUDA-graph capture (batch.GraphBatch: many independent products on concurrent
  // streams) launch gaps are already gone, and early-launched dependents would hold SM slots the
  // other products' kernels need (C1 batched: 8.3k vs 10.1k products/s), so capture uses plain edges
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  const bool capturing = cudaStreamIsCapturing(st, &cap) == cudaSuccess && cap != cudaStreamCaptureStatusNone;
  cfg.numAttrs = (pdl_enabled() && !capturing) ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

#define APX_REQUIRE(cond, ...)          \
  do {                                  \
    if (!(cond)) {                      \
      ::apx::set_error(__VA_ARGS__);    \
      return ::apx::E_ARG;              \
    }                                   \
  } while (0)

#define APX_TRY(expr)            \
  do {                           \
    int _r = (expr);             \
    if (_r != ::apx::OK) return _r; \
  } while (0)

// Bump allocator over the caller-owned workspace (no allocation inside the library).
struct Workspace {
  char* base;
  size_t cap;
  size_t off = 0;
  bool dry;  // size-query mode: base may be null
  Workspace(void* b, size_t c, bool d = false) : base((char*)b), cap(c), dry(d) {}
  template <typename T>
  T* take(size_t count) {
    size_t a = (off + 255) & ~size_t(255);
    off = a + count * sizeof(T);
    if (dry) return nullptr;
    return (T*)(base + a);
  }
  bool ok() const { return dry || off <= cap; }
};

#define APX_WS_CHECK(ws)                                                                 \
  do {                                                                                  \
    if (!(ws).ok()) {                                                                   \
      ::apx::set_error("workspace too small: need %zu bytes, have %zu", (ws).off, (ws).cap); \
      return ::apx::E_WS;                                                               \
    }                                                                                   \
  } while (0)

__host__ __device__ inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

__device__ __forceinline__ int wrap_mod(int64_t v, int64_t n) {
  int64_t r = v % n;
  return (int)(r < 0 ? r + n : r);
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Deterministic block sum (fixed tree); result valid in thread 0. `sh` holds >= 32 entries.
template <typename T>
__device__ __forceinline__ T block_sum(T v, T* sh) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) sh[w] = v;
  __syncthreads();
  T r = 0;
  if (w == 0) {
    int nw = (blockDim.x + 31) >> 5;
    r = lane < nw ? sh[lane] : T(0);
    r = warp_sum(r);
  }
  return r;
}

// ---- scaled f16 storage of the mixed product's residual term (see mixed_f16.cu) ---------------
// Binary exponent e with ||X||_F < 2^e (fro2 = ||X||_F^2): scaling X by 2^(15 - e) keeps every
// entry below 2^15 < 65504 (|x_ij| <= ||X||_F), so no value can overflow f16. Zero or non-finite
// norms give e = 0; e is clamped so the fp32 scale factors stay normal.
__host__ __device__ inline int f16_scale_exp(double fro2) {
  if (!(fro2 > 0.0) || !(fro2 < 1e300)) return 0;
  int e = 0;
  frexp(sqrt(fro2), &e);
  return e < -100 ? -100 : (e > 140 ? 140 : e);
}
// two floats -> packed f16x2, round to nearest even (lo in bits 0..15)
__device__ __forceinline__ uint32_t pack_half2(float lo, float hi) {
  uint32_t d;
  asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(d) : "f"(hi), "f"(lo));
  return d;
}

}  // namespace apx
