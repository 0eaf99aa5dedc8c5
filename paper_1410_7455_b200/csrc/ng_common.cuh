// ng_common.cuh -- shared plumbing of libngsgd.so: status/error reporting, CUDA checks,
// device error flags, warp/block reductions.  No method arithmetic lives here.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include <cstring>
#include <string>

#include "../../include/ngsgd.h"

namespace ng {

// Thread-local last-error message (ng_last_error).
void set_error(const std::string& msg);
const char* last_error();

#define NG_CUDA_TRY(expr)                                                              \
  do {                                                                                 \
    cudaError_t _e = (expr);                                                           \
    if (_e != cudaSuccess) {                                                           \
      ::ng::set_error(std::string(#expr) + ": " + cudaGetErrorString(_e) + " at " +    \
                      __FILE__ + ":" + std::to_string(__LINE__));                      \
      return NG_ECUDA;                                                                 \
    }                                                                                  \
  } while (0)

#define NG_TRY(expr)                    \
  do {                                  \
    ng_status _s = (expr);              \
    if (_s != NG_OK) return _s;         \
  } while (0)

#define NG_REQUIRE(cond, code, msg)                                \
  do {                                                             \
    if (!(cond)) {                                                 \
      ::ng::set_error(std::string(__func__) + ": " + (msg));       \
      return (code);                                               \
    }                                                              \
  } while (0)

// Sticky device error bits (reported at the next synchronising call).
enum : uint32_t {
  kErrNonFinite = 1u << 0,
  kErrLabel = 1u << 1,
  kErrNotPD = 1u << 2,
};

ng_status status_from_flags(uint32_t flags, const char* where);

// Launch counter (ng_kernel_launches) and per-group CUDA-event timing (ng_profile_*).
void count_launch();
struct ProfScope {
  int group = -1, slot = -1;
  cudaStream_t st = nullptr;
  ProfScope(int group, cudaStream_t st, double flops, double bytes);
  ~ProfScope();
};

// Check the last launch; returns NG_ECUDA with a message on failure.
inline ng_status check_launch(const char* what) {
  count_launch();
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error(std::string("launch of ") + what + " failed: " + cudaGetErrorString(e));
    return NG_ECUDA;
  }
  return NG_OK;
}

// Integer tuning knob from the environment (read by the caller once and cached).
inline int tune_int(const char* name, int def) {
  const char* e = getenv(name);
  return e ? atoi(e) : def;
}

// Programmatic dependent launch (PDL) on the main stream's kernel chain: a kernel launched
// with launch_pdl may be scheduled while its predecessor is still running; it runs its
// prologue (barrier init, TMEM alloc, tensor-map prefetch), then pdl_wait() blocks until the
// predecessor grid has completed and its writes are visible.  Every kernel launched with
// launch_pdl calls pdl_wait() before touching global memory the stream produced; kernels
// call pdl_trigger() early so their successor's prologue overlaps their own work.
// NG_TUNE_PDL=0 turns the attribute off (A/B measurements).
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
inline bool pdl_enabled() {
  static const int v = tune_int("NG_TUNE_PDL", 1);
  return v != 0;
}
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              Args... args) {
  cudaLaunchConfig_t cfg;
  memset(&cfg, 0, sizeof(cfg));
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

inline int64_t round_up(int64_t x, int64_t m) { return (x + m - 1) / m * m; }
inline int ceil_div(int64_t a, int64_t b) { return (int)((a + b - 1) / b); }

// ----------------------------------------------------------------- device helpers

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

template <typename T>
__device__ __forceinline__ T warp_max(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Block-wide sum with a fixed reduction tree (deterministic).  `scratch` needs
// blockDim.x/32 elements.  Result valid in all threads.
template <typename T>
__device__ __forceinline__ T block_sum(T v, T* scratch) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) scratch[wid] = v;
  __syncthreads();
  T r = (lane < nw) ? scratch[lane] : T(0);
  r = warp_sum(r);
  return r;
}

template <typename T>
__device__ __forceinline__ T block_max(T v, T* scratch) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  v = warp_max(v);
  __syncthreads();
  if (lane == 0) scratch[wid] = v;
  __syncthreads();
  T r = (lane < nw) ? scratch[lane] : scratch[0];
  r = warp_max(r);
  return r;
}

}  // namespace ng
