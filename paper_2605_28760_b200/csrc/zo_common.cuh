// Shared device/host helpers for libzob200.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <utility>

#include "../../include/zob200.h"

namespace zo {

// Error codes: the ZO_OK / ZO_ERR_* macros of the C ABI (include/zob200.h).

#define ZO_CUDA_TRY(expr)                                                             \
  do {                                                                                \
    cudaError_t _e = (expr);                                                          \
    if (_e != cudaSuccess) {                                                          \
      throw ::zo::Error(ZO_ERR_CUDA, std::string(#expr " failed: ") +           \
                                               cudaGetErrorString(_e) + " at " +      \
                                               __FILE__ + ":" + std::to_string(__LINE__)); \
    }                                                                                 \
  } while (0)

struct Error {
  int code;
  std::string msg;
  Error(int c, std::string m) : code(c), msg(std::move(m)) {}
};

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// ---------------------------------------------------------------- programmatic dependent launch
// The per-layer kernels of the scorer (GEMMs, LN, attention, extension finalize) are
// launched with programmatic stream serialization: each one lets its successor begin
// launching as soon as all of its own CTAs are resident (pdl_launch_dependents at the
// top), and waits for its predecessor's completion + memory flush (pdl_wait) before
// touching data the predecessor wrote -- so a kernel's launch and prologue (barrier
// init, TMEM alloc, descriptor prefetch) overlap the previous kernel's tail.
// Both are no-ops for an ordinary launch.
__device__ __forceinline__ void pdl_launch_dependents() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

bool pdl_enabled();  // ZO_PDL=0 disables (zob200.cu)

template <typename... KArgs, typename... Args>
inline void launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
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
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  ZO_CUDA_TRY(cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...));
}

}  // namespace zo
