// Shared device/host helpers for libzob200.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

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

}  // namespace zo
