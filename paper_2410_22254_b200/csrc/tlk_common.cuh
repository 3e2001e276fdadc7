// Shared host-side helpers of libtlk: thread-local error text, CUDA checks.
#pragma once
#include <cstdarg>
#include <cstdio>
#include <string>

#include <cuda_runtime.h>

#include "../../include/tlk.h"

namespace tlk {

void set_error(const char* fmt, ...);
int fail(int code, const char* fmt, ...);
int cuda_fail(cudaError_t e, const char* what);

}  // namespace tlk

#define TLK_CUDA(call)                                      \
  do {                                                      \
    cudaError_t e_ = (call);                                \
    if (e_ != cudaSuccess) return ::tlk::cuda_fail(e_, #call); \
  } while (0)

#define TLK_CHECK(cond, code, ...)                 \
  do {                                             \
    if (!(cond)) return ::tlk::fail(code, __VA_ARGS__); \
  } while (0)
