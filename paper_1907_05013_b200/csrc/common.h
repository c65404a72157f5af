// common.h -- error plumbing shared by the host side of libpooch.
#pragma once
#include <cuda_runtime.h>

#include <cstdarg>
#include <cstdio>
#include <string>

#include "../../include/pooch.h"

namespace pooch {

// Kernel launches issued by the library (process-wide; read per step by the executor).
long long& launch_counter();
inline void count_launch() { ++launch_counter(); }

// Last error of calls made without a context (and the fallback for context calls).
std::string& tls_error();

inline pooch_status fail(pooch_status st, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  tls_error() = buf;
  return st;
}

#define POOCH_CUDA(expr)                                                                     \
  do {                                                                                       \
    cudaError_t e_ = (expr);                                                                 \
    if (e_ != cudaSuccess)                                                                   \
      return ::pooch::fail(POOCH_ECUDA, "%s:%d %s: %s", __FILE__, __LINE__, #expr,            \
                           cudaGetErrorString(e_));                                          \
  } while (0)

#define POOCH_CHECK(st)                 \
  do {                                  \
    pooch_status s_ = (st);             \
    if (s_ != POOCH_OK) return s_;      \
  } while (0)

}  // namespace pooch
