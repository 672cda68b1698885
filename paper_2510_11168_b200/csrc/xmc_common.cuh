// Host-side helpers shared by the translation units of libxmc_b200.so:
// thread-local error message + status-returning macros (xmc_head.h error
// convention), small integer helpers and per-device scratch.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "../../include/xmc_head.h"

// Record a message for xmc_last_error() and return s (defined in xmc_api.cu).
xmc_status xmc_fail(xmc_status s, const char* fmt, ...);

#define CUDA_TRY(expr)                                                                     \
  do {                                                                                     \
    cudaError_t e_ = (expr);                                                               \
    if (e_ != cudaSuccess)                                                                 \
      return xmc_fail(XMC_ERR_CUDA, "%s failed: %s (%s:%d)", #expr, cudaGetErrorString(e_), \
                      __FILE__, __LINE__);                                                 \
  } while (0)

#define XMC_TRY(expr)              \
  do {                             \
    xmc_status s_ = (expr);        \
    if (s_ != XMC_OK) return s_;   \
  } while (0)

static inline int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }
static inline size_t align_up(size_t a, size_t b) { return (a + b - 1) / b * b; }

// A 64-byte device status scratch of the CURRENT device (one per device, made
// on first use) for the elementwise entry points that own no handle.
int32_t* xmc_device_scratch_status();
