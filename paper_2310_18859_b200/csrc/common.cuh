// Shared helpers of the sm_100a SiDA library: status plumbing and small
// device utilities. Every exported entry point returns a SIDA_* status and
// records a thread-local message (see sida_b200.h).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include "../../include/sida_b200.h"

namespace sida {

void set_error(const char* fmt, ...);
// Process-wide count of this library's kernel launches (sida_launch_count).
void count_launch();

// Return-on-failure helpers for the extern "C" wrappers.
#define SIDA_REQUIRE(cond, code, ...)        \
  do {                                       \
    if (!(cond)) {                           \
      ::sida::set_error(__VA_ARGS__);        \
      return (code);                         \
    }                                        \
  } while (0)

#define SIDA_CUDA(expr)                                                            \
  do {                                                                             \
    cudaError_t _e = (expr);                                                       \
    if (_e != cudaSuccess) {                                                       \
      ::sida::set_error("%s failed: %s (%s:%d)", #expr, cudaGetErrorString(_e),    \
                        __FILE__, __LINE__);                                       \
      return SIDA_ERR_CUDA;                                                        \
    }                                                                              \
  } while (0)

#define SIDA_LAUNCH_CHECK()                                                        \
  do {                                                                             \
    ::sida::count_launch();                                                        \
    cudaError_t _e = cudaGetLastError();                                           \
    if (_e != cudaSuccess) {                                                       \
      ::sida::set_error("kernel launch failed: %s (%s:%d)", cudaGetErrorString(_e), \
                        __FILE__, __LINE__);                                       \
      return SIDA_ERR_CUDA;                                                        \
    }                                                                              \
  } while (0)

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

constexpr int kNumSMs = 148;

__host__ __device__ inline int ceil_div(int a, int b) { return (a + b - 1) / b; }
__host__ __device__ inline size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

__device__ __forceinline__ float bf16_to_f32(uint16_t b) {
  return __uint_as_float(static_cast<uint32_t>(b) << 16);
}

// Round-to-nearest-even float -> bf16 bits (inputs here are finite).
__device__ __forceinline__ uint16_t f32_to_bf16(float f) {
  uint32_t u = __float_as_uint(f);
  u += 0x7FFFu + ((u >> 16) & 1u);
  return static_cast<uint16_t>(u >> 16);
}

__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
  return static_cast<uint32_t>(f32_to_bf16(lo)) | (static_cast<uint32_t>(f32_to_bf16(hi)) << 16);
}

}  // namespace sida
