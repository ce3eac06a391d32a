// Shared device/host helpers for libgoom (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cmath>
#include <string>

#include "../../include/goom.h"

namespace goom {

constexpr float kPi = 3.14159265358979323846f;  // == (float)M_PI == 0x40490FDB
constexpr float kNegInf = -INFINITY;

// ---- error plumbing -------------------------------------------------------
void set_error(const std::string& msg);
int fail(int code, const std::string& msg);
int cuda_fail(cudaError_t e, const char* where);

#define GOOM_CHECK_LAUNCH(where)                                   \
  do {                                                             \
    cudaError_t _e = cudaGetLastError();                           \
    if (_e != cudaSuccess) return ::goom::cuda_fail(_e, (where));  \
  } while (0)

#define GOOM_TRY(expr)            \
  do {                            \
    int _rc = (expr);             \
    if (_rc != GOOM_OK) return _rc; \
  } while (0)

// ---- GOOM element helpers ---------------------------------------------------
// sign parity from the imaginary part: -1 iff cos(imag) < 0 (canonical 0 / pi fast)
__device__ __forceinline__ float goom_sign(float im) {
  if (im == 0.0f) return 1.0f;
  if (im == kPi) return -1.0f;
  return cosf(im) < 0.0f ? -1.0f : 1.0f;
}

__device__ __forceinline__ float2 goom_make(float log_mag, bool negative) {
  return make_float2(log_mag, negative ? kPi : 0.0f);
}

// log|v| and sign(v) of a real, canonical output (v == 0 -> (-inf, +))
__device__ __forceinline__ float2 goom_from_value(float v) {
  return make_float2(logf(fabsf(v)), v < 0.0f ? kPi : 0.0f);
}

// order-preserving float <-> uint map for deterministic atomicMax on floats
__device__ __forceinline__ unsigned int float_to_ordered(float f) {
  unsigned int u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float ordered_to_float(unsigned int u) {
  return __uint_as_float((u & 0x80000000u) ? (u & 0x7fffffffu) : ~u);
}

__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// ---- operand addressing -----------------------------------------------------
struct Operand {
  const float2* ptr;
  int64_t stride;
  int64_t div;
  __host__ __device__ __forceinline__ const float2* at(int64_t b) const {
    return ptr + (b / div) * stride;
  }
};

inline Operand make_operand(const goom_c64* p, int64_t stride, int64_t div) {
  return Operand{reinterpret_cast<const float2*>(p), stride, div < 1 ? 1 : div};
}
inline Operand make_operand(const float2* p, int64_t stride, int64_t div = 1) {
  return Operand{p, stride, div < 1 ? 1 : div};
}

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

inline int ceil_div(int64_t a, int64_t b) { return (int)((a + b - 1) / b); }

int num_sms();

}  // namespace goom
