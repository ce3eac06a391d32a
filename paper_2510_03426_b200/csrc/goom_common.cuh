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

// every kernel launch site goes through this: error check + the launch counter
// behind goom_kernel_launches() (bench.py reports it as gpu_launches)
void count_launch();
#define GOOM_CHECK_LAUNCH(where)                                   \
  do {                                                             \
    ::goom::count_launch();                                        \
    cudaError_t _e = cudaGetLastError();                           \
    if (_e != cudaSuccess) return ::goom::cuda_fail(_e, (where));  \
  } while (0)

#define GOOM_TRY(expr)            \
  do {                            \
    int _rc = (expr);             \
    if (_rc != GOOM_OK) return _rc; \
  } while (0)

// ---- GOOM element helpers ---------------------------------------------------
// Sign parity from the imaginary part: negative iff the phase lies within a quarter
// turn of pi (== cos(imag) < 0, the reference adapter's rule, except exactly at
// +-pi/2 where the phase carries no sign). Branch-free: FMUL, FRND, FADD, FSETP —
// no cosf range reduction on the hot path, any 2*pi multiple accepted.
__device__ __forceinline__ bool phase_negative(float im) {
  const float t = im * 0.15915494309189535f;  // 1 / (2 pi)
  return fabsf(t - rintf(t)) > 0.25f;
}
__device__ __forceinline__ bool phase_negative(double im) {
  const double t = im * 0.15915494309189535;
  return fabs(t - rint(t)) > 0.25;
}
__device__ __forceinline__ float goom_sign(float im) { return phase_negative(im) ? -1.0f : 1.0f; }

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

// ---- precision-generic helpers (complex64 = float2, complex128 = double2) -------
template <class R> struct CxOf;
template <> struct CxOf<float> { using type = float2; };
template <> struct CxOf<double> { using type = double2; };
template <class R> using Cx = typename CxOf<R>::type;

template <class R> __host__ __device__ __forceinline__ R pi_of();
template <> __host__ __device__ __forceinline__ float pi_of<float>() { return kPi; }
template <> __host__ __device__ __forceinline__ double pi_of<double>() {
  return 3.14159265358979323846;
}

__device__ __forceinline__ float gexp(float x) { return expf(x); }
__device__ __forceinline__ double gexp(double x) { return exp(x); }
__device__ __forceinline__ float glog(float x) { return logf(x); }
__device__ __forceinline__ double glog(double x) { return log(x); }
__device__ __forceinline__ float add_rn(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ float sub_rn(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ double sub_rn(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ float mul_rn(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ float gfma(float a, float b, float c) { return fmaf(a, b, c); }
__device__ __forceinline__ double gfma(double a, double b, double c) { return fma(a, b, c); }
__device__ __forceinline__ float gmax(float a, float b) { return fmaxf(a, b); }
__device__ __forceinline__ double gmax(double a, double b) { return fmax(a, b); }

template <class R> __device__ __forceinline__ R goom_sign_t(R im) {
  return phase_negative(im) ? R(-1) : R(1);
}
template <class R> __device__ __forceinline__ Cx<R> cx(R re, R im) {
  Cx<R> z;
  z.x = re;
  z.y = im;
  return z;
}
template <class R> __device__ __forceinline__ R warp_max_t(R v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = gmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// ---- operand addressing -----------------------------------------------------
template <class C>
struct OperandT {
  const C* ptr;
  int64_t stride;
  int64_t div;
  __host__ __device__ __forceinline__ const C* at(int64_t b) const {
    return ptr + (b / div) * stride;
  }
};
using Operand = OperandT<float2>;

inline Operand make_operand(const goom_c64* p, int64_t stride, int64_t div) {
  return Operand{reinterpret_cast<const float2*>(p), stride, div < 1 ? 1 : div};
}
inline Operand make_operand(const float2* p, int64_t stride, int64_t div = 1) {
  return Operand{p, stride, div < 1 ? 1 : div};
}

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

inline int ceil_div(int64_t a, int64_t b) { return (int)((a + b - 1) / b); }

int num_sms();
// once per (kernel, device), thread-safe (abi.cu): opt a kernel into `bytes` of dynamic
// shared memory on the current device
int smem_attr(const void* kernel, int bytes, const char* what);
// a value computed once per (key, device), thread-safe (e.g. an occupancy query)
int per_device_value(const void* key, int (*query)());

}  // namespace goom
