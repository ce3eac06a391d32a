// Library plumbing: thread-local error messages, version, device checks.
#include <atomic>
#include <mutex>
#include <string>

#include "goom_internal.cuh"

namespace goom {

namespace {
thread_local std::string g_last_error;
std::atomic<long long> g_launches{0};
}

void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

void set_error(const std::string& msg) { g_last_error = msg; }

int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

int cuda_fail(cudaError_t e, const char* where) {
  g_last_error = std::string(where) + ": " + cudaGetErrorString(e);
  return GOOM_ECUDA;
}

int num_sms() {
  static int cached[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) dev = 0;
  if (!cached[dev]) {
    int v = 0;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0)
      v = 148;
    cached[dev] = v;
  }
  return cached[dev];
}

}  // namespace goom

extern "C" {

const char* goom_last_error(void) { return goom::g_last_error.c_str(); }

const char* goom_version(void) { return "goom-b200 0.1.0 (sm_100a)"; }

int goom_device_supported(int device) {
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, device) != cudaSuccess) return 0;
  return prop.major == 10 && prop.minor == 0 ? 1 : 0;
}

}  // extern "C"

extern "C" long long goom_kernel_launches(void) { return goom::g_launches.load(); }
