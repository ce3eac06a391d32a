// Library plumbing: thread-local error messages, version, device checks.
#include <atomic>
#include <map>
#include <utility>
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

// One-time per-(kernel, device) setup, thread-safe: the dynamic shared-memory opt-in is a
// per-device function attribute, so a process driving several GPUs sets it once on each
// (a process-wide static flag would leave every device but the first at 48 KB).
namespace {
std::mutex g_setup_mu;
std::map<std::pair<const void*, int>, int>& setup_cache() {
  static std::map<std::pair<const void*, int>, int> m;
  return m;
}
int current_device() {
  int dev = 0;
  cudaGetDevice(&dev);
  return dev;
}
}  // namespace

int smem_attr(const void* kernel, int bytes, const char* what) {
  const auto key = std::make_pair(kernel, current_device());
  std::lock_guard<std::mutex> lock(g_setup_mu);
  auto& m = setup_cache();
  if (m.count(key)) return GOOM_OK;
  if (cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes) !=
      cudaSuccess)
    return cuda_fail(cudaGetLastError(), what);
  m[key] = 1;
  return GOOM_OK;
}

int per_device_value(const void* key_ptr, int (*query)()) {
  // distinct key space from smem_attr: tag the pointer's low bit (function pointers are
  // at least 2-byte aligned)
  const auto key = std::make_pair(
      reinterpret_cast<const void*>(reinterpret_cast<uintptr_t>(key_ptr) | 1u), current_device());
  {
    std::lock_guard<std::mutex> lock(g_setup_mu);
    auto it = setup_cache().find(key);
    if (it != setup_cache().end()) return it->second;
  }
  const int v = query();  // outside the lock: the query may itself call smem_attr
  std::lock_guard<std::mutex> lock(g_setup_mu);
  setup_cache()[key] = v;
  return v;
}

int num_sms() {
  static std::atomic<int> cached[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) dev = 0;
  int v = cached[dev].load(std::memory_order_relaxed);
  if (!v) {
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0)
      v = 148;
    cached[dev].store(v, std::memory_order_relaxed);
  }
  return v;
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
