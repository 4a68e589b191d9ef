// Library-level plumbing of the C ABI: thread-local error strings, launch
// accounting and device-property caching.
#include <atomic>
#include <cstdio>

#include "common.cuh"

namespace sfb {

static thread_local std::string g_last_error;
static std::atomic<int64_t> g_launches{0};

void set_error(const std::string& msg) { g_last_error = msg; }

int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

int check_launch(const char* what) {
  g_launches.fetch_add(1, std::memory_order_relaxed);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    char buf[512];
    std::snprintf(buf, sizeof(buf), "%s: CUDA launch failed: %s", what, cudaGetErrorString(e));
    return fail(SFB_ECUDA, buf);
  }
  return SFB_OK;
}

int current_device() {
  int dev = 0;
  return cudaGetDevice(&dev) == cudaSuccess && dev >= 0 ? dev : 0;
}

int num_sms() {
  static std::atomic<int> cached[kMaxDevices];
  const int dev = current_device();
  int v = dev < kMaxDevices ? cached[dev].load(std::memory_order_relaxed) : 0;
  if (v == 0) {
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0)
      v = kNumSMs;
    if (dev < kMaxDevices) cached[dev].store(v, std::memory_order_relaxed);
  }
  return v;
}

}  // namespace sfb

extern "C" const char* sfb_last_error(void) { return sfb::g_last_error.c_str(); }
extern "C" int sfb_version(void) { return 100; }
extern "C" int64_t sfb_launch_count(void) { return sfb::g_launches.load(); }
