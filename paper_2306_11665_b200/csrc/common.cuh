// Shared helpers for the sm_100a sum-factorized Hadamard / flux-differencing kernels.
//
// Conventions:
//  * node flat index r = r0 + r1*n + r2*n^2 (x fastest), as in the reference's
//    indexing.py:1-10; direction j has stride n^j.
//  * every entry point is stream-ordered on the caller's cudaStream_t, never
//    allocates, never synchronises, and reports errors through sfb_last_error().
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <string>

#include "../../include/sumfac_b200.h"

namespace sfb {

void set_error(const std::string& msg);
int fail(int code, const std::string& msg);
int check_launch(const char* what);

constexpr int kNumSMs = 148;  // B200; only used as a grid-size hint (the
                              // runtime value is queried once per device and cached).
int num_sms();  // SMs of the current device

// Resident CTAs per SM of `kern` at (threads, smem) on the current device,
// after opting the kernel in to `smem` bytes of dynamic shared memory (a
// per-device function attribute).  Cached per device in `cache`, one slot per
// device ordinal; concurrent first calls only repeat the same idempotent setup.
constexpr int kMaxDevices = 64;
using DeviceCache = std::atomic<int>[kMaxDevices];
int current_device();
template <typename Kern>
int resident_ctas(Kern kern, int threads, size_t smem, DeviceCache& cache) {
  const int dev = current_device();
  int v = dev < kMaxDevices ? cache[dev].load(std::memory_order_relaxed) : 0;
  if (v == 0) {
    if (smem > 48 * 1024)
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int b = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, kern, threads, smem);
    v = b > 0 ? b : 1;
    if (dev < kMaxDevices) cache[dev].store(v, std::memory_order_relaxed);
  }
  return v;
}

// ---------------------------------------------------------------------------
// FP64 helpers
// ---------------------------------------------------------------------------

// MUFU.RCP64H seed (about 2^-23 relative) refined by one cubic Newton step
// (e = 1 - x r; r += r (e + e^2)): ~2^-66 before rounding, i.e. within an ulp
// or two of the correctly rounded reciprocal.  Used where the quotient feeds
// a 1e-12-parity result and never a branch decision.
__device__ __forceinline__ double rcp_approx(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  return r;
}

__device__ __forceinline__ double rcp_refined(double x) {
  double r = rcp_approx(x);
  double e = fma(-x, r, 1.0);
  double e2 = fma(e, e, e);
  return fma(r, e2, r);
}

// Guaranteed branch-free select (PTX selp).  A C++ ternary on doubles may be
// lowered to a branch, which splits the basic block and stops ptxas from
// interleaving independent work around it.
__device__ __forceinline__ double dsel(bool p, double a, double b) {
  double r;
  asm("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %3, 0;\n\tselp.f64 %0, %1, %2, q;\n\t}"
      : "=d"(r)
      : "d"(a), "d"(b), "r"((int)p));
  return r;
}

// Stream-lined load of read-once data: bypass L1 allocation.
__device__ __forceinline__ double2 ld_stream_d2(const double* p) {
  double2 v;
  asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];"
               : "=d"(v.x), "=d"(v.y)
               : "l"(p));
  return v;
}

// 256-bit loads (LDG.E.ENL2.256, sm_100): one request per 32 B row segment.
struct d4 {
  double x, y, z, w;
};
__device__ __forceinline__ d4 ld_stream_d4(const double* p) {
  d4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.f64 {%0, %1, %2, %3}, [%4];"
               : "=d"(v.x), "=d"(v.y), "=d"(v.z), "=d"(v.w)
               : "l"(p));
  return v;
}
__device__ __forceinline__ d4 ld_ro_d4(const double* p) {
  d4 v;
  asm("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];"
      : "=d"(v.x), "=d"(v.y), "=d"(v.z), "=d"(v.w)
      : "l"(p));
  return v;
}

__device__ __forceinline__ void st_stream_d2(double* p, double2 v) {
  asm volatile("st.global.L1::no_allocate.v2.f64 [%0], {%1, %2};" ::"l"(p), "d"(v.x), "d"(v.y)
               : "memory");
}


}  // namespace sfb

#define SFB_CHECK_ARG(cond, msg)                    \
  do {                                              \
    if (!(cond)) return ::sfb::fail(SFB_EINVAL, msg); \
  } while (0)
