// Host-buffer entry points: the reference-facing call with numpy-style host
// arrays.  Element chunks are pipelined over three streams (H2D copy, kernel,
// D2H copy), so with pinned buffers the PCIe transfers in both directions
// overlap each other and the kernel.  One cached device staging arena per
// device (grown on demand, never shrunk) is the only allocation the library
// makes; calls on one device serialise on its arena, different devices run
// independently.
#include <cstdlib>
#include <mutex>

#include "common.cuh"

namespace sfb {
int euler_cartesian_dispatch(int64_t E, int64_t n, const double* D_host, double gamma,
                             double scale, const double* U, double* R, cudaStream_t s);

namespace {
constexpr int kStreams = 3;
struct Arena {
  std::mutex mu;
  cudaStream_t streams[kStreams] = {};
  double* buf[kStreams] = {};
  size_t cap = 0;  // doubles per stream buffer
};
Arena g_arenas[kMaxDevices];

int arena_reserve(Arena& a, size_t doubles) {
  for (int i = 0; i < kStreams; ++i) {
    if (!a.streams[i] &&
        cudaStreamCreateWithFlags(&a.streams[i], cudaStreamNonBlocking) != cudaSuccess)
      return fail(SFB_ECUDA, "cudaStreamCreate failed");
  }
  if (doubles > a.cap) {
    for (int i = 0; i < kStreams; ++i) {
      if (a.buf[i]) cudaFree(a.buf[i]);
      a.buf[i] = nullptr;
    }
    a.cap = 0;
    for (int i = 0; i < kStreams; ++i)
      if (cudaMalloc(&a.buf[i], doubles * sizeof(double)) != cudaSuccess)
        return fail(SFB_ECUDA, "staging arena allocation failed");
    a.cap = doubles;
  }
  return SFB_OK;
}

// wait for everything queued on the arena's streams (also on error paths, so
// no copy still reads or writes the caller's host buffers after the return)
int arena_drain(Arena& a, int rc) {
  for (int k = 0; k < kStreams; ++k) {
    if (!a.streams[k]) continue;
    const cudaError_t e = cudaStreamSynchronize(a.streams[k]);
    if (e != cudaSuccess && rc == SFB_OK)
      rc = fail(SFB_ECUDA, std::string("pipeline failed: ") + cudaGetErrorString(e));
  }
  return rc;
}
}  // namespace

}  // namespace sfb

using namespace sfb;

extern "C" int sfb_euler_volume_cartesian_host(int64_t E, int64_t n, const double* D_host,
                                               double gamma, double scale, const double* U_host,
                                               double* R_host) {
  SFB_CHECK_ARG(E >= 0 && n >= 2 && n <= 8, "bad extents (n must be in 2..8)");
  SFB_CHECK_ARG(D_host && U_host && R_host, "null pointer");
  SFB_CHECK_ARG(gamma > 1.0, "gamma must exceed 1");
  if (E == 0) return SFB_OK;
  const int dev = current_device();
  SFB_CHECK_ARG(dev < kMaxDevices, "device ordinal out of range");
  Arena& a = g_arenas[dev];
  std::lock_guard<std::mutex> lock(a.mu);
  const int64_t per = 5 * n * n * n;
  // ~32 MB of state per chunk: large enough to amortise the launch, small
  // enough that the pipeline fills quickly.
  int64_t chunk_doubles = (int64_t)(4 << 20);
  // (SFB_HOST_CHUNK_MB overrides for experiments; 8/16/32/64 MB measured
  // 16.3/15.2/14.9/15.0 ms per config-3 step)
  if (const char* env = getenv("SFB_HOST_CHUNK_MB")) {
    const int mb = atoi(env);
    if (mb > 0 && mb <= 4096) chunk_doubles = (int64_t)mb << 17;
  }
  int64_t chunk = chunk_doubles / per;
  if (chunk < 1) chunk = 1;
  if (chunk > E) chunk = E;
  int rc = arena_reserve(a, (size_t)(2 * chunk * per));
  if (rc) return rc;
  const int64_t nchunks = (E + chunk - 1) / chunk;
  for (int64_t c = 0; c < nchunks && rc == SFB_OK; ++c) {
    const int k = (int)(c % kStreams);
    cudaStream_t s = a.streams[k];
    double* dU = a.buf[k];
    double* dR = dU + chunk * per;
    const int64_t e0 = c * chunk;
    const int64_t ne = (E - e0) < chunk ? (E - e0) : chunk;
    if (cudaMemcpyAsync(dU, U_host + e0 * per, ne * per * sizeof(double), cudaMemcpyHostToDevice,
                        s) != cudaSuccess) {
      rc = fail(SFB_ECUDA, "H2D copy failed");
      break;
    }
    rc = euler_cartesian_dispatch(ne, n, D_host, gamma, scale, dU, dR, s);
    if (rc) break;
    if (cudaMemcpyAsync(R_host + e0 * per, dR, ne * per * sizeof(double), cudaMemcpyDeviceToHost,
                        s) != cudaSuccess)
      rc = fail(SFB_ECUDA, "D2H copy failed");
  }
  return arena_drain(a, rc);
}
