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
                             double scale, const double* U, double* R, void* ws,
                             cudaStream_t s);

namespace {
constexpr int kStreams = 3;
struct Arena {
  std::mutex mu;
  cudaStream_t streams[kStreams] = {};
  char* buf[kStreams] = {};
  size_t cap = 0;  // bytes per stream buffer
  double* aux = nullptr;  // small per-call operands (basis factors)
  size_t aux_cap = 0;     // doubles
  unsigned long long* ws = nullptr;  // one 8-byte claim counter per stream
};
Arena g_arenas[kMaxDevices];

int arena_reserve(Arena& a, size_t bytes) {
  for (int i = 0; i < kStreams; ++i) {
    if (!a.streams[i] &&
        cudaStreamCreateWithFlags(&a.streams[i], cudaStreamNonBlocking) != cudaSuccess)
      return fail(SFB_ECUDA, "cudaStreamCreate failed");
  }
  if (!a.ws && cudaMalloc(&a.ws, 256 * kStreams) != cudaSuccess)
    return fail(SFB_ECUDA, "staging arena allocation failed");
  if (bytes > a.cap) {
    for (int i = 0; i < kStreams; ++i) {
      if (a.buf[i]) cudaFree(a.buf[i]);
      a.buf[i] = nullptr;
    }
    a.cap = 0;
    for (int i = 0; i < kStreams; ++i)
      if (cudaMalloc(&a.buf[i], bytes) != cudaSuccess)
        return fail(SFB_ECUDA, "staging arena allocation failed");
    a.cap = bytes;
  }
  return SFB_OK;
}

int arena_aux(Arena& a, size_t doubles) {
  if (doubles > a.aux_cap) {
    if (a.aux) cudaFree(a.aux);
    a.aux = nullptr;
    a.aux_cap = 0;
    if (cudaMalloc(&a.aux, doubles * sizeof(double)) != cudaSuccess)
      return fail(SFB_ECUDA, "staging arena allocation failed");
    a.aux_cap = doubles;
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

// One host array of the pipeline: `per` doubles per element.
struct HostArray {
  const double* in;  // host input (H2D per chunk), or
  double* out;       // host output (D2H per chunk)
  int64_t per;
};

int64_t round_up(int64_t x, int64_t a) { return (x + a - 1) / a * a; }

// Element chunks of every array, round-robin over the arena's streams:
// H2D of the chunk's inputs, launch(ne, device pointers, stream, workspace),
// D2H of its outputs.  ~chunk_bytes of inputs per chunk (32 MB: large enough
// to amortise the launch, small enough that the pipeline fills quickly;
// SFB_HOST_CHUNK_MB overrides for experiments, 8/16/32/64 MB measured
// 16.3/15.2/14.9/15.0 ms per config-3 step).
template <int N, typename Launch>
int pipeline(Arena& a, int64_t E, const HostArray (&arr)[N], Launch launch) {
  int64_t chunk_bytes = (int64_t)32 << 20;
  if (const char* env = getenv("SFB_HOST_CHUNK_MB")) {
    const int mb = atoi(env);
    if (mb > 0 && mb <= 4096) chunk_bytes = (int64_t)mb << 20;
  }
  int64_t in_per = 0, all_per = 0;
  for (int i = 0; i < N; ++i) {
    if (arr[i].in) in_per += arr[i].per;
    all_per += arr[i].per;
  }
  int64_t chunk = chunk_bytes / (8 * (in_per > 0 ? in_per : all_per));
  if (chunk < 1) chunk = 1;
  if (chunk > E) chunk = E;
  int64_t off[N], bytes = 0;
  for (int i = 0; i < N; ++i) {
    off[i] = bytes;
    bytes += round_up(chunk * arr[i].per * 8, 256);
  }
  int rc = arena_reserve(a, (size_t)bytes);
  if (rc) return rc;
  const int64_t nchunks = (E + chunk - 1) / chunk;
  for (int64_t c = 0; c < nchunks && rc == SFB_OK; ++c) {
    const int k = (int)(c % kStreams);
    cudaStream_t s = a.streams[k];
    const int64_t e0 = c * chunk;
    const int64_t ne = (E - e0) < chunk ? (E - e0) : chunk;
    double* dev[N];
    for (int i = 0; i < N; ++i) dev[i] = (double*)(a.buf[k] + off[i]);
    for (int i = 0; i < N && rc == SFB_OK; ++i)
      if (arr[i].in && cudaMemcpyAsync(dev[i], arr[i].in + e0 * arr[i].per,
                                       ne * arr[i].per * 8, cudaMemcpyHostToDevice,
                                       s) != cudaSuccess)
        rc = fail(SFB_ECUDA, "H2D copy failed");
    if (rc) break;
    rc = launch(ne, dev, s, (void*)((char*)a.ws + 256 * k));
    for (int i = 0; i < N && rc == SFB_OK; ++i)
      if (arr[i].out && cudaMemcpyAsync(arr[i].out + e0 * arr[i].per, dev[i],
                                        ne * arr[i].per * 8, cudaMemcpyDeviceToHost,
                                        s) != cudaSuccess)
        rc = fail(SFB_ECUDA, "D2H copy failed");
  }
  return arena_drain(a, rc);
}

Arena* lock_arena(std::unique_lock<std::mutex>& lk) {
  const int dev = current_device();
  if (dev >= kMaxDevices) return nullptr;
  Arena& a = g_arenas[dev];
  lk = std::unique_lock<std::mutex>(a.mu);
  return &a;
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
  std::unique_lock<std::mutex> lk;
  Arena* a = lock_arena(lk);
  SFB_CHECK_ARG(a, "device ordinal out of range");
  const int64_t per = 5 * n * n * n;
  const HostArray arr[2] = {{U_host, nullptr, per}, {nullptr, R_host, per}};
  return pipeline(*a, E, arr, [&](int64_t ne, double* const* dev, cudaStream_t s, void* ws) {
    return euler_cartesian_dispatch(ne, n, D_host, gamma, scale, dev[0], dev[1], ws, s);
  });
}

extern "C" int sfb_hadamard_rowsum_batched_host(int64_t E, int64_t m, int64_t n, int64_t d,
                                                const double* basis_host, const double* F_host,
                                                double* out_sum_host) {
  SFB_CHECK_ARG(E >= 0 && m >= 1 && n >= 1 && d >= 1 && d <= 16, "bad extents");
  SFB_CHECK_ARG(basis_host && F_host && out_sum_host, "null pointer");
  if (E == 0) return SFB_OK;
  int64_t R = m;
  for (int64_t i = 1; i < d; ++i) R *= n;
  std::unique_lock<std::mutex> lk;
  Arena* a = lock_arena(lk);
  SFB_CHECK_ARG(a, "device ordinal out of range");
  const int64_t nb = d * R * n;
  int rc = arena_aux(*a, (size_t)nb);
  if (rc) return rc;
  // the basis factors are shared by every chunk: one synchronous upload
  if (cudaMemcpy(a->aux, basis_host, nb * 8, cudaMemcpyHostToDevice) != cudaSuccess)
    return fail(SFB_ECUDA, "H2D copy of the basis factors failed");
  const HostArray arr[2] = {{F_host, nullptr, d * R * n}, {nullptr, out_sum_host, R}};
  double* basis = a->aux;
  return pipeline(*a, E, arr, [&](int64_t ne, double* const* dev, cudaStream_t s, void*) {
    return sfb_hadamard_rowsum_batched(ne, m, n, d, basis, dev[0], nullptr, dev[1],
                                       (sfb_stream_t)s);
  });
}

extern "C" int sfb_euler_volume_curvilinear_modal_host(int64_t E, int64_t n, const double* V,
                                                       const double* Pi, const double* D,
                                                       double gamma, double scale,
                                                       const double* Uhat_host,
                                                       const double* Ja_host, double* Rhat_host,
                                                       double* sumsq_host) {
  SFB_CHECK_ARG(E >= 0 && n >= 2 && n <= 8, "bad extents (n must be in 2..8)");
  SFB_CHECK_ARG(V && Pi && D && Uhat_host && Ja_host && Rhat_host, "null pointer");
  SFB_CHECK_ARG(gamma > 1.0, "gamma must exceed 1");
  if (E == 0) return SFB_OK;
  std::unique_lock<std::mutex> lk;
  Arena* a = lock_arena(lk);
  SFB_CHECK_ARG(a, "device ordinal out of range");
  const int64_t nodes = n * n * n;
  const HostArray arr[4] = {{Uhat_host, nullptr, 5 * nodes},
                            {Ja_host, nullptr, 9 * nodes},
                            {nullptr, Rhat_host, 5 * nodes},
                            {nullptr, sumsq_host, sumsq_host ? 1 : 0}};
  return pipeline(*a, E, arr, [&](int64_t ne, double* const* dev, cudaStream_t s, void* ws) {
    return sfb_euler_volume_curvilinear_modal(ne, n, V, Pi, D, gamma, scale, dev[0], dev[1],
                                              dev[2], sumsq_host ? dev[3] : nullptr, ws,
                                              (sfb_stream_t)s);
  });
}
