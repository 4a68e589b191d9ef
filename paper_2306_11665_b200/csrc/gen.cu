// Seeded, element-addressable synthetic inputs and deterministic block sums.
//
// The generator is a counter-based hash (splitmix64 finaliser), so every value
// is a pure function of (seed, global index): the host restatement in
// paper_2306_11665_b200/synth.py produces bit-identical arrays, a shard of
// elements [e0, e0+E) is identical whatever the number of ranks, and inputs for
// the full-size benchmarks are created on the device in milliseconds.  All
// arithmetic is written with explicit round-to-nearest intrinsics (no FMA
// contraction) to stay bitwise equal to numpy.
#include "common.cuh"

namespace sfb {

__host__ __device__ __forceinline__ uint64_t splitmix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// uniform double in [0, 1) with 53 random bits
__device__ __forceinline__ double u01(uint64_t key, uint64_t idx) {
  return (double)(splitmix64(key + idx) >> 11) * 0x1.0p-53;
}

__device__ __forceinline__ double uniform(uint64_t key, uint64_t idx, double lo, double width) {
  return __dadd_rn(lo, __dmul_rn(width, u01(key, idx)));
}

__global__ void generate_uniform_kernel(int64_t count, int64_t i0, uint64_t key, double lo,
                                        double width, double* __restrict__ out) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  for (; t < count; t += (int64_t)gridDim.x * blockDim.x)
    out[t] = uniform(key, (uint64_t)(i0 + t), lo, width);
}

// Primitive draw index: ((e * 5 + k) * nodes + r), k = 0 rho, 1..3 v, 4 p.
__global__ void generate_euler_kernel(int64_t E, int64_t e0, int64_t nodes, uint64_t key,
                                      double gm1, double rlo, double rw, double vlo, double vw,
                                      double plo, double pw, double* __restrict__ U) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t total = E * nodes;
  for (; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    int64_t e = t / nodes;
    int64_t r = t - e * nodes;
    uint64_t g = (uint64_t)(e0 + e) * 5 * (uint64_t)nodes + (uint64_t)r;
    double rho = uniform(key, g, rlo, rw);
    double v0 = uniform(key, g + nodes, vlo, vw);
    double v1 = uniform(key, g + 2 * nodes, vlo, vw);
    double v2 = uniform(key, g + 3 * nodes, vlo, vw);
    double p = uniform(key, g + 4 * nodes, plo, pw);
    double vv = __dadd_rn(__dadd_rn(__dmul_rn(v0, v0), __dmul_rn(v1, v1)), __dmul_rn(v2, v2));
    double et = __dadd_rn(__ddiv_rn(p, gm1), __dmul_rn(__dmul_rn(0.5, rho), vv));
    double* u = U + e * 5 * nodes + r;
    u[0] = rho;
    u[nodes] = __dmul_rn(rho, v0);
    u[2 * nodes] = __dmul_rn(rho, v1);
    u[3 * nodes] = __dmul_rn(rho, v2);
    u[4 * nodes] = et;
  }
}

// Modal coefficients (config 5): idx = (e*5 + v)*modes + k,
// Uhat = (amp_v 2^-(k0+k1+k2)) (2u - 1)  (+ mean_v c0 at k = 0).
struct ModalGenParams {
  double mean[5], amp[5], c0;
};

__global__ void generate_modal_kernel(int64_t E, int64_t e0, int n, uint64_t key,
                                      ModalGenParams prm, double* __restrict__ Uhat) {
  const int64_t modes = (int64_t)n * n * n;
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t total = E * 5 * modes;
  for (; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = t / (5 * modes);
    const int64_t rem = t - e * 5 * modes;
    const int v = (int)(rem / modes);
    const int k = (int)(rem - (int64_t)v * modes);
    const uint64_t idx = ((uint64_t)(e0 + e) * 5 + v) * (uint64_t)modes + k;
    const double w = __dsub_rn(__dmul_rn(2.0, u01(key, idx)), 1.0);
    const int deg = k % n + (k / n) % n + k / (n * n);
    double x = __dmul_rn(__dmul_rn(prm.amp[v], ldexp(1.0, -deg)), w);
    if (k == 0) x = __dadd_rn(__dmul_rn(prm.mean[v], prm.c0), x);
    Uhat[t] = x;
  }
}

// Warped-lattice metric cofactors (config 5); see synth.metric_cofactors.
struct MetricGenParams {
  double nodes[16];
  double phi[9];
  double h, amp;
  int64_t K;
};

__global__ void generate_metric_kernel(int64_t E, int64_t e0, int n, MetricGenParams prm,
                                       double* __restrict__ Ja) {
  const int64_t nodes = (int64_t)n * n * n;
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t total = E * nodes;
  const double two_pi = 6.283185307179586;
  for (; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = t / nodes;
    const int r = (int)(t - e * nodes);
    const int64_t cell = (e0 + e) % (prm.K * prm.K * prm.K);
    const int64_t c[3] = {cell % prm.K, (cell / prm.K) % prm.K, cell / (prm.K * prm.K)};
    const int rr[3] = {r % n, (r / n) % n, r / (n * n)};
    double X[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) X[k] = ((double)c[k] + (prm.nodes[rr[k]] + 1.0) * 0.5) * prm.h;
    double G[3][3];
#pragma unroll
    for (int m = 0; m < 3; ++m) {
      double sn[3], cs[3];
#pragma unroll
      for (int k = 0; k < 3; ++k) sincos(two_pi * (X[k] + prm.phi[m * 3 + k]), &sn[k], &cs[k]);
#pragma unroll
      for (int i = 0; i < 3; ++i) {
        const double prod = cs[i] * sn[(i + 1) % 3] * sn[(i + 2) % 3];
        G[m][i] = 0.5 * prm.h * ((m == i ? 1.0 : 0.0) + prm.amp * two_pi * prod);
      }
    }
    double* out = Ja + e * 9 * nodes + r;
#pragma unroll
    for (int i = 0; i < 3; ++i) {
#pragma unroll
      for (int m = 0; m < 3; ++m) {
        const int a = m == 0 ? 1 : 0, b = m == 2 ? 1 : 2;
        const int cc = i == 0 ? 1 : 0, d = i == 2 ? 1 : 2;
        const double minor = G[a][cc] * G[b][d] - G[a][d] * G[b][cc];
        out[(i * 3 + m) * nodes] = ((i + m) % 2 == 0) ? minor : -minor;
      }
    }
  }
}

// Perfect binary tree within each block: level k adds entries 2i and 2i+1 of
// level k-1.  The order is a property of the data, not of the launch.
__global__ void block_sums_kernel(const double* __restrict__ x, int64_t block,
                                  double* __restrict__ partial) {
  extern __shared__ double s[];  // 2 * block: ping-pong levels
  const double* xb = x + (int64_t)blockIdx.x * block;
  for (int64_t i = threadIdx.x; i < block; i += blockDim.x) s[i] = xb[i];
  __syncthreads();
  double* src = s;
  double* dst = s + block;
  for (int64_t width = block / 2; width >= 1; width /= 2) {
    for (int64_t i = threadIdx.x; i < width; i += blockDim.x)
      dst[i] = __dadd_rn(src[2 * i], src[2 * i + 1]);
    __syncthreads();
    double* t = src;
    src = dst;
    dst = t;
  }
  if (threadIdx.x == 0) partial[blockIdx.x] = src[0];
}

}  // namespace sfb

using namespace sfb;

static int grid_cap(int64_t work) {
  int64_t b = (work + 255) / 256;
  int64_t cap = (int64_t)num_sms() * 32;
  return (int)(b < 1 ? 1 : (b > cap ? cap : b));
}

extern "C" int sfb_generate_uniform(int64_t count, int64_t i0, uint64_t seed, double lo,
                                    double hi, double* out, sfb_stream_t stream) {
  SFB_CHECK_ARG(count >= 0 && i0 >= 0, "negative count/offset");
  if (count == 0) return SFB_OK;
  SFB_CHECK_ARG(out != nullptr, "null output");
  generate_uniform_kernel<<<grid_cap(count), 256, 0, (cudaStream_t)stream>>>(
      count, i0, splitmix64(seed), lo, hi - lo, out);
  return check_launch("generate_uniform");
}

extern "C" int sfb_generate_euler_states(int64_t E, int64_t e0, int64_t n, uint64_t seed,
                                         double gamma, const double* b, double* U,
                                         sfb_stream_t stream) {
  SFB_CHECK_ARG(E >= 0 && e0 >= 0 && n >= 1, "bad extents");
  SFB_CHECK_ARG(b != nullptr, "null bounds (host array of 6)");
  if (E == 0) return SFB_OK;
  SFB_CHECK_ARG(U != nullptr, "null output");
  int64_t nodes = n * n * n;
  generate_euler_kernel<<<grid_cap(E * nodes), 256, 0, (cudaStream_t)stream>>>(
      E, e0, nodes, splitmix64(seed), gamma - 1.0, b[0], b[1] - b[0], b[2], b[3] - b[2], b[4],
      b[5] - b[4], U);
  return check_launch("generate_euler_states");
}

extern "C" int sfb_generate_modal_states(int64_t E, int64_t e0, int64_t n, uint64_t seed,
                                         const double* means5, const double* amps5, double c0,
                                         double* Uhat, sfb_stream_t stream) {
  SFB_CHECK_ARG(E >= 0 && e0 >= 0 && n >= 1 && n <= 16, "bad extents");
  SFB_CHECK_ARG(means5 && amps5, "null means/amps (host arrays of 5)");
  if (E == 0) return SFB_OK;
  SFB_CHECK_ARG(Uhat != nullptr, "null output");
  ModalGenParams prm;
  for (int v = 0; v < 5; ++v) {
    prm.mean[v] = means5[v];
    prm.amp[v] = amps5[v];
  }
  prm.c0 = c0;
  generate_modal_kernel<<<grid_cap(E * 5 * n * n * n), 256, 0, (cudaStream_t)stream>>>(
      E, e0, (int)n, splitmix64(seed), prm, Uhat);
  return check_launch("generate_modal_states");
}

extern "C" int sfb_generate_metric(int64_t E, int64_t e0, int64_t n, uint64_t seed,
                                   const double* nodes, int64_t K, double amp, double* Ja,
                                   sfb_stream_t stream) {
  SFB_CHECK_ARG(E >= 0 && e0 >= 0 && n >= 1 && n <= 16 && K >= 1, "bad extents");
  SFB_CHECK_ARG(nodes != nullptr, "null nodes (host array of n)");
  if (E == 0) return SFB_OK;
  SFB_CHECK_ARG(Ja != nullptr, "null output");
  MetricGenParams prm;
  for (int i = 0; i < n; ++i) prm.nodes[i] = nodes[i];
  const uint64_t key = splitmix64(seed);
  for (int i = 0; i < 9; ++i)
    prm.phi[i] = (double)(splitmix64(key + (uint64_t)i) >> 11) * 0x1.0p-53;
  prm.h = 1.0 / (double)K;
  prm.amp = amp;
  prm.K = K;
  generate_metric_kernel<<<grid_cap(E * n * n * n), 256, 0, (cudaStream_t)stream>>>(
      E, e0, (int)n, prm, Ja);
  return check_launch("generate_metric");
}

extern "C" int sfb_block_sums(const double* x, int64_t count, int64_t block, double* partial,
                              sfb_stream_t stream) {
  SFB_CHECK_ARG(block >= 1 && block <= 4096 && (block & (block - 1)) == 0,
                "block must be a power of two <= 4096");
  SFB_CHECK_ARG(count >= 0 && count % block == 0, "count must be a multiple of block");
  if (count == 0) return SFB_OK;
  SFB_CHECK_ARG(x && partial, "null pointer");
  int64_t nb = count / block;
  SFB_CHECK_ARG(nb <= 0x7fffffff, "too many blocks");
  if (2 * block * sizeof(double) > 48 * 1024)
    cudaFuncSetAttribute(block_sums_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)(2 * block * sizeof(double)));
  block_sums_kernel<<<(unsigned)nb, 256, 2 * block * sizeof(double), (cudaStream_t)stream>>>(x, block,
                                                                                      partial);
  return check_launch("block_sums");
}
