// SURVEY 8(f) rows f1 + f3: the periodic Burgers element's full time
// derivative (volume + interface term) and classic RK4 time integration with
// on-device entropy / mass monitoring, over a batch of independent elements.
//
// Reference (sumfac 0.1.0):
//   time_derivative   burgers.py:159-162  = volume_residual + _surface_residual
//   volume_residual   burgers.py:117-131  -(2/omega_r) sum_j sum_l Q_j[r,l] f(u_r, u_l)
//   _surface_residual burgers.py:134-156  per direction j: right-face nodes
//                     -= (f*(u_R, u_L) - u_R^2/2) / w[n-1], left-face nodes
//                     += (f*(u_R, u_L) - u_L^2/2) / w[0], directions in order
//   rk4               demos/burgers_entropy.py:25-33
//   total_entropy     burgers.py:165-169  0.5 * dot(omega, u*u)
// Every operation is the reference's, in its order and rounding (no FMA
// contraction, numpy's summation order), so time derivatives and RK4
// trajectories are bitwise equal to the reference's; the entropy / mass
// monitors are fixed-order sums (numpy's dot goes through BLAS, whose order is
// not specified: those match to rounding).
//
// Kernel shape: one CTA per element (threads = nodes rounded up to a warp),
// the element's stage state in shared memory, u and the RK4 stage sum in
// registers; each RK4 stage is one barrier-separated evaluation of the time
// derivative, so a whole multi-step integration is ONE launch with no host
// round trip.
#include "numpy_order.cuh"

namespace sfb {

// du/dt at node r of the element whose values are v (shared or global).
// LARGE: n > 128 rows need numpy's recursive split; the other instantiation
// carries no recursion (no stack frame, no spills).
template <bool LARGE>
__device__ __forceinline__ double burgers_dudt_node(int64_t r, int n, int d, int64_t nodes,
                                                    const double* __restrict__ qf,
                                                    const double* __restrict__ omega, int flux,
                                                    double w0, double wn, const double* v) {
  const double ur = v[r];
  // volume: -(2/omega_r) sum_j (sum_l Q_j[r,l] f(u_r, u_{r(j->l)})), numpy order
  double acc = 0.0;
  int64_t stride = 1;
  for (int j = 0; j < d; ++j) {
    const int64_t digit = (r / stride) % n;
    const int64_t base = r - digit * stride;
    const double* q = qf + ((int64_t)j * nodes + r) * n;
    auto ld = [&](int64_t l) { return __dmul_rn(__ldg(q + l), two_point(flux, ur, v[base + l * stride])); };
    double s;
    if constexpr (LARGE) s = numpy_pairwise_sum(ld, 0, n);
    else s = numpy_sum_small(ld, n);
    acc = (j == 0) ? s : __dadd_rn(acc, s);
    stride *= n;
  }
  const double vol = __ddiv_rn(__dmul_rn(-2.0, acc), __ldg(omega + r));
  // periodic interface term, directions in order (the node is a right face,
  // a left face or neither in each direction)
  const double pf = __dmul_rn(__dmul_rn(0.5, ur), ur);
  double surf = 0.0;
  stride = 1;
  for (int j = 0; j < d; ++j) {
    const int64_t digit = (r / stride) % n;
    if (digit == n - 1) {
      const double fs = two_point(flux, ur, v[r - (int64_t)(n - 1) * stride]);
      surf = __dsub_rn(surf, __ddiv_rn(__dsub_rn(fs, pf), wn));
    } else if (digit == 0) {
      const double fs = two_point(flux, v[r + (int64_t)(n - 1) * stride], ur);
      surf = __dadd_rn(surf, __ddiv_rn(__dsub_rn(fs, pf), w0));
    }
    stride *= n;
  }
  return __dadd_rn(vol, surf);
}

template <bool LARGE>
__global__ void burgers_dudt_kernel(int64_t E, int n, int d, int64_t nodes,
                                    const double* __restrict__ qf,
                                    const double* __restrict__ omega, int flux, double w0,
                                    double wn, const double* __restrict__ u,
                                    double* __restrict__ dudt) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t total = E * nodes;
  for (; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = t / nodes;
    dudt[t] = burgers_dudt_node<LARGE>(t - e * nodes, n, d, nodes, qf, omega, flux, w0, wn,
                                u + e * nodes);
  }
}

// Fixed-order block sum of x over the CTA (thread r holds x_r, 0 for r >= nodes):
// per-warp xor butterflies, then the warps in order.  Returns the sum to thread 0.
__device__ __forceinline__ double block_sum_fixed(double x, double* wsum) {
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  const int wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  __syncthreads();  // wsum may still be read from the previous call
  if ((threadIdx.x & 31) == 0) wsum[wid] = x;
  __syncthreads();
  double t = 0.0;
  if (threadIdx.x == 0) {
    t = wsum[0];
    for (int w = 1; w < nw; ++w) t += wsum[w];
  }
  return t;
}

template <bool LARGE>
__global__ void burgers_rk4_kernel(int64_t E, int n, int d, int64_t nodes,
                                   const double* __restrict__ qf,
                                   const double* __restrict__ omega, int flux, double w0,
                                   double wn, double dt, int steps, int every,
                                   double* __restrict__ u, double* __restrict__ entropy,
                                   double* __restrict__ mass) {
  extern __shared__ double v[];  // [nodes] stage input
  __shared__ double wsum[32];
  const int64_t r = threadIdx.x;
  const bool act = r < nodes;
  const double h = 0.5 * dt, dt6 = dt / 6.0;  // the demo's scalars (0.5 * dt, dt / 6.0)
  const int nrec = every > 0 ? steps / every + 1 : 0;
  for (int64_t e = blockIdx.x; e < E; e += gridDim.x) {
    double* ue = u + e * nodes;
    double ur = act ? ue[r] : 0.0;
    const double om = act ? omega[r] : 0.0;
    for (int step = 0; step <= steps; ++step) {
      if (every > 0 && step % every == 0) {  // monitors, before the step (demo order)
        const double s = block_sum_fixed(act ? __dmul_rn(om, __dmul_rn(ur, ur)) : 0.0, wsum);
        const double m = block_sum_fixed(act ? __dmul_rn(om, ur) : 0.0, wsum);
        if (threadIdx.x == 0) {
          if (entropy) entropy[e * nrec + step / every] = 0.5 * s;
          if (mass) mass[e * nrec + step / every] = m;
        }
      }
      if (step == steps) break;
      // k1 .. k4 with the stage inputs u + (dt/2) k1, u + (dt/2) k2, u + dt k3
      double sum = 0.0;
#pragma unroll 1
      for (int stage = 0; stage < 4; ++stage) {
        __syncthreads();  // everyone is done reading the previous stage input
        if (act) v[r] = (stage == 0) ? ur : v[r];
        __syncthreads();
        const double k =
            act ? burgers_dudt_node<LARGE>(r, n, d, nodes, qf, omega, flux, w0, wn, v) : 0.0;
        __syncthreads();  // all reads of this stage's input are done
        if (act) {
          if (stage == 0) sum = k;
          else if (stage == 3) sum = __dadd_rn(sum, k);
          else sum = __dadd_rn(sum, __dmul_rn(2.0, k));
          if (stage < 3) v[r] = __dadd_rn(ur, __dmul_rn(stage < 2 ? h : dt, k));
        }
      }
      if (act) ur = __dadd_rn(ur, __dmul_rn(dt6, sum));
    }
    if (act) ue[r] = ur;
    __syncthreads();
  }
}

static int grid_cap(int64_t work, int per_block) {
  int64_t blocks = (work + per_block - 1) / per_block;
  int64_t cap = (int64_t)num_sms() * 32;
  if (blocks > cap) blocks = cap;
  return blocks < 1 ? 1 : (int)blocks;
}

}  // namespace sfb

using namespace sfb;

extern "C" int sfb_burgers_time_derivative(int64_t E, int64_t n, int64_t d,
                                           const double* qfactors, const double* omega,
                                           double w0, double wn, int flux, const double* u,
                                           double* dudt, sfb_stream_t stream) {
  SFB_CHECK_ARG(E >= 0 && n >= 2 && d >= 1, "need E >= 0, n >= 2, d >= 1");
  SFB_CHECK_ARG(flux == SFB_FLUX_BURGERS_EC || flux == SFB_FLUX_BURGERS_AVG,
                "flux must be a built-in Burgers two-point flux");
  if (E == 0) return SFB_OK;
  SFB_CHECK_ARG(qfactors && omega && u && dudt, "null pointer");
  int64_t nodes = 1;
  for (int64_t i = 0; i < d; ++i) nodes *= n;
  auto kern = n <= 128 ? burgers_dudt_kernel<false> : burgers_dudt_kernel<true>;
  kern<<<grid_cap(E * nodes, 256), 256, 0, (cudaStream_t)stream>>>(
      E, (int)n, (int)d, nodes, qfactors, omega, flux, w0, wn, u, dudt);
  return check_launch("burgers_time_derivative");
}

extern "C" int sfb_burgers_rk4(int64_t E, int64_t n, int64_t d, const double* qfactors,
                               const double* omega, double w0, double wn, int flux, double dt,
                               int64_t steps, int64_t every, double* u, double* entropy,
                               double* mass, sfb_stream_t stream) {
  SFB_CHECK_ARG(E >= 0 && n >= 2 && d >= 1, "need E >= 0, n >= 2, d >= 1");
  SFB_CHECK_ARG(flux == SFB_FLUX_BURGERS_EC || flux == SFB_FLUX_BURGERS_AVG,
                "flux must be a built-in Burgers two-point flux");
  SFB_CHECK_ARG(steps >= 0 && steps < (1ll << 31) && every >= 0, "bad step counts");
  SFB_CHECK_ARG(every > 0 || (entropy == nullptr && mass == nullptr),
                "monitors need every > 0");
  if (E == 0) return SFB_OK;
  SFB_CHECK_ARG(qfactors && omega && u, "null pointer");
  int64_t nodes = 1;
  for (int64_t i = 0; i < d; ++i) nodes *= n;
  SFB_CHECK_ARG(nodes <= 1024, "rk4: one element per CTA needs n^d <= 1024");
  const int threads = (int)((nodes + 31) / 32 * 32);
  int64_t grid = E;
  const int64_t cap = (int64_t)num_sms() * (2048 / threads);
  if (grid > cap) grid = cap;
  // (nodes <= 1024 implies n <= 1024; rows above 128 only for d = 1)
  auto kern = n <= 128 ? burgers_rk4_kernel<false> : burgers_rk4_kernel<true>;
  kern<<<(unsigned)grid, threads, nodes * sizeof(double), (cudaStream_t)stream>>>(
      E, (int)n, (int)d, nodes, qfactors, omega, flux, w0, wn, dt, (int)steps, (int)every, u,
      entropy, mass);
  return check_launch("burgers_rk4");
}
