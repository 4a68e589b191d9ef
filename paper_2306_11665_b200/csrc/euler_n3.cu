// K3 at n = 3 (config 4's second point): the Cartesian Euler volume term
//
//   R[e,:,r] = scale * sum_j sum_l D[r_j,l] F#_j(U[e,:,r], U[e,:,r(j->l)])
//
// (burgers.py:117-131 generalised, as euler.cu) in registers and shuffles.
// Nine threads own one element (three elements per warp, lanes 27-31 shadow
// lane 0..4's work without writing); thread (x0, x1) holds the three nodes of
// its x2-line (x2 = 0, 1, 2): their records, diagonal terms and accumulators.
//   direction 2: the line is the thread's own - its three pairs are local;
//   directions 0 and 1: a line's three nodes sit in three threads (x0 or x1 =
//     0, 1, 2) and n = 3 needs one round: thread x evaluates the pair
//     (x, x+1 mod 3) at each of its three x2 levels with the partner's
//     records fetched by shuffles, and receives, also by shuffles, the three
//     fluxes of the pairs (x-1 mod 3, x) evaluated by its other neighbour.
// Every pair once (27 per direction and element); no shared memory, no
// barriers (the warp kernel this replaces at n = 3 was shared-memory and
// latency bound, profiles/r02/ncu_c4_n3.txt).
#include "euler_common.cuh"

#ifndef SFB_N3_L2PF
#define SFB_N3_L2PF 1  // 0.426 vs 0.430 ms
#endif
#ifndef SFB_N3_THREADS
#define SFB_N3_THREADS 128
#endif
#ifndef SFB_N3_MINB
#define SFB_N3_MINB 3
#endif

namespace sfb {

namespace {

__device__ __forceinline__ NodeRec rot3(const NodeRec& a, int j) {
  NodeRec r = a;
  if (j == 1) {
    r.hv0 = a.hv1;
    r.hv1 = a.hv2;
    r.hv2 = a.hv0;
  } else if (j == 2) {
    r.hv0 = a.hv2;
    r.hv1 = a.hv0;
    r.hv2 = a.hv1;
  }
  return r;
}

__device__ __forceinline__ void add_rot3(double (&acc)[5], double c, const double (&f)[5], int j) {
  acc[0] = fma(c, f[0], acc[0]);
  acc[1 + j] = fma(c, f[1], acc[1 + j]);
  acc[1 + (j + 1) % 3] = fma(c, f[2], acc[1 + (j + 1) % 3]);
  acc[1 + (j + 2) % 3] = fma(c, f[3], acc[1 + (j + 2) % 3]);
  acc[4] = fma(c, f[4], acc[4]);
}

__device__ __forceinline__ NodeRec shfl_rec_idx(const NodeRec& q, int src) {
  NodeRec r;
  r.hr = __shfl_sync(0xffffffffu, q.hr, src);
  r.hv0 = __shfl_sync(0xffffffffu, q.hv0, src);
  r.hv1 = __shfl_sync(0xffffffffu, q.hv1, src);
  r.hv2 = __shfl_sync(0xffffffffu, q.hv2, src);
  r.hb = __shfl_sync(0xffffffffu, q.hb, src);
  r.hlr = __shfl_sync(0xffffffffu, q.hlr, src);
  r.hlb = __shfl_sync(0xffffffffu, q.hlb, src);
  return r;
}

// one direction j in {0, 1} across threads: at each x2 level this thread
// evaluates (me, partner) and receives the flux of (receiver-side) pair
template <int J>
__device__ __forceinline__ void cross_dir(const NodeRec (&rq)[3], int srcP, int srcF, double cOwn,
                                          double cRecv, double gm1, double (&acc)[3][5]) {
  NodeRec A[3], B[3];
#pragma unroll
  for (int z = 0; z < 3; ++z) {
    A[z] = rot3(rq[z], J);
    B[z] = rot3(shfl_rec_idx(rq[z], srcP), J);
  }
  const NodeRec* PA[3] = {&A[0], &A[1], &A[2]};
  const NodeRec* PB[3] = {&B[0], &B[1], &B[2]};
  double f[3][5];
  chandrashekar_cart_v2<3>(PA, PB, gm1, f);
#pragma unroll
  for (int z = 0; z < 3; ++z) {
    double g[5];
#pragma unroll
    for (int v = 0; v < 5; ++v) g[v] = __shfl_sync(0xffffffffu, f[z][v], srcF);
    add_rot3(acc[z], cOwn, f[z], J);
    add_rot3(acc[z], cRecv, g, J);
  }
}

__global__ void __launch_bounds__(SFB_N3_THREADS, SFB_N3_MINB)
    euler_cart_n3_kernel(int64_t E, const __grid_constant__ DMat<3> Dm, double gm1,
                         const double* __restrict__ U,
                         double* __restrict__ R) {
  constexpr int N = 3, NN = 27, KU = 135;
  const double hgm1 = 0.5 * gm1;
  const int lane = threadIdx.x & 31;
  const int slot = lane < 27 ? lane / 9 : 0;  // element of the warp's three
  const int w = lane < 27 ? lane - slot * 9 : lane - 27;  // thread of the element (shadow)
  const int x0 = w % 3, x1 = w / 3;
  const int gbase = slot * 9;
  // shuffle partners and coefficients: direction 0 pairs (x0, x0+1), received
  // from (x0-1); direction 1 likewise in x1
  const int p0 = gbase + (x0 + 1) % 3 + 3 * x1, q0 = gbase + (x0 + 2) % 3 + 3 * x1;
  const int p1 = gbase + x0 + 3 * ((x1 + 1) % 3), q1 = gbase + x0 + 3 * ((x1 + 2) % 3);
  const double cO0 = Dm.d[x0 * N + (x0 + 1) % 3], cR0 = Dm.d[x0 * N + (x0 + 2) % 3];
  const double cO1 = Dm.d[x1 * N + (x1 + 1) % 3], cR1 = Dm.d[x1 * N + (x1 + 2) % 3];
  const double dd0 = Dm.d[x0 * (N + 1)], dd1 = Dm.d[x1 * (N + 1)];
  const int64_t warps_total = (int64_t)gridDim.x * (blockDim.x / 32);
  const int64_t warp_id = (int64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  // warp-uniform loop over groups of three elements
  for (int64_t g3 = warp_id; 3 * g3 < E; g3 += warps_total) {
    const int64_t e_raw = 3 * g3 + slot;
    const bool valid = lane < 27 && e_raw < E;
    const int64_t e = valid ? e_raw : 3 * g3;
    const double* u = U + e * KU + x0 + 3 * x1;
#if SFB_N3_L2PF
    {  // the warp's next three elements (3.2 KB contiguous) into L2
      const int64_t ng = g3 + warps_total;
      if (lane == 0 && 3 * ng < E) {
        const int64_t ne = (E - 3 * ng) < 3 ? (E - 3 * ng) : 3;
        // 16-byte granules inside [first, last) of the three elements
        const uintptr_t a0 = (uintptr_t)(U + 3 * ng * KU) & ~(uintptr_t)15;
        const uintptr_t a1 = (uintptr_t)(U + (3 * ng + ne) * KU) & ~(uintptr_t)15;
        if (a1 > a0)
          asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a0),
                       "r"((uint32_t)(a1 - a0))
                       : "memory");
      }
    }
#endif
    NodeRec rq[3];
    double acc[3][5];
#pragma unroll
    for (int z = 0; z < 3; ++z) {
      const double rho = __ldcs(u + 9 * z), m0 = __ldcs(u + NN + 9 * z),
                   m1 = __ldcs(u + 2 * NN + 9 * z), m2 = __ldcs(u + 3 * NN + 9 * z),
                   et = __ldcs(u + 4 * NN + 9 * z);
      const double irho = rcp_refined(rho);
      const double hirho = 0.5 * irho;
      const double mm = fma(m2, m2, fma(m1, m1, m0 * m0));
      const double X2 = fma(rho, et + et, -mm);
      const double iX2 = rcp_refined(X2);
      const double p = (hgm1 * X2) * irho;
      const double hbeta = (rho * rho) * iX2;
      rq[z].hr = 0.5 * rho;
      rq[z].hv0 = m0 * hirho;
      rq[z].hv1 = m1 * hirho;
      rq[z].hv2 = m2 * hirho;
      rq[z].hb = hbeta;
      rq[z].hlr = log_half_tab(rho);
      rq[z].hlb = log_half_tab(hbeta);
      const double dd2 = Dm.d[z * (N + 1)];
      const double mass = fma(m2, dd2, fma(m1, dd1, m0 * dd0));
      const double wv = mass * irho;
      acc[z][0] = mass;
      acc[z][1] = fma(m0, wv, p * dd0);
      acc[z][2] = fma(m1, wv, p * dd1);
      acc[z][3] = fma(m2, wv, p * dd2);
      acc[z][4] = (et + p) * wv;
    }
    // direction 2: the thread's own line, pairs (0,1), (0,2), (1,2)
    {
      const NodeRec a0 = rot3(rq[0], 2), a1 = rot3(rq[1], 2), a2 = rot3(rq[2], 2);
      const NodeRec* PA[3] = {&a0, &a0, &a1};
      const NodeRec* PB[3] = {&a1, &a2, &a2};
      double f[3][5];
      chandrashekar_cart_v2<3>(PA, PB, gm1, f);
      add_rot3(acc[0], Dm.d[0 * N + 1], f[0], 2);
      add_rot3(acc[1], Dm.d[1 * N + 0], f[0], 2);
      add_rot3(acc[0], Dm.d[0 * N + 2], f[1], 2);
      add_rot3(acc[2], Dm.d[2 * N + 0], f[1], 2);
      add_rot3(acc[1], Dm.d[1 * N + 2], f[2], 2);
      add_rot3(acc[2], Dm.d[2 * N + 1], f[2], 2);
    }
    cross_dir<0>(rq, p0, q0, cO0, cR0, gm1, acc);
    cross_dir<1>(rq, p1, q1, cO1, cR1, gm1, acc);
    if (valid) {
      double* r = R + e * KU + x0 + 3 * x1;
#pragma unroll
      for (int z = 0; z < 3; ++z)
#pragma unroll
        for (int v = 0; v < 5; ++v) __stcs(r + v * NN + 9 * z, acc[z][v]);
    }
  }
}

}  // namespace

int launch_euler_cart_n3(int64_t E, const double* Dh, double gamma, double scale,
                         const double* U, double* R, cudaStream_t s) {
  DMat<3> Dm;
  for (int k = 0; k < 9; ++k) Dm.d[k] = scale * Dh[k];
  static DeviceCache cache;
  const int ps = resident_ctas(euler_cart_n3_kernel, SFB_N3_THREADS, 0, cache);
  int64_t grid = (int64_t)num_sms() * ps;
  const int64_t warps = (E + 2) / 3;
  const int64_t need = (warps * 32 + SFB_N3_THREADS - 1) / SFB_N3_THREADS;
  if (grid > need) grid = need;
  euler_cart_n3_kernel<<<(unsigned)grid, SFB_N3_THREADS, 0, s>>>(E, Dm, gamma - 1.0, U, R);
  return check_launch("euler_volume_cartesian");
}

}  // namespace sfb
