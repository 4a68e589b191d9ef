// K3 at n = 2 (config 4's first point): the Cartesian Euler volume term
//
//   R[e,:,r] = scale * sum_j sum_l D[r_j,l] F#_j(U[e,:,r], U[e,:,r(j->l)])
//
// (burgers.py:117-131 generalised, as euler.cu) with everything in registers:
// an n = 2 element has 8 nodes and 12 pairs (one per line, 4 lines per
// direction), so two threads (lanes 2k, 2k+1) own one element, each the four
// nodes of one x2 layer (h = x2, local node q = x0 + 2 x1, node r = q + 4h).
// Per thread: five 32-byte loads (the layer's four nodes of each variable,
// consecutive lanes -> consecutive bytes), the four node records and diagonal
// terms, the four pairs inside the layer (directions 0 and 1), then two of the
// four x2 pairs: the partner layer's records come by shuffles (lane ^ 1), and
// each evaluated F goes back the same way for the other layer's node.  No shared memory,
// no barriers: the warp kernel this replaces at n = 2 was shared-memory bound
// (mio_throttle + short_scoreboard 63% of the stalls, profiles/r02/ncu_c4_n2.txt).
#include "euler_common.cuh"

namespace sfb {

namespace {

__device__ __forceinline__ NodeRec rotate(const NodeRec& a, int j) {
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

// acc[0..4] += c * f with the momentum components of f (in direction j's
// rotated frame) put back in place
__device__ __forceinline__ void add_rot(double (&acc)[5], double c, const double (&f)[5], int j) {
  acc[0] = fma(c, f[0], acc[0]);
  acc[1 + j] = fma(c, f[1], acc[1 + j]);
  acc[1 + (j + 1) % 3] = fma(c, f[2], acc[1 + (j + 1) % 3]);
  acc[1 + (j + 2) % 3] = fma(c, f[3], acc[1 + (j + 2) % 3]);
  acc[4] = fma(c, f[4], acc[4]);
}

__device__ __forceinline__ NodeRec shfl_rec_xor(const NodeRec& q, int m) {
  NodeRec r;
  r.hr = __shfl_xor_sync(0xffffffffu, q.hr, m);
  r.hv0 = __shfl_xor_sync(0xffffffffu, q.hv0, m);
  r.hv1 = __shfl_xor_sync(0xffffffffu, q.hv1, m);
  r.hv2 = __shfl_xor_sync(0xffffffffu, q.hv2, m);
  r.hb = __shfl_xor_sync(0xffffffffu, q.hb, m);
  r.hlr = __shfl_xor_sync(0xffffffffu, q.hlr, m);
  r.hlb = __shfl_xor_sync(0xffffffffu, q.hlb, m);
  return r;
}

#ifndef SFB_N2_L2PF
#define SFB_N2_L2PF 0  // L2 prefetch of the warp's next 16 elements: 0.312 vs 0.306 ms
#endif
#ifndef SFB_N2_THREADS
#define SFB_N2_THREADS 128
#endif
#ifndef SFB_N2_MINB
#define SFB_N2_MINB 3  // 12 warps per SM at 162 registers: 0.306 ms (256 x 2 at 128 regs, spilling: 0.327)
#endif

__global__ void __launch_bounds__(SFB_N2_THREADS, SFB_N2_MINB) euler_cart_n2_kernel(int64_t E, const DMat<2> Dm,
                                                            double gm1,
                                                            const double* __restrict__ U,
                                                            double* __restrict__ R) {
  constexpr int NN = 8, KU = 40;
  const double hgm1 = 0.5 * gm1;
  const double d00 = Dm.d[0], d01 = Dm.d[1], d10 = Dm.d[2], d11 = Dm.d[3];
  const int lane = threadIdx.x & 31;
  const int h = lane & 1;
  const int64_t nthreads = 2 * E;
  const int64_t wstride = (int64_t)gridDim.x * blockDim.x;
  // warp-uniform loop (the shuffles need both lanes of every element)
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31); base < nthreads;
       base += wstride) {
    const int64_t t = base + lane;
    const bool valid = t < nthreads;
    const int64_t e = valid ? t >> 1 : 0;
    const double* u = U + e * KU + 4 * h;
#if SFB_N2_L2PF
    {  // the warp's next 16 elements (5 KB contiguous) into L2 while this one computes
      const int64_t nb = base + wstride;
      if (lane == 0 && nb < nthreads) {
        const int64_t e0 = nb >> 1;
        const int64_t ne = (E - e0) < 16 ? (E - e0) : 16;
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(U + e0 * KU),
                     "r"((uint32_t)(ne * KU * 8))
                     : "memory");
      }
    }
#endif
    // ---- node records + diagonal terms of this layer --------------------------
    double st[5][4];
#pragma unroll
    for (int v = 0; v < 5; ++v) {
      const double2 a = ld_stream_d2(u + v * NN);
      const double2 b = ld_stream_d2(u + v * NN + 2);
      st[v][0] = a.x;
      st[v][1] = a.y;
      st[v][2] = b.x;
      st[v][3] = b.y;
    }
    NodeRec rq[4];
    double acc[4][5];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const double rho = st[0][q], m0 = st[1][q], m1 = st[2][q], m2 = st[3][q], et = st[4][q];
      const double irho = rcp_refined(rho);
      const double hirho = 0.5 * irho;
      const double mm = fma(m2, m2, fma(m1, m1, m0 * m0));
      const double X2 = fma(rho, et + et, -mm);
      const double iX2 = rcp_refined(X2);
      const double p = (hgm1 * X2) * irho;
      const double hbeta = (rho * rho) * iX2;
      rq[q].hr = 0.5 * rho;
      rq[q].hv0 = m0 * hirho;
      rq[q].hv1 = m1 * hirho;
      rq[q].hv2 = m2 * hirho;
      rq[q].hb = hbeta;
      rq[q].hlr = log_half_tab(rho);
      rq[q].hlb = log_half_tab(hbeta);
      // digits (x0, x1, x2) = (q & 1, q >> 1, h): D[r_j][r_j]
      const double dd0 = (q & 1) ? d11 : d00, dd1 = (q >> 1) ? d11 : d00, dd2 = h ? d11 : d00;
      const double mass = fma(m2, dd2, fma(m1, dd1, m0 * dd0));
      const double wv = mass * irho;
      acc[q][0] = mass;
      acc[q][1] = fma(m0, wv, p * dd0);
      acc[q][2] = fma(m1, wv, p * dd1);
      acc[q][3] = fma(m2, wv, p * dd2);
      acc[q][4] = (et + p) * wv;
    }
    // ---- the four pairs inside the layer: direction 0 (q, q^1), 1 (q, q^2) ----
    {
      const NodeRec a0 = rq[0], a1 = rq[2], a2 = rq[0], a3 = rq[1];
      const NodeRec b0 = rq[1], b1 = rq[3], b2 = rq[2], b3 = rq[3];
      const NodeRec A0 = rotate(a0, 0), A1 = rotate(a1, 0), B0 = rotate(b0, 0),
                    B1 = rotate(b1, 0);
      const NodeRec A2 = rotate(a2, 1), A3 = rotate(a3, 1), B2 = rotate(b2, 1),
                    B3 = rotate(b3, 1);
      {
        const NodeRec* PA[2] = {&A0, &A1};
        const NodeRec* PB[2] = {&B0, &B1};
        double f[2][5];
        chandrashekar_cart_v2<2>(PA, PB, gm1, f);
        add_rot(acc[0], d01, f[0], 0);
        add_rot(acc[1], d10, f[0], 0);
        add_rot(acc[2], d01, f[1], 0);
        add_rot(acc[3], d10, f[1], 0);
      }
      {
        const NodeRec* PA[2] = {&A2, &A3};
        const NodeRec* PB[2] = {&B2, &B3};
        double f[2][5];
        chandrashekar_cart_v2<2>(PA, PB, gm1, f);
        add_rot(acc[0], d01, f[0], 1);
        add_rot(acc[2], d10, f[0], 1);
        add_rot(acc[1], d01, f[1], 1);
        add_rot(acc[3], d10, f[1], 1);
      }
    }
    // ---- direction 2: pairs (q, q + 4); layer 0 evaluates q = 0, 1, layer 1
    //      q = 2, 3 (its nodes 6, 7 with nodes 2, 3 of layer 0) -------------------
    {
      // each lane sends the two records the other layer needs: layer 0 its
      // q = 2, 3, layer 1 its q = 0, 1
      const NodeRec s0 = h ? rq[0] : rq[2];
      const NodeRec s1 = h ? rq[1] : rq[3];
      const NodeRec p0 = shfl_rec_xor(s0, 1), p1 = shfl_rec_xor(s1, 1);
      const NodeRec o0 = h ? rq[2] : rq[0];  // own node of each evaluated pair
      const NodeRec o1 = h ? rq[3] : rq[1];
      const NodeRec A0 = rotate(o0, 2), A1 = rotate(o1, 2), B0 = rotate(p0, 2),
                    B1 = rotate(p1, 2);
      const NodeRec* PA[2] = {&A0, &A1};
      const NodeRec* PB[2] = {&B0, &B1};
      double f[2][5];
      chandrashekar_cart_v2<2>(PA, PB, gm1, f);
      // every direction-2 pair joins a node of layer 0 and one of layer 1, so
      // both what a lane evaluated and what it receives land on its own layer's
      // nodes with the coefficient D[h][1-h]
      const double c = h ? d10 : d01;
      double g[2][5];
#pragma unroll
      for (int k = 0; k < 2; ++k)
#pragma unroll
        for (int v = 0; v < 5; ++v) g[k][v] = __shfl_xor_sync(0xffffffffu, f[k][v], 1);
      // layer 0 owns pairs with its q = 0, 1 and receives for its q = 2, 3;
      // layer 1 owns its q = 2, 3 and receives for its q = 0, 1
      if (h == 0) {
        add_rot(acc[0], c, f[0], 2);
        add_rot(acc[1], c, f[1], 2);
        add_rot(acc[2], c, g[0], 2);
        add_rot(acc[3], c, g[1], 2);
      } else {
        add_rot(acc[2], c, f[0], 2);
        add_rot(acc[3], c, f[1], 2);
        add_rot(acc[0], c, g[0], 2);
        add_rot(acc[1], c, g[1], 2);
      }
    }
    if (valid) {
      double* r = R + e * KU + 4 * h;
#pragma unroll
      for (int v = 0; v < 5; ++v) {
        st_stream_d2(r + v * NN, make_double2(acc[0][v], acc[1][v]));
        st_stream_d2(r + v * NN + 2, make_double2(acc[2][v], acc[3][v]));
      }
    }
  }
}

}  // namespace

int launch_euler_cart_n2(int64_t E, const double* Dh, double gamma, double scale,
                         const double* U, double* R, cudaStream_t s) {
  DMat<2> Dm;
  for (int k = 0; k < 4; ++k) Dm.d[k] = scale * Dh[k];
  static DeviceCache cache;
  const int ps = resident_ctas(euler_cart_n2_kernel, SFB_N2_THREADS, 0, cache);
  int64_t grid = (int64_t)num_sms() * ps;
  const int64_t need = (2 * E + SFB_N2_THREADS - 1) / SFB_N2_THREADS;
  if (grid > need) grid = need;
  euler_cart_n2_kernel<<<(unsigned)grid, SFB_N2_THREADS, 0, s>>>(E, Dm, gamma - 1.0, U, R);
  return check_launch("euler_volume_cartesian");
}

}  // namespace sfb
