// K3 variant (n = 4): no warp specialisation.  Every warp of a small CTA does
// the pair work of block it, the store of block it, and then - together - the
// node records of block it+1 (whose states the bulk copy brought in during
// block it).  Three CTA barriers per block; several CTAs per SM overlap each
// other's barriers.  Kept as a measured alternative to euler.cu's prep/line
// split.  Default for n = 4 (SFB_FUSED_N4=1): measured
// 0.587 ms vs 0.611 ms for the warp-specialised kernel.
#include "euler_common.cuh"

#ifndef SFB_FUSED_MINBLOCKS
#define SFB_FUSED_MINBLOCKS 3
#endif
#ifndef SFB_FUSED_EPB
#define SFB_FUSED_EPB 2
#endif
#ifndef SFB_FUSED_K
#define SFB_FUSED_K 3
#endif

namespace sfb {

struct Fused4Cfg {
  static constexpr int N = 4;
  static constexpr int NN = 64;
  static constexpr int kEPB = SFB_FUSED_EPB;
  static constexpr int kThreads = 3 * 16 * kEPB;  // one thread per line; warps direction-uniform
  static constexpr int kVals = kEPB * 5 * NN;
  static constexpr int kRecVals = 8 * kEPB * NN;
  static constexpr size_t kSmem = (size_t)(2 * kVals + 2 * kRecVals + 3 * kVals + 8) * sizeof(double);
};

__global__ void __launch_bounds__(Fused4Cfg::kThreads, SFB_FUSED_MINBLOCKS)
    euler_cart4_fused_kernel(int64_t E, const DMat<4> Dm, double gm1, double c_gamma,
                             double gam_ratio, const double* __restrict__ U,
                             double* __restrict__ R) {
  using Cfg = Fused4Cfg;
  constexpr int N = 4, NN = 64, EPB = Cfg::kEPB, kVals = Cfg::kVals, S = EPB * NN;
  constexpr int T = Cfg::kThreads;
  extern __shared__ __align__(16) double smem[];
  double* ibuf = smem;                      // [2][kVals]
  double* recb = smem + 2 * kVals;          // [2][8][S]
  double* resb = recb + 2 * Cfg::kRecVals;  // [3][kVals]
  double* ddiag = resb + 3 * kVals;
  __shared__ uint64_t full[2];
  const int tid = threadIdx.x;
  const int64_t nblocks = (E + EPB - 1) / EPB;
  const int niter = blockIdx.x < nblocks ? (int)((nblocks - 1 - blockIdx.x) / gridDim.x) + 1 : 0;
  const double c_hbeta = 0.5 * c_gamma;
  if (tid == 0) {
#pragma unroll
    for (int i = 0; i < N; ++i) ddiag[i] = Dm.d[i * N + i];
    mbar_init(&full[0], 1);
    mbar_init(&full[1], 1);
    fence_mbar_init();
  }
  __syncthreads();
  auto nel_of = [&](int64_t blk) {
    const int64_t e0 = blk * EPB;
    return (E - e0) < EPB ? (int)(E - e0) : EPB;
  };
  auto issue = [&](int it) {
    const int64_t blk = (int64_t)blockIdx.x + (int64_t)it * gridDim.x;
    const uint32_t bytes = (uint32_t)nel_of(blk) * 5 * NN * 8;
    mbar_arrive_expect_tx(&full[it & 1], bytes);
    bulk_g2s(ibuf + (it & 1) * kVals, U + blk * EPB * 5 * NN, bytes, &full[it & 1]);
  };
  auto prep = [&](int it) {  // node records of this CTA's it-th block into set it&1
    const double* in = ibuf + (it & 1) * kVals;
    double* rec = recb + (it & 1) * Cfg::kRecVals;
    for (int i = tid; i < S; i += T) {
      const int e = i / NN, r = i - e * NN;
      const double* uu = in + e * 5 * NN + r;
      const double rho = uu[0], m0 = uu[NN], m1 = uu[2 * NN], m2 = uu[3 * NN], et = uu[4 * NN];
      const double hirho = 0.5 * rcp_refined(rho);
      const double mm = fma(m2, m2, fma(m1, m1, m0 * m0));
      const double X = fma(rho, et, -0.5 * mm);
      const double iX = rcp_refined(X);
      const double p = (2.0 * gm1) * X * hirho;
      const double hbeta = (rho * rho) * (c_hbeta * iX);
      const int q = e * NN + swz<N>(r % N, (r / N) % N, r / (N * N));
      rec[q] = 0.5 * rho;
      rec[S + q] = m0 * hirho;
      rec[2 * S + q] = m1 * hirho;
      rec[3 * S + q] = m2 * hirho;
      rec[4 * S + q] = hbeta;
      rec[5 * S + q] = log_half(rho);
      rec[6 * S + q] = log_half(2.0 * hbeta);
      rec[7 * S + q] = p;
    }
  };

  const int dir = tid / (EPB * 16);
  const int rem = tid - dir * EPB * 16;
  const int el = rem / 16, L = rem - el * 16;
  const int u = L % N, w = L / N;
  int pos[N];
#pragma unroll
  for (int a = 0; a < N; ++a) {
    const int r0 = dir == 0 ? a : u;
    const int r1 = dir == 1 ? a : (dir == 0 ? u : w);
    const int r2 = dir == 2 ? a : w;
    pos[a] = swz<N>(r0, r1, r2);
  }
  const int vp0 = (1 + dir) * S, vp1 = (1 + (dir + 1) % 3) * S, vp2 = (1 + (dir + 2) % 3) * S;
  const int mp0 = (1 + dir) * NN, mp1 = (1 + (dir + 1) % 3) * NN, mp2 = (1 + (dir + 2) % 3) * NN;

  uint32_t parity_bits = 0;
  if (niter > 0) {
    if (tid == 0) {
      issue(0);
      if (niter > 1) issue(1);
    }
    mbar_wait_parity(&full[0], 0);
    parity_bits ^= 1u;
    prep(0);
    __syncthreads();
    if (tid == 0 && niter > 2) {  // slot 0 consumed by prep(0)
      fence_proxy_async_smem();
      issue(2);
    }
  }
  for (int it = 0; it < niter; ++it) {
    const int s = it & 1;
    const double* rec = recb + s * Cfg::kRecVals + el * NN;
    // ---- pair work ----------------------------------------------------------
    double acc[N][5];
#pragma unroll
    for (int a = 0; a < N; ++a)
#pragma unroll
      for (int v = 0; v < 5; ++v) acc[a][v] = 0.0;
    {
      NodeRec nrec[N];
#pragma unroll
      for (int a = 0; a < N; ++a) {
        const double* pr = rec + pos[a];
        nrec[a].hr = pr[0];
        nrec[a].hv0 = pr[vp0];
        nrec[a].hv1 = pr[vp1];
        nrec[a].hv2 = pr[vp2];
        nrec[a].hb = pr[4 * S];
        nrec[a].hlr = pr[5 * S];
        nrec[a].hlb = pr[6 * S];
      }
      constexpr PairOrder<N> po;
      constexpr int P = PairOrder<N>::kPairs;
      constexpr int K = SFB_FUSED_K;
#pragma unroll
      for (int k0 = 0; k0 < P; k0 += K) {
        const NodeRec* A[K];
        const NodeRec* B[K];
#pragma unroll
        for (int k = 0; k < K; ++k) {
          const int kk = (k0 + k < P) ? k0 + k : P - 1;
          A[k] = &nrec[po.a[kk]];
          B[k] = &nrec[po.b[kk]];
        }
        double f[K][5];
        chandrashekar_cart_k<K>(A, B, c_gamma, f);
#pragma unroll
        for (int k = 0; k < K; ++k) {
          if (k0 + k >= P) break;
          const int a = po.a[k0 + k], b = po.b[k0 + k];
          const double dab = Dm.d[a * N + b], dba = Dm.d[b * N + a];
#pragma unroll
          for (int v = 0; v < 5; ++v) {
            acc[a][v] = fma(dab, f[k][v], acc[a][v]);
            acc[b][v] = fma(dba, f[k][v], acc[b][v]);
          }
        }
      }
    }
    {
      double* rs = resb + dir * kVals + el * 5 * NN;
#pragma unroll
      for (int a = 0; a < N; ++a) {
        rs[pos[a]] = acc[a][0];
        rs[pos[a] + mp0] = acc[a][1];
        rs[pos[a] + mp1] = acc[a][2];
        rs[pos[a] + mp2] = acc[a][3];
        rs[pos[a] + 4 * NN] = acc[a][4];
      }
    }
    __syncthreads();
    // ---- store: diag + sum of the directions --------------------------------
    {
      const int64_t blk = (int64_t)blockIdx.x + (int64_t)it * gridDim.x;
      const int64_t e0 = blk * EPB;
      const int nn = nel_of(blk) * NN;
      const double* recs = recb + s * Cfg::kRecVals;
      double* Rb = R + e0 * 5 * NN;
      for (int i = tid; i < nn; i += T) {
        const int e = i / NN, r = i - e * NN;
        const int c0 = r % N, c1 = (r / N) % N, c2 = r / (N * N);
        const int qn = swz<N>(c0, c1, c2);
        const double* rc = recs + e * NN + qn;
        const double hr = rc[0], h0 = rc[S], h1 = rc[2 * S], h2 = rc[3 * S], p = rc[7 * S];
        const double q = fma(h2, h2, fma(h1, h1, h0 * h0));
        const double d0 = ddiag[c0], d1 = ddiag[c1], d2 = ddiag[c2];
        const double wv = 2.0 * fma(d2, h2, fma(d1, h1, d0 * h0));
        const double rw = 2.0 * hr * wv;
        const double ep = fma(gam_ratio, p, 4.0 * hr * q);
        const double diag[5] = {rw, fma(2.0 * rw, h0, p * d0), fma(2.0 * rw, h1, p * d1),
                                fma(2.0 * rw, h2, p * d2), ep * wv};
        const double* r0 = resb + e * 5 * NN + qn;
#pragma unroll
        for (int v = 0; v < 5; ++v)
          __stcs(Rb + e * 5 * NN + v * NN + r,
                 ((diag[v] + r0[v * NN]) + r0[kVals + v * NN]) + r0[2 * kVals + v * NN]);
      }
    }
    // ---- records of the next block (its states arrived during this block) -----
    if (it + 1 < niter) {
      const int ns = (it + 1) & 1;
      mbar_wait_parity(&full[ns], (parity_bits >> ns) & 1u);
      parity_bits ^= 1u << ns;
      prep(it + 1);
    }
    __syncthreads();
    if (tid == 0 && it + 3 < niter) {  // slot (it+1)&1 consumed by prep(it+1)
      fence_proxy_async_smem();
      issue(it + 3);
    }
  }
}

int launch_euler_cart4_fused(int64_t E, const double* Dh, double gamma, double scale,
                             const double* U, double* R, cudaStream_t s) {
  using Cfg = Fused4Cfg;
  DMat<4> Dm;
  for (int i = 0; i < 16; ++i) Dm.d[i] = scale * Dh[i];
  static int per_sm = 0;
  if (per_sm == 0) {
    cudaFuncSetAttribute(euler_cart4_fused_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)Cfg::kSmem);
    int b = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, euler_cart4_fused_kernel, Cfg::kThreads,
                                                  Cfg::kSmem);
    per_sm = b > 0 ? b : 1;
  }
  const int64_t nblocks = (E + Cfg::kEPB - 1) / Cfg::kEPB;
  int64_t grid = (int64_t)num_sms() * per_sm;
  if (grid > nblocks) grid = nblocks;
  const double gm1 = gamma - 1.0;
  euler_cart4_fused_kernel<<<(unsigned)grid, Cfg::kThreads, Cfg::kSmem, s>>>(
      E, Dm, gm1, 1.0 / (2.0 * gm1), gamma / gm1, U, R);
  return check_launch("euler_volume_cartesian(n=4, fused roles)");
}

}  // namespace sfb
