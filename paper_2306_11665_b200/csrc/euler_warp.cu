// K3, n = 4, warp-autonomous: every warp owns a private pipeline over pairs of
// elements and never waits on another warp.
//
// Why: the CTA-wide variants (euler.cu, euler_fused.cu) map one thread to one
// line, so a CTA has 3/4 as many threads as nodes and the per-node stages
// (records, store) split unevenly over its warps; ncu put ~26% of warp
// samples on the CTA barriers around them.  Here one lane owns one line in
// EVERY direction (16 lanes per element, 2 elements per warp), so each lane
// does exactly 4 nodes of records, one line per direction and 4 nodes of
// store: no imbalance, and __syncwarp is the only synchronisation.
//
// Per warp and element pair (smem, 17 KB per warp):
//   slot  [5][2*64]  conserved states of the pair (one bulk copy)
//   rec   [7][2*64]  node records hr, hv0..2, hb, hlr, hlb (swizzled nodes;
//                    hb = (gamma-1) beta, see chandrashekar_cart_v2)
//   res   [5][2*64]  residual accumulator, seeded with the diagonal term
// Phases: records + diagonal (slot -> rec, res); refill the slot with the
// next pair (bulk copy, lands during the line work); lines along x2 and x1
// (read-modify-write res); lines along x0 add res and store straight to HBM
// (a lane's x0 line is 4 contiguous doubles of every variable).
#include "euler_common.cuh"

#ifndef SFB_WARP_WPC
#define SFB_WARP_WPC 1  // warps per CTA
#endif
#ifndef SFB_WARP_K
#define SFB_WARP_K 3
#endif
#ifndef SFB_EXP_NO_PREP
#define SFB_EXP_NO_PREP 0
#endif
#ifndef SFB_WARP_LDG
#define SFB_WARP_LDG 1  // states read straight from HBM/L2 (no smem slot)
#endif
#ifndef SFB_EXP_NO_MEM
#define SFB_EXP_NO_MEM 0
#endif
#ifndef SFB_EXP_NO_LINE
#define SFB_EXP_NO_LINE 0
#endif
#ifndef SFB_WARP_MINBLOCKS
#define SFB_WARP_MINBLOCKS 12
#endif

namespace sfb {

namespace {
constexpr int kN = 4, kNN = 64, kEPW = 2, kS = kEPW * kNN;  // nodes per warp block
constexpr int kSlotVals = kEPW * 5 * kNN;
constexpr int kWarpVals = (SFB_WARP_LDG ? 0 : kSlotVals) + 7 * kS + 5 * kS;
constexpr size_t kWarpSmem = (size_t)kWarpVals * sizeof(double);
}  // namespace

// Accumulate the 6 pairs of one line (nodes pos[0..3] in the swizzled record
// planes, velocity planes permuted so plane vp0 is along the line).
__device__ __forceinline__ void line_pairs4(const double* __restrict__ rec, const int (&pos)[4],
                                            int vp0, int vp1, int vp2, const DMat<4> Dm,
                                            double gm1, double (&acc)[4][5]) {
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int v = 0; v < 5; ++v) acc[a][v] = 0.0;
  if (SFB_EXP_NO_LINE) return;  // ablation builds only
  NodeRec nrec[4];
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    const double* pr = rec + pos[a];
    nrec[a].hr = pr[0];
    nrec[a].hv0 = pr[vp0];
    nrec[a].hv1 = pr[vp1];
    nrec[a].hv2 = pr[vp2];
    nrec[a].hb = pr[4 * kS];
    nrec[a].hlr = pr[5 * kS];
    nrec[a].hlb = pr[6 * kS];
    nrec[a].q = 0.0;
  }
  constexpr PairOrder<4> po;
  constexpr int P = PairOrder<4>::kPairs;
  constexpr int K = SFB_WARP_K;
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
    chandrashekar_cart_v2<K>(A, B, gm1, f);
#pragma unroll
    for (int k = 0; k < K; ++k) {
      if (k0 + k >= P) break;
      const int a = po.a[k0 + k], b = po.b[k0 + k];
      const double dab = Dm.d[a * 4 + b], dba = Dm.d[b * 4 + a];
#pragma unroll
      for (int v = 0; v < 5; ++v) {
        acc[a][v] = fma(dab, f[k][v], acc[a][v]);
        acc[b][v] = fma(dba, f[k][v], acc[b][v]);
      }
    }
  }
}

__global__ void __launch_bounds__(32 * SFB_WARP_WPC, SFB_WARP_MINBLOCKS)
    euler_cart4_warp_kernel(int64_t E, const DMat<4> Dm, double gm1, double c_gamma,
                            double gam_ratio, const double* __restrict__ U,
                            double* __restrict__ R) {
  constexpr int N = kN, NN = kNN, S = kS;
  extern __shared__ __align__(16) double smem[];
  __shared__ uint64_t full[SFB_WARP_WPC];
  __shared__ double ddiag[4];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* slot = smem + warp * kWarpVals;
  double* rec = slot + (SFB_WARP_LDG ? 0 : kSlotVals);
  double* res = rec + 7 * S;
  if (threadIdx.x == 0) {  // static indices: a dynamic index would copy Dm to local memory
#pragma unroll
    for (int i = 0; i < 4; ++i) ddiag[i] = Dm.d[i * 5];
  }
  if (lane == 0) {
    mbar_init(&full[warp], 1);
    fence_mbar_init();
  }
  __syncthreads();  // the only CTA barrier

  const int64_t nwb = (E + kEPW - 1) / kEPW;  // warp blocks (element pairs)
  const int64_t g = (int64_t)blockIdx.x * SFB_WARP_WPC + warp;
  const int64_t G = (int64_t)gridDim.x * SFB_WARP_WPC;
  const int niter = g < nwb ? (int)((nwb - 1 - g) / G) + 1 : 0;
  auto nel_of = [&](int64_t wb) {
    const int64_t e0 = wb * kEPW;
    return (E - e0) < kEPW ? (int)(E - e0) : kEPW;
  };
  auto issue = [&](int it) {
    const int64_t wb = g + (int64_t)it * G;
    const uint32_t bytes = (uint32_t)nel_of(wb) * 5 * NN * 8;
    mbar_arrive_expect_tx(&full[warp], bytes);
    bulk_g2s(slot, U + wb * kEPW * 5 * NN, bytes, &full[warp]);
  };

  // this lane's line in each direction: element el, transverse (u, w)
  const int el = lane >> 4, L = lane & 15, u = L & 3, w = L >> 2;
  const double hgm1 = 0.5 * gm1;
  const double* rl = rec + el * NN;
  double* rs = res + el * NN;
  int pos2[N], pos1[N], pos0[N];
#pragma unroll
  for (int a = 0; a < N; ++a) {
    pos0[a] = swz<N>(a, u, w);
    pos1[a] = swz<N>(u, a, w);
    pos2[a] = swz<N>(u, w, a);
  }

  // the D diagonal at this lane's prep nodes (c0, c1 fixed per lane; c2 by j parity)
  const double dd0 = ddiag[lane & 3], dd1 = ddiag[(lane >> 2) & 3];
  const double dd2e = ddiag[lane >> 4], dd2o = ddiag[(lane >> 4) + 2];
  auto prefetch = [&](int it) {
    const int64_t wb = g + (int64_t)it * G;
    const uint32_t bytes = (uint32_t)nel_of(wb) * 5 * NN * 8;
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(U + wb * kEPW * 5 * NN),
                 "r"(bytes)
                 : "memory");
  };

  if (SFB_WARP_LDG) {
    if (lane == 0 && niter > 0) prefetch(0);
    if (lane == 0 && niter > 1) prefetch(1);
  } else if (niter > 0 && lane == 0) {
    issue(0);
  }
  for (int it = 0; it < niter; ++it) {
    const int64_t wb = g + (int64_t)it * G;
    const int nel = nel_of(wb);
    if (SFB_WARP_LDG) {
      if (lane == 0 && it + 2 < niter) prefetch(it + 2);
    } else if (!SFB_EXP_NO_MEM || it == 0) {
      mbar_wait_parity(&full[warp], it & 1);
    }
    // ---- node records + diagonal term (4 nodes per lane) ----------------------
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      if (SFB_EXP_NO_PREP && it > 0) break;  // ablation builds only
      const int i = lane + 32 * j;
      const int e = i >> 6, r = i & 63;
      double rho, m0, m1, m2, et;
      if (SFB_WARP_LDG) {
        const double* uu = U + (wb * kEPW + (e < nel ? e : 0)) * 5 * NN + r;
        rho = __ldcs(uu);
        m0 = __ldcs(uu + NN);
        m1 = __ldcs(uu + 2 * NN);
        m2 = __ldcs(uu + 3 * NN);
        et = __ldcs(uu + 4 * NN);
      } else {
        const double* uu = slot + e * 5 * NN + r;
        rho = uu[0], m0 = uu[NN], m1 = uu[2 * NN], m2 = uu[3 * NN], et = uu[4 * NN];
      }
      const double irho = rcp_refined(rho);
      const double hirho = 0.5 * irho;
      const double mm = fma(m2, m2, fma(m1, m1, m0 * m0));
      const double X2 = fma(rho, et + et, -mm);  // 2 (rho E - |m|^2/2)
      const double iX2 = rcp_refined(X2);
      const double p = (hgm1 * X2) * irho;
      const double hbeta = (rho * rho) * iX2;  // (gamma - 1) beta = rho^2 / (2X)
      const int c0 = r & 3, c1 = (r >> 2) & 3, c2 = r >> 4;
      const int q = e * NN + swz<N>(c0, c1, c2);
      rec[q] = 0.5 * rho;
      rec[S + q] = m0 * hirho;
      rec[2 * S + q] = m1 * hirho;
      rec[3 * S + q] = m2 * hirho;
      rec[4 * S + q] = hbeta;
      rec[5 * S + q] = log_half_tab(rho);
      rec[6 * S + q] = log_half_tab(hbeta);
      // diagonal term sum_j D_{c_j c_j} f_j(u, u): with mass = D.m and
      // w = mass / rho:  (mass, w m + p D, (E + p) w)
      const double d0 = dd0, d1 = dd1, d2 = (j & 1) ? dd2o : dd2e;
      const double mass = fma(d2, m2, fma(d1, m1, d0 * m0));
      const double wv = mass * irho;
      res[q] = mass;
      res[S + q] = fma(wv, m0, p * d0);
      res[2 * S + q] = fma(wv, m1, p * d1);
      res[3 * S + q] = fma(wv, m2, p * d2);
      res[4 * S + q] = (et + p) * wv;
    }
    __syncwarp();
    if (!SFB_WARP_LDG && !SFB_EXP_NO_MEM && lane == 0 && it + 1 < niter) {  // slot consumed: refill
      fence_proxy_async_smem();
      issue(it + 1);
    }
    double acc[N][5];
    // ---- lines along x2, then x1: read-modify-write the accumulator -----------
    line_pairs4(rl, pos2, 3 * S, 1 * S, 2 * S, Dm, gm1, acc);
#pragma unroll
    for (int a = 0; a < N; ++a) {
      double* p = rs + pos2[a];
      p[0] += acc[a][0];
      p[3 * S] += acc[a][1];
      p[S] += acc[a][2];
      p[2 * S] += acc[a][3];
      p[4 * S] += acc[a][4];
    }
    line_pairs4(rl, pos1, 2 * S, 3 * S, 1 * S, Dm, gm1, acc);
    __syncwarp();
#pragma unroll
    for (int a = 0; a < N; ++a) {
      double* p = rs + pos1[a];
      p[0] += acc[a][0];
      p[2 * S] += acc[a][1];
      p[3 * S] += acc[a][2];
      p[S] += acc[a][3];
      p[4 * S] += acc[a][4];
    }
    // ---- lines along x0: finish and store (4 contiguous doubles per variable) --
    line_pairs4(rl, pos0, 1 * S, 2 * S, 3 * S, Dm, gm1, acc);
    __syncwarp();
    if (SFB_EXP_NO_MEM ? (nel == 12345) : (el < nel)) {
      double* out = R + (wb * kEPW + el) * 5 * NN + 4 * L;
#pragma unroll
      for (int v = 0; v < 5; ++v) {
        // two 16-B stores: the ABI guarantees 16-B alignment of R
        st_stream_d2(out + v * NN, make_double2(rs[v * S + pos0[0]] + acc[0][v],
                                                rs[v * S + pos0[1]] + acc[1][v]));
        st_stream_d2(out + v * NN + 2, make_double2(rs[v * S + pos0[2]] + acc[2][v],
                                                    rs[v * S + pos0[3]] + acc[3][v]));
      }
    }
    __syncwarp();  // rec/res are rewritten by the next block's records
  }
}

int launch_euler_cart4_warp(int64_t E, const double* Dh, double gamma, double scale,
                            const double* U, double* R, cudaStream_t s) {
  constexpr int T = 32 * SFB_WARP_WPC;
  constexpr size_t smem = SFB_WARP_WPC * kWarpSmem;
  DMat<4> Dm;
  for (int i = 0; i < 16; ++i) Dm.d[i] = scale * Dh[i];
  static int per_sm = 0;
  if (per_sm == 0) {
    cudaFuncSetAttribute(euler_cart4_warp_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
    int b = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, euler_cart4_warp_kernel, T, smem);
    per_sm = b > 0 ? b : 1;
  }
  const int64_t nwb = (E + kEPW - 1) / kEPW;
  const int64_t ncta = (nwb + SFB_WARP_WPC - 1) / SFB_WARP_WPC;
  int64_t grid = (int64_t)num_sms() * per_sm;
  if (grid > ncta) grid = ncta;
  const double gm1 = gamma - 1.0;
  euler_cart4_warp_kernel<<<(unsigned)grid, T, smem, s>>>(E, Dm, gm1, 1.0 / (2.0 * gm1),
                                                          gamma / gm1, U, R);
  return check_launch("euler_volume_cartesian(n=4, warp-autonomous)");
}

}  // namespace sfb
