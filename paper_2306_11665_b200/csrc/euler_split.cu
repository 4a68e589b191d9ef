// K3 for n = 4 (the headline config 3): the Cartesian Euler volume term with
// each line split over TWO lanes.
//
// Same pipeline as euler.cu (persistent CTAs, one prep warp streaming the
// next block in with a bulk copy and building node records, line warps doing
// the pair work, the store stage adding the diagonal term), but a line's six
// pairs are shared by a lane pair (lane, lane^1) that each OWN two of its four
// rows:
//     lane A (h=0) owns rows {0,1}: pairs (0,1), (0,2), (1,3)
//     lane B (h=1) owns rows {2,3}: pairs (2,3), (2,1), (3,0)
// Each lane keeps D[own,oth] F for its own row and hands the raw flux F to its
// partner with one warp shuffle per cross pair; the partner applies
// D[oth,own].  Every pair is still evaluated exactly once, the FP64 count is
// unchanged, but a lane holds 10 accumulators instead of 20 and three
// independent flux chains, so twice as many line warps fit per SM and the
// FP64 pipe sees more independent work (it needs ~4 chains per warp,
// tools/peaks/fp64_latency.cu).  A warp is one (element, direction): 16 lines
// x 2 lanes, so all selects on the direction are warp-uniform.
#include "euler_common.cuh"

#ifndef SFB_SPLIT_EPB
#define SFB_SPLIT_EPB 1
#endif
#ifndef SFB_SPLIT_MINBLOCKS
#define SFB_SPLIT_MINBLOCKS 5
#endif

namespace sfb {

struct Split4Cfg {
  static constexpr int N = 4;
  static constexpr int kNodes = 64;
  static constexpr int kEPB = SFB_SPLIT_EPB;
  static constexpr int kLineThreads = 96 * kEPB;  // warps = (element, direction)
  static constexpr int kPrepT = 32;
  static constexpr int kThreads = kLineThreads + kPrepT;
  static constexpr int kVals = kEPB * 5 * kNodes;
  static constexpr int kPlanes = 8;  // 7 record planes + pressure
  static constexpr int kRecVals = kPlanes * kEPB * kNodes;
  static constexpr size_t kSmem = (size_t)(2 * kVals + 2 * kRecVals + 3 * kVals + 8) * sizeof(double);
};

__device__ __forceinline__ double shfl1(double x) { return __shfl_xor_sync(0xffffffffu, x, 1); }

__global__ void __launch_bounds__(Split4Cfg::kThreads, SFB_SPLIT_MINBLOCKS)
    euler_cart4_split_kernel(int64_t E, const DMat<4> Dm, double gm1, double c_gamma,
                             double gam_ratio, const double* __restrict__ U,
                             double* __restrict__ R) {
  using Cfg = Split4Cfg;
  constexpr int N = 4;
  constexpr int NN = Cfg::kNodes;
  constexpr int EPB = Cfg::kEPB;
  constexpr int kVals = Cfg::kVals;
  constexpr int S = EPB * NN;
  constexpr int kLineT = Cfg::kLineThreads;
  constexpr int kPrepT = Cfg::kPrepT;
  constexpr int kAll = Cfg::kThreads;
  enum { REC_FULL = 1, REC_EMPTY = 3, LINE_ONLY = 5, PREP_ONLY = 6 };
  extern __shared__ __align__(16) double smem[];
  double* ibuf = smem;                      // [2][EPB][5][NN] bulk-copy target
  double* recb = smem + 2 * kVals;          // [2][8][EPB*NN] swizzled records + p
  double* resb = recb + 2 * Cfg::kRecVals;  // [3][EPB][5][NN] swizzled direction residuals
  double* ddiag = resb + 3 * kVals;         // [N] scale*D[i][i]
  __shared__ uint64_t full[2];

  const int tid = threadIdx.x;
  const int64_t nblocks = (E + EPB - 1) / EPB;
  if (tid == 0) {
#pragma unroll
    for (int i = 0; i < N; ++i) ddiag[i] = Dm.d[i * N + i];
    mbar_init(&full[0], 1);
    mbar_init(&full[1], 1);
    fence_mbar_init();
  }
  __syncthreads();
  const int niter = blockIdx.x < nblocks ? (int)((nblocks - 1 - blockIdx.x) / gridDim.x) + 1 : 0;

  if (tid < kLineT) {
    // =========================== line warps ==================================
    const int w = tid >> 5, lane = tid & 31;
    const int el = w / 3, dir = w - 3 * el;
    const int L = lane >> 1, h = lane & 1;
    const int u = L % N, v2 = L / N;
    int pos[N];
#pragma unroll
    for (int a = 0; a < N; ++a) {
      const int r0 = dir == 0 ? a : u;
      const int r1 = dir == 1 ? a : (dir == 0 ? u : v2);
      const int r2 = dir == 2 ? a : v2;
      pos[a] = swz<N>(r0, r1, r2);
    }
    // own rows o0 = 2h, o1 = 2h+1; cross partners: lane A (0,2),(1,3); lane B (2,1),(3,0)
    const int p_o0 = h ? pos[2] : pos[0];
    const int p_o1 = h ? pos[3] : pos[1];
    const int p_x1 = h ? pos[1] : pos[2];
    const int p_x2 = h ? pos[0] : pos[3];
    const bool hb = h != 0;
    const double di0 = dsel(hb, Dm.d[2 * N + 3], Dm.d[0 * N + 1]);  // D[o0][o1]
    const double di1 = dsel(hb, Dm.d[3 * N + 2], Dm.d[1 * N + 0]);  // D[o1][o0]
    const double dk1 = dsel(hb, Dm.d[2 * N + 1], Dm.d[0 * N + 2]);  // D[o0][x1]
    const double dk2 = dsel(hb, Dm.d[3 * N + 0], Dm.d[1 * N + 3]);  // D[o1][x2]
    const double dr0 = dsel(hb, Dm.d[2 * N + 0], Dm.d[0 * N + 3]);  // received into o0
    const double dr1 = dsel(hb, Dm.d[3 * N + 1], Dm.d[1 * N + 2]);  // received into o1
    const int vp0 = (1 + dir) * S, vp1 = (1 + (dir + 1) % 3) * S, vp2 = (1 + (dir + 2) % 3) * S;
    const int mp0 = (1 + dir) * NN, mp1 = (1 + (dir + 1) % 3) * NN, mp2 = (1 + (dir + 2) % 3) * NN;
    for (int it = 0; it < niter; ++it) {
      const int s = it & 1;
      const double* rec = recb + s * Cfg::kRecVals + el * NN;
      nbar_sync(REC_FULL + s, kAll);
      auto load = [&](int p) {
        NodeRec q;
        const double* r = rec + p;
        q.hr = r[0];
        q.hv0 = r[vp0];  // rotated (normal, t1, t2) velocity
        q.hv1 = r[vp1];
        q.hv2 = r[vp2];
        q.hb = r[4 * S];
        q.hlr = r[5 * S];
        q.hlb = r[6 * S];
        q.q = 0.0;
        return q;
      };
      const NodeRec n0 = load(p_o0), n1 = load(p_o1), x1 = load(p_x1), x2 = load(p_x2);
      const NodeRec* A[3] = {&n0, &n0, &n1};
      const NodeRec* B[3] = {&n1, &x1, &x2};
      double f[3][5];
      chandrashekar_cart_k<3>(A, B, c_gamma, f);
      double a0[5], a1[5];
#pragma unroll
      for (int v = 0; v < 5; ++v) {
        a0[v] = fma(dk1, f[1][v], di0 * f[0][v]);
        a1[v] = fma(dk2, f[2][v], di1 * f[0][v]);
      }
#pragma unroll
      for (int v = 0; v < 5; ++v) {
        const double r1 = shfl1(f[1][v]);  // partner's first cross flux
        const double r2 = shfl1(f[2][v]);  // partner's second cross flux
        a0[v] = fma(dr0, dsel(hb, r1, r2), a0[v]);
        a1[v] = fma(dr1, dsel(hb, r2, r1), a1[v]);
      }
      double* rs = resb + dir * kVals + el * 5 * NN;
      rs[p_o0] = a0[0];
      rs[p_o0 + mp0] = a0[1];
      rs[p_o0 + mp1] = a0[2];
      rs[p_o0 + mp2] = a0[3];
      rs[p_o0 + 4 * NN] = a0[4];
      rs[p_o1] = a1[0];
      rs[p_o1 + mp0] = a1[1];
      rs[p_o1 + mp1] = a1[2];
      rs[p_o1 + mp2] = a1[3];
      rs[p_o1 + 4 * NN] = a1[4];
      nbar_sync(LINE_ONLY, kLineT);  // all three direction residuals written
      // residual = diag + (R_0 + R_1) + R_2 per node (diag from the node record)
      {
        const int64_t blk = (int64_t)blockIdx.x + (int64_t)it * gridDim.x;
        const int64_t e0 = blk * EPB;
        const int nel = (E - e0) < EPB ? (int)(E - e0) : EPB;
        const double* recs = recb + s * Cfg::kRecVals;
        double* Rb = R + e0 * 5 * NN;
        const int nn = nel * NN;
        for (int i = tid; i < nn; i += kLineT) {
          const int e = i / NN;
          const int r = i - e * NN;
          const int c0 = r % N, c1 = (r / N) % N, c2 = r / (N * N);
          const int qn = swz<N>(c0, c1, c2);
          const double* rc = recs + e * NN + qn;
          const double hr = rc[0], h0 = rc[S], h1 = rc[2 * S], h2 = rc[3 * S];
          const double p = rc[7 * S];
          const double q = fma(h2, h2, fma(h1, h1, h0 * h0));  // |v|^2 / 4
          const double d0 = ddiag[c0], d1 = ddiag[c1], d2 = ddiag[c2];
          const double wv = 2.0 * fma(d2, h2, fma(d1, h1, d0 * h0));  // sum_j d_j v_j
          const double rho = 2.0 * hr;
          const double rw = rho * wv;
          const double ep = fma(gam_ratio, p, 4.0 * hr * q);  // E + p
          const double diag[5] = {rw, fma(2.0 * rw, h0, p * d0), fma(2.0 * rw, h1, p * d1),
                                  fma(2.0 * rw, h2, p * d2), ep * wv};
          const double* r0 = resb + e * 5 * NN + qn;
          const double* r1 = r0 + kVals;
          const double* r2 = r1 + kVals;
#pragma unroll
          for (int v = 0; v < 5; ++v)
            __stcs(Rb + e * 5 * NN + v * NN + r,
                   ((diag[v] + r0[v * NN]) + r1[v * NN]) + r2[v * NN]);
        }
      }
      nbar_arrive(REC_EMPTY + s, kAll);  // record set s (incl. p) consumed
      nbar_sync(LINE_ONLY, kLineT);      // residual buffers free again
    }
  } else {
    // =========================== prep warp ===================================
    const int pt = tid - kLineT;
    auto block_bytes = [&](int64_t blk) {
      const int64_t e0 = blk * EPB;
      const int nel = (E - e0) < EPB ? (int)(E - e0) : EPB;
      return (uint32_t)nel * 5 * NN * 8;
    };
    auto issue = [&](int64_t blk, int slot) {
      const uint32_t bytes = block_bytes(blk);
      mbar_arrive_expect_tx(&full[slot], bytes);
      bulk_g2s(ibuf + slot * kVals, U + blk * EPB * 5 * NN, bytes, &full[slot]);
    };
    int64_t blk = blockIdx.x;
    if (pt == 0 && niter > 0) issue(blk, 0);
    uint32_t parity_bits = 0;
    for (int it = 0; it < niter; ++it, blk += gridDim.x) {
      const int slot = it & 1;
      const int s = it & 1;
      double* in = ibuf + slot * kVals;
      __syncwarp();  // the prep warp is done reading the other input slot (block it-1)
      const int64_t nxt = blk + gridDim.x;
      if (pt == 0 && it + 1 < niter) {
        fence_proxy_async_smem();
        issue(nxt, slot ^ 1);
      }
      mbar_wait_parity(&full[slot], (parity_bits >> slot) & 1u);
      parity_bits ^= 1u << slot;
      if (it >= 2) nbar_sync(REC_EMPTY + s, kAll);  // record set s read for block it-2
      double* rec = recb + s * Cfg::kRecVals;
      constexpr int kPer = S / kPrepT;
#pragma unroll
      for (int k = 0; k < kPer; ++k) {
        const int i = pt + k * kPrepT;
        const int e = i / NN;
        const int r = i - e * NN;
        const double* uu = in + e * 5 * NN + r;
        const double rho = uu[0], m0 = uu[NN], m1 = uu[2 * NN], m2 = uu[3 * NN], et = uu[4 * NN];
        const double irho = rcp_refined(rho);
        const double v0 = m0 * irho, v1 = m1 * irho, v2 = m2 * irho;
        const double vv = fma(v2, v2, fma(v1, v1, v0 * v0));
        const double p = gm1 * fma(-0.5 * rho, vv, et);
        const double beta = 0.5 * rho * rcp_refined(p);
        const int q = e * NN + swz<N>(r % N, (r / N) % N, r / (N * N));
        rec[q] = 0.5 * rho;
        rec[S + q] = 0.5 * v0;
        rec[2 * S + q] = 0.5 * v1;
        rec[3 * S + q] = 0.5 * v2;
        rec[4 * S + q] = 0.5 * beta;
        rec[5 * S + q] = 0.5 * log_pos(rho);
        rec[6 * S + q] = 0.5 * log_pos(beta);
        rec[7 * S + q] = p;
      }
      nbar_arrive(REC_FULL + s, kAll);
    }
    for (int k = niter - 2 > 0 ? niter - 2 : 0; k < niter; ++k)
      nbar_sync(REC_EMPTY + (k & 1), kAll);
  }
}

int launch_euler_cart4_split(int64_t E, const double* Dh, double gamma, double scale,
                             const double* U, double* R, cudaStream_t s) {
  using Cfg = Split4Cfg;
  DMat<4> Dm;
  for (int i = 0; i < 16; ++i) Dm.d[i] = scale * Dh[i];
  static int per_sm = 0;
  if (per_sm == 0) {
    cudaFuncSetAttribute(euler_cart4_split_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)Cfg::kSmem);
    int b = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, euler_cart4_split_kernel, Cfg::kThreads,
                                                  Cfg::kSmem);
    per_sm = b > 0 ? b : 1;
  }
  const int64_t nblocks = (E + Cfg::kEPB - 1) / Cfg::kEPB;
  int64_t grid = (int64_t)num_sms() * per_sm;
  if (grid > nblocks) grid = nblocks;
  const double gm1 = gamma - 1.0;
  euler_cart4_split_kernel<<<(unsigned)grid, Cfg::kThreads, Cfg::kSmem, s>>>(
      E, Dm, gm1, 1.0 / (2.0 * gm1), gamma / gm1, U, R);
  return check_launch("euler_volume_cartesian(n=4, split lines)");
}

}  // namespace sfb
