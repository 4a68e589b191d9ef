// K4, warp-specialised (n = 4..6): the curvilinear modal Euler volume term
// with a prep warp and line warps working on consecutive elements.
//
//   prep warp  (element it)  : wait for the element's Uhat|Ja bulk copy, V^3 in
//                              three smem passes (slot <-> record set), node
//                              records in place -> REC_FULL
//   line warps (element it-1): contravariant pair work (each symmetric pair of
//                              a line once, metric-averaged normals) into three
//                              direction residuals; then per node
//                              r = diag + R0 + R1 + R2 (diag from the record and
//                              Ja at the node); once Ja is consumed one lane
//                              issues the bulk copy of element it+1 into the
//                              freed slot; Pi^3 in three passes; Rhat and the
//                              fixed-order sum of squares out -> REC_EMPTY
// Two slots / record sets, handed over with named barriers as in euler.cu.
// Same arithmetic as modal.cu (the reference path of the fused kernel).
#include "euler_common.cuh"

#ifndef SFB_MODALWS_K
#define SFB_MODALWS_K 3
#endif
#ifndef SFB_MODALWS_MINB
#define SFB_MODALWS_MINB 2
#endif

namespace sfb {

template <int N>
struct ModalOpsWS {
  double D[N * N];  // scale * D / 2 (metric average folded in)
  double V[N * N];
  double P[N * N];
  double Dd[N];     // scale * D[i][i]
};

template <int N>
struct ModalWSCfg {
  static constexpr int kNodes = N * N * N;
  static constexpr int kLines = N * N;
  static constexpr int kLineThreads = 3 * kLines;
  static constexpr int kLineT = (kLineThreads + 31) / 32 * 32;
  static constexpr int kPrepT = 32;
  static constexpr int kThreads = kLineT + kPrepT;
  static constexpr int kU = 5 * kNodes;
  static constexpr int kJ = 9 * kNodes;
  static constexpr int kSlot = (kU + kJ + 1) / 2 * 2;
  static constexpr int kRec = 8 * kNodes;  // hr hv0 hv1 hv2 hb hlr hlb p (also V^3 scratch)
  static constexpr int kRedPow2 = kLineT <= 128 ? 128 : 256;
  static constexpr size_t kSmem =
      (size_t)(2 * kSlot + 2 * kRec + 3 * kU + kRedPow2) * sizeof(double);
  static constexpr int kMinBlocks = (N == 6) ? SFB_MODALWS_MINB : 1;
};

template <int N>
__device__ __forceinline__ void kron_pass_ws(const double* __restrict__ A, int j,
                                             const double* __restrict__ in,
                                             double* __restrict__ out, int tid, int nthreads) {
  constexpr int NN = N * N * N;
  const int stride = j == 0 ? 1 : (j == 1 ? N : N * N);
  for (int t = tid; t < 5 * N * N; t += nthreads) {
    const int v = t / (N * N);
    const int L = t - v * N * N;
    const int u0 = L % N, u1 = L / N;
    const int base = j == 0 ? u0 * N + u1 * N * N : (j == 1 ? u0 + u1 * N * N : u0 + u1 * N);
    const double* src = in + v * NN + base;
    double x[N];
#pragma unroll
    for (int c = 0; c < N; ++c) x[c] = src[c * stride];
    double* dst = out + v * NN + base;
#pragma unroll
    for (int a = 0; a < N; ++a) {
      double acc = A[a * N] * x[0];
#pragma unroll
      for (int c = 1; c < N; ++c) acc = fma(A[a * N + c], x[c], acc);
      dst[a * stride] = acc;
    }
  }
}

template <int N>
struct WSPairs {
  static constexpr int kPairs = N * (N - 1) / 2;
  int a[kPairs], b[kPairs];
  constexpr WSPairs() : a{}, b{} {
    const int M = (N % 2 == 0) ? N : N + 1;
    int k = 0;
    for (int round = 0; round < M - 1; ++round)
      for (int i = 0; i < M / 2; ++i) {
        int x = (i == 0) ? M - 1 : (round + i) % (M - 1);
        int y = (i == 0) ? round : (round - i + (M - 1)) % (M - 1);
        if (x >= N || y >= N) continue;
        a[k] = x < y ? x : y;
        b[k] = x < y ? y : x;
        ++k;
      }
  }
};

// contravariant flux for K pairs (normals n = Ja_a + Ja_b; 1/2 folded into D)
template <int K>
__device__ __forceinline__ void flux_curv_k(const NodeRec (&A)[K], const NodeRec (&B)[K],
                                            const double (&nx)[K], const double (&ny)[K],
                                            const double (&nz)[K], double c_gamma,
                                            double (&f)[K][5]) {
  double vb0[K], vb1[K], vb2[K], nr[K], dr[K], nb[K], db[K];
#pragma unroll
  for (int k = 0; k < K; ++k) {
    vb0[k] = A[k].hv0 + B[k].hv0;
    vb1[k] = A[k].hv1 + B[k].hv1;
    vb2[k] = A[k].hv2 + B[k].hv2;
    logmean_parts(A[k].hr, B[k].hr, A[k].hlr, B[k].hlr, nr[k], dr[k]);
    logmean_parts(A[k].hb, B[k].hb, A[k].hlb, B[k].hlb, nb[k], db[k]);
  }
#pragma unroll
  for (int k = 0; k < K; ++k) {
    const double sr = __dadd_rn(A[k].hr, B[k].hr);
    const double sb = __dadd_rn(A[k].hb, B[k].hb);
    const double p1 = dr[k] * nb[k];
    const double rr = rcp_refined(p1 * sb);
    const double inv_sb = rr * p1;
    const double t = rr * sb;
    const double rho_ln = nr[k] * (t * nb[k]);
    const double ibeta = db[k] * (t * dr[k]);
    const double phat = 0.5 * sr * inv_sb;
    const double vn = fma(vb2[k], nz[k], fma(vb1[k], ny[k], vb0[k] * nx[k]));
    const double f1 = rho_ln * vn;
    f[k][0] = f1;
    f[k][1] = fma(f1, vb0[k], phat * nx[k]);
    f[k][2] = fma(f1, vb1[k], phat * ny[k]);
    f[k][3] = fma(f1, vb2[k], phat * nz[k]);
    const double dot = fma(A[k].hv2, B[k].hv2, fma(A[k].hv1, B[k].hv1, A[k].hv0 * B[k].hv0));
    const double g = fma(2.0, dot, c_gamma * ibeta);
    f[k][4] = fma(f1, g, phat * vn);
  }
}

template <int N>
__global__ void __launch_bounds__(ModalWSCfg<N>::kThreads, ModalWSCfg<N>::kMinBlocks)
    euler_modal_ws_kernel(int64_t E, const ModalOpsWS<N> ops, double gm1, double c_gamma,
                          double gam_ratio, const double* __restrict__ Uhat,
                          const double* __restrict__ Ja, double* __restrict__ Rhat,
                          double* __restrict__ sumsq) {
  using Cfg = ModalWSCfg<N>;
  constexpr int NN = Cfg::kNodes;
  constexpr int kLineT = Cfg::kLineT;
  constexpr int kAll = Cfg::kThreads;
  constexpr int kU = Cfg::kU, kJ = Cfg::kJ;
  enum { REC_FULL = 1, REC_EMPTY = 3, LINE_ONLY = 5 };
  extern __shared__ __align__(16) double smem[];
  double* slots = smem;                         // [2][Uhat | Ja]
  double* recs = smem + 2 * Cfg::kSlot;         // [2][8][NN]
  double* resd = recs + 2 * Cfg::kRec;          // [3][5][NN] direction residuals
  double* red = resd + 3 * kU;                  // [kRedPow2]
  __shared__ uint64_t full[2];
  __shared__ double sops[3 * N * N + N];
  const int tid = threadIdx.x;
  if (tid == 0) {
#pragma unroll
    for (int i = 0; i < N * N; ++i) {
      sops[i] = ops.D[i];
      sops[N * N + i] = ops.V[i];
      sops[2 * N * N + i] = ops.P[i];
    }
#pragma unroll
    for (int i = 0; i < N; ++i) sops[3 * N * N + i] = ops.Dd[i];
    mbar_init(&full[0], 1);
    mbar_init(&full[1], 1);
    fence_mbar_init();
  }
  __syncthreads();
  const double* sD = sops;
  const double* sV = sops + N * N;
  const double* sP = sops + 2 * N * N;
  const double* sDd = sops + 3 * N * N;
  const int niter = blockIdx.x < E ? (int)((E - 1 - blockIdx.x) / gridDim.x) + 1 : 0;
  auto issue = [&](int it) {  // bulk copy of this CTA's it-th element into slot it&1
    const int64_t e = (int64_t)blockIdx.x + (int64_t)it * gridDim.x;
    double* dst = slots + (it & 1) * Cfg::kSlot;
    mbar_arrive_expect_tx(&full[it & 1], (uint32_t)(kU + kJ) * 8);
    bulk_g2s(dst, Uhat + e * kU, (uint32_t)kU * 8, &full[it & 1]);
    bulk_g2s(dst + kU, Ja + e * kJ, (uint32_t)kJ * 8, &full[it & 1]);
  };

  if (tid < kLineT) {
    // =========================== line warps ==================================
    const int dir = tid / Cfg::kLines;
    const int L = tid - dir * Cfg::kLines;
    const bool active = tid < Cfg::kLineThreads;
    const int u0 = L % N, u1 = L / N;
    const int base = dir == 0 ? u0 * N + u1 * N * N : (dir == 1 ? u0 + u1 * N * N : u0 + u1 * N);
    const int stride = dir == 0 ? 1 : (dir == 1 ? N : N * N);
    if (tid == 0) {
      if (niter > 0) issue(0);
      if (niter > 1) issue(1);
    }
    for (int it = 0; it < niter; ++it) {
      const int s = it & 1;
      const int64_t e = (int64_t)blockIdx.x + (int64_t)it * gridDim.x;
      const double* rec = recs + s * Cfg::kRec;
      double* slot = slots + s * Cfg::kSlot;
      const double* jin = slot + kU;
      nbar_sync(REC_FULL + s, kAll);
      // ---- pair stage --------------------------------------------------------
      if (active) {
        double acc[N][5];
#pragma unroll
        for (int a = 0; a < N; ++a)
#pragma unroll
          for (int v = 0; v < 5; ++v) acc[a][v] = 0.0;
        constexpr WSPairs<N> po;
        constexpr int P = WSPairs<N>::kPairs;
        constexpr int K = N >= 6 ? SFB_MODALWS_K : 2;
        const double* jd = jin + (dir * 3) * NN;
        auto load = [&](int a) {
          NodeRec q;
          const int k = base + a * stride;
          q.hr = rec[k];
          q.hv0 = rec[NN + k];
          q.hv1 = rec[2 * NN + k];
          q.hv2 = rec[3 * NN + k];
          q.hb = rec[4 * NN + k];
          q.hlr = rec[5 * NN + k];
          q.hlb = rec[6 * NN + k];
          q.q = 0.0;
          return q;
        };
#pragma unroll
        for (int k0 = 0; k0 < P; k0 += K) {
          NodeRec A[K], B[K];
          double nx[K], ny[K], nz[K];
#pragma unroll
          for (int k = 0; k < K; ++k) {
            const int kk = (k0 + k < P) ? k0 + k : P - 1;
            const int a = po.a[kk], b = po.b[kk];
            A[k] = load(a);
            B[k] = load(b);
            const int ka = base + a * stride, kb = base + b * stride;
            nx[k] = jd[ka] + jd[kb];
            ny[k] = jd[NN + ka] + jd[NN + kb];
            nz[k] = jd[2 * NN + ka] + jd[2 * NN + kb];
          }
          double f[K][5];
          flux_curv_k<K>(A, B, nx, ny, nz, c_gamma, f);
#pragma unroll
          for (int k = 0; k < K; ++k) {
            if (k0 + k >= P) break;
            const int a = po.a[k0 + k], b = po.b[k0 + k];
            const double dab = sD[a * N + b], dba = sD[b * N + a];
#pragma unroll
            for (int v = 0; v < 5; ++v) {
              acc[a][v] = fma(dab, f[k][v], acc[a][v]);
              acc[b][v] = fma(dba, f[k][v], acc[b][v]);
            }
          }
        }
        double* rd = resd + dir * kU + base;
#pragma unroll
        for (int a = 0; a < N; ++a)
#pragma unroll
          for (int v = 0; v < 5; ++v) rd[v * NN + a * stride] = acc[a][v];
      }
      nbar_sync(LINE_ONLY, kLineT);
      // ---- diag + direction sum (into R0); last use of Ja and the records ----
      for (int r = tid; r < NN; r += kLineT) {
        const int c0 = r % N, c1 = (r / N) % N, c2 = r / (N * N);
        const double d0 = sDd[c0], d1 = sDd[c1], d2 = sDd[c2];
        double nd[3];
#pragma unroll
        for (int m = 0; m < 3; ++m)
          nd[m] = fma(d2, jin[(6 + m) * NN + r], fma(d1, jin[(3 + m) * NN + r], d0 * jin[m * NN + r]));
        const double hr = rec[r], h0 = rec[NN + r], h1 = rec[2 * NN + r], h2 = rec[3 * NN + r];
        const double p = rec[7 * NN + r];
        const double rho = 2.0 * hr;
        const double vn = 2.0 * fma(h2, nd[2], fma(h1, nd[1], h0 * nd[0]));  // v . n_diag
        const double q = fma(h2, h2, fma(h1, h1, h0 * h0));                  // |v|^2 / 4
        const double rvn = rho * vn;
        const double diag[5] = {rvn, fma(2.0 * rvn, h0, p * nd[0]), fma(2.0 * rvn, h1, p * nd[1]),
                                fma(2.0 * rvn, h2, p * nd[2]),
                                fma(gam_ratio, p, 4.0 * hr * q) * vn};
#pragma unroll
        for (int v = 0; v < 5; ++v) {
          const int i = v * NN + r;
          resd[i] = ((diag[v] + resd[i]) + resd[kU + i]) + resd[2 * kU + i];
        }
      }
      nbar_sync(LINE_ONLY, kLineT);
      nbar_arrive(REC_EMPTY + s, kAll);  // records of set s consumed
      if (tid == 0 && it + 2 < niter) {  // slot s free: prefetch this CTA's element it+2
        fence_proxy_async_smem();
        issue(it + 2);
      }
      // ---- Rhat = Pi^3 r (R0 -> R1 -> R0 -> R1), store, sum of squares --------
      kron_pass_ws<N>(sP, 0, resd, resd + kU, tid, kLineT);
      nbar_sync(LINE_ONLY, kLineT);
      kron_pass_ws<N>(sP, 1, resd + kU, resd, tid, kLineT);
      nbar_sync(LINE_ONLY, kLineT);
      kron_pass_ws<N>(sP, 2, resd, resd + kU, tid, kLineT);
      nbar_sync(LINE_ONLY, kLineT);
      const double* out = resd + kU;
      double* Rg = Rhat + e * kU;
      double ss = 0.0;
      for (int i = tid; i < kU; i += kLineT) {
        const double x = out[i];
        __stcs(Rg + i, x);
        ss = fma(x, x, ss);
      }
      if (sumsq) {  // fixed-shape tree: deterministic per element
        constexpr int RP = Cfg::kRedPow2;
        red[tid] = ss;
        for (int i = kLineT + tid; i < RP; i += kLineT) red[i] = 0.0;
        nbar_sync(LINE_ONLY, kLineT);
        for (int w = RP / 2; w >= 1; w /= 2) {
          for (int i = tid; i < w; i += kLineT) red[i] = red[i] + red[i + w];
          nbar_sync(LINE_ONLY, kLineT);
        }
        if (tid == 0) sumsq[e] = red[0];
      }
      nbar_sync(LINE_ONLY, kLineT);  // residual buffers free for the next element
    }
  } else {
    // =========================== prep warp ===================================
    const int pt = tid - kLineT;
    uint32_t parity_bits = 0;
    for (int it = 0; it < niter; ++it) {
      const int s = it & 1;
      double* slot = slots + s * Cfg::kSlot;
      double* rec = recs + s * Cfg::kRec;
      if (it >= 2) nbar_sync(REC_EMPTY + s, kAll);  // record set s read for element it-2
      mbar_wait_parity(&full[s], (parity_bits >> s) & 1u);
      parity_bits ^= 1u << s;
      // V^3: slot -> rec -> slot -> rec (u in rec planes 0..4)
      kron_pass_ws<N>(sV, 0, slot, rec, pt, 32);
      __syncwarp();
      kron_pass_ws<N>(sV, 1, rec, slot, pt, 32);
      __syncwarp();
      kron_pass_ws<N>(sV, 2, slot, rec, pt, 32);
      __syncwarp();
      // node records in place (each lane reads its nodes' u, then overwrites them)
      for (int r = pt; r < NN; r += 32) {
        const double rho = rec[r], m0 = rec[NN + r], m1 = rec[2 * NN + r], m2 = rec[3 * NN + r],
                     et = rec[4 * NN + r];
        const double hirho = 0.5 * rcp_refined(rho);
        const double mm = fma(m2, m2, fma(m1, m1, m0 * m0));
        const double X = fma(rho, et, -0.5 * mm);
        const double iX = rcp_refined(X);
        const double p = (2.0 * gm1) * X * hirho;
        const double hbeta = (rho * rho) * ((0.5 * c_gamma) * iX);
        rec[r] = 0.5 * rho;
        rec[NN + r] = m0 * hirho;
        rec[2 * NN + r] = m1 * hirho;
        rec[3 * NN + r] = m2 * hirho;
        rec[4 * NN + r] = hbeta;
        rec[5 * NN + r] = log_half(rho);
        rec[6 * NN + r] = log_half(2.0 * hbeta);
        rec[7 * NN + r] = p;
      }
      __syncwarp();
      nbar_arrive(REC_FULL + s, kAll);
    }
    for (int k = niter - 2 > 0 ? niter - 2 : 0; k < niter; ++k) nbar_sync(REC_EMPTY + (k & 1), kAll);
  }
}

template <int N>
int launch_modal_ws(int64_t E, const double* V, const double* Pi, const double* D, double gamma,
                    double scale, const double* Uhat, const double* Ja, double* Rhat,
                    double* sumsq, cudaStream_t s) {
  using Cfg = ModalWSCfg<N>;
  ModalOpsWS<N> ops;
  for (int i = 0; i < N * N; ++i) {
    ops.D[i] = 0.5 * scale * D[i];
    ops.V[i] = V[i];
    ops.P[i] = Pi[i];
  }
  for (int i = 0; i < N; ++i) ops.Dd[i] = scale * D[i * N + i];
  static int per_sm = 0;
  if (per_sm == 0) {
    cudaFuncSetAttribute(euler_modal_ws_kernel<N>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)Cfg::kSmem);
    int b = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, euler_modal_ws_kernel<N>, Cfg::kThreads,
                                                  Cfg::kSmem);
    per_sm = b > 0 ? b : 1;
  }
  int64_t grid = (int64_t)num_sms() * per_sm;
  if (grid > E) grid = E;
  const double gm1 = gamma - 1.0;
  euler_modal_ws_kernel<N><<<(unsigned)grid, Cfg::kThreads, Cfg::kSmem, s>>>(
      E, ops, gm1, 1.0 / (2.0 * gm1), gamma / gm1, Uhat, Ja, Rhat, sumsq);
  return check_launch("euler_volume_curvilinear_modal(warp-specialised)");
}

template int launch_modal_ws<4>(int64_t, const double*, const double*, const double*, double,
                                double, const double*, const double*, double*, double*,
                                cudaStream_t);
template int launch_modal_ws<6>(int64_t, const double*, const double*, const double*, double,
                                double, const double*, const double*, double*, double*,
                                cudaStream_t);

}  // namespace sfb
