// K3: fused flux-differencing volume term for the 3-D compressible Euler
// equations on affine Cartesian elements (BASELINE configs 3 and 4).
//
//   R[e,:,r] = scale * sum_j sum_l D[r_j,l] F#_j(U[e,:,r], U[e,:,r(j->l)])
//
// This is the reference's flux-differencing volume term (burgers.py:117-131:
// Hadamard product of the Kronecker factor with the two-point flux matrix,
// row-summed, summed over directions) for a 5-variable state with the
// Chandrashekar flux.  The reference evaluates it as pattern -> operand
// gather -> hadamard_evaluate -> hadamard_row_sum (kernel.py:195-266); here the
// whole chain is one persistent kernel and only U and R touch HBM.
//
// Per CTA, loop over blocks of EPB elements (grid = resident CTAs):
//   prefetch  one elected thread streams the NEXT block (EPB*5*N^3 doubles,
//             contiguous) into the other half of a double buffer with a 1-D
//             bulk copy (cp.async.bulk -> UBLKCP) completing on an mbarrier,
//             so HBM traffic overlaps the FP64 work of the current block;
//   stage 1   one thread per node: primitives, per-node logarithms, the node
//             record of euler_flux.cuh, and the diagonal term
//             sum_j D[r_j,r_j] f_j(u_r) (the residual's initial value);
//   stage 2   one thread per (element, direction, line), warp-uniform in the
//             direction (template DIR): each symmetric pair a<b of the line is
//             evaluated ONCE and scattered to both rows with D[a,b], D[b,a]
//             (Theorem 1's n(n-1)/2 per line, halved by symmetry);
//   stage 3   direction-ordered accumulation into the shared residual
//             (barrier-separated phases: deterministic, no atomics);
//   stage 4   coalesced 16-byte streaming stores of the residual.
// Node records and the residual use a plane-rotation swizzle
//   pos(r0,r1,r2) = r2 N^2 + ((r0+r2) mod N) + N ((r1+r2) mod N)
// which makes the stride-1, stride-N and stride-N^2 line accesses of all three
// directions bank-conflict free for N = 4.
#include "euler_common.cuh"

#ifndef SFB_PAIR_BATCH_N4
#define SFB_PAIR_BATCH_N4 2
#endif
#ifndef SFB_MINBLOCKS_N4
#define SFB_MINBLOCKS_N4 4
#endif
#ifndef SFB_REC_SETS_N4
#define SFB_REC_SETS_N4 3
#endif
#ifndef SFB_EXP_NO_LINE
#define SFB_EXP_NO_LINE 0
#endif
#ifndef SFB_EXP_NO_PREP
#define SFB_EXP_NO_PREP 0
#endif
#ifndef SFB_WARP_N4
#define SFB_WARP_N4 1  // warp-autonomous kernel (euler_warp.cu)
#endif
// per-n tuning of the CTA kernel (config-4 sweep; defaults measured best)
#ifndef SFB_EPB_N6
#define SFB_EPB_N6 1
#endif
#ifndef SFB_MB_N5
#define SFB_MB_N5 2
#endif
#ifndef SFB_MB_N6
#define SFB_MB_N6 2
#endif
#ifndef SFB_MB_N8
#define SFB_MB_N8 1
#endif
#ifndef SFB_K_N5
#define SFB_K_N5 1
#endif
#ifndef SFB_K_N6
#define SFB_K_N6 2
#endif
#ifndef SFB_K_N7
#define SFB_K_N7 1
#endif
#ifndef SFB_K_N8
#define SFB_K_N8 2
#endif
#ifndef SFB_LEAN_N7
#define SFB_LEAN_N7 1  // register-lean line loop: 2 CTAs/SM at n = 7 (1.47 -> 1.34 ms)
#endif
#ifndef SFB_LEAN_N5
#define SFB_LEAN_N5 1  // 0.809 -> 0.788 ms
#endif
#ifndef SFB_LEAN_N8
#define SFB_LEAN_N8 1  // 1.317 -> 1.267 ms (still 1 CTA/SM: 168 KB of shared memory)
#endif
#ifndef SFB_REC_SETS_N8
#define SFB_REC_SETS_N8 2
#endif
#ifndef SFB_LEAN_N6
#define SFB_LEAN_N6 1  // with EPB 1 and 2 CTAs/SM: 1.115 -> 1.013 ms
#endif
#ifndef SFB_GENERIC_TABLOG
#define SFB_GENERIC_TABLOG 0  // table log: +30% at n=6 (the single prep warp is latency-bound)
#endif
#ifndef SFB_MINBLOCKS_N7
#define SFB_MINBLOCKS_N7 2  // with the lean line loop (without it 2 spilled: 1.86 vs 1.54 ms)
#endif
#ifndef SFB_WARP_SMALL
#define SFB_WARP_SMALL 1  // 1: n = 2, 3 on the warp-autonomous kernel; 2: n = 5 too
#endif
#ifndef SFB_RECS_IN_REGS
#define SFB_RECS_IN_REGS 1
#endif
#ifndef SFB_PREP_WARPS_N4
#define SFB_PREP_WARPS_N4 1
#endif

// n = 5..8 on the barrier-synchronised CTA kernel (euler_sync.cu) instead of
// the warp-specialised one below; config-4 points (ms, sync vs this file's):
// n = 5 1.00 vs 0.79, n = 6 0.95 vs 1.01, n = 7 1.46 (3 CTAs at 136 regs) /
// 1.98 (2 CTAs) vs 1.34, n = 8 1.33 vs 1.27: only n = 6 takes it
// n = 2 on the register-only two-threads-per-element kernel (euler_n2.cu)
#ifndef SFB_N2_REGS
#define SFB_N2_REGS 1
#endif
// n = 3 on the register/shuffle kernel, nine threads per element (euler_n3.cu)
#ifndef SFB_N3_REGS
#define SFB_N3_REGS 1
#endif
// n = 5..8 on the lane-per-node kernel (euler_node.cu); config-4 points (ms,
// dynamic claims; node kernel vs the default of each n): n = 5 1.00 vs 0.78,
// n = 6 1.17 vs 0.95, n = 7 1.27 vs 1.31, n = 8 1.52 vs 1.26 - only n = 7
// takes it
#ifndef SFB_NODE_N5
#define SFB_NODE_N5 0
#endif
#ifndef SFB_NODE_N6
#define SFB_NODE_N6 0
#endif
#ifndef SFB_NODE_N7
#define SFB_NODE_N7 1
#endif
#ifndef SFB_NODE_N8
#define SFB_NODE_N8 0
#endif
#ifndef SFB_SYNC_N5
#define SFB_SYNC_N5 0
#endif
#ifndef SFB_SYNC_N6
#define SFB_SYNC_N6 1
#endif
#ifndef SFB_SYNC_N7
#define SFB_SYNC_N7 0
#endif
#ifndef SFB_SYNC_N8
#define SFB_SYNC_N8 0
#endif

namespace sfb {

template <int N>
struct EulerCartCfg {
  static constexpr int kNodes = N * N * N;
  static constexpr int kLines = N * N;
  // elements per block; line threads = 3 EPB N^2 (padded to warps), chosen so
  // the padding is small and the line warps are direction-uniform for N = 4
  // (EPB*5*N^3*8 bytes must be a multiple of 16 for the 1-D bulk copy)
  static constexpr int kEPB = (N == 2) ? 8 : (N == 3) ? 8 : (N >= 7) ? 1 : (N == 6 ? SFB_EPB_N6 : 2);
  static constexpr int kLineThreads = 3 * kLines * kEPB;
  static constexpr int kLineWarps = (kLineThreads + 31) / 32;
  // prep warps balance node preprocessing + stores against the line work
  static constexpr int kPrepWarps = (N <= 3) ? 3 : (N == 4 ? SFB_PREP_WARPS_N4 : 1);
  static constexpr int kThreads = 32 * (kLineWarps + kPrepWarps);
  static constexpr int kMinBlocks =
      (N == 4) ? SFB_MINBLOCKS_N4
               : (N == 7 ? SFB_MINBLOCKS_N7
                         : (N == 6 ? SFB_MB_N6 : (N == 8 ? SFB_MB_N8 : (N == 5 ? SFB_MB_N5 : 2))));
  static constexpr int kVals = kEPB * 5 * kNodes;  // doubles per block of states
  static constexpr int kPlanes = 8;                // 7 record planes + pressure
  static constexpr int kRecVals = kPlanes * kEPB * kNodes;
  // smem (doubles): 2 input buffers + 2 record sets + 3 direction residuals + diag(D)
  static constexpr int kSlot = (kVals + 3) / 2 * 2;  // input slot: +1 double of alignment shift, kept even (16-B aligned slots)
  static constexpr int kRecSets = (N == 4) ? SFB_REC_SETS_N4 : (N == 8 ? SFB_REC_SETS_N8 : 2);  // record-set ring depth
  static constexpr size_t kSmem = (size_t)(2 * kSlot + kRecSets * kRecVals + 3 * kVals + 8) * sizeof(double);
};

// pairs evaluated side by side per line thread (ILP knob)
template <int N>
constexpr int kPairBatch = (N == 4)   ? SFB_PAIR_BATCH_N4
                           : (N == 5) ? SFB_K_N5
                           : (N == 6) ? SFB_K_N6
                           : (N == 7) ? SFB_K_N7
                           : (N == 8) ? SFB_K_N8
                                      : 2;

template <int N>
struct LineOut {
  int vplane[3];  // record-plane offsets of the rotated velocity components
  int pos[N];
  double acc[N][5];
};

template <int N>
__device__ __forceinline__ void line_work(const double* __restrict__ rec, int el, int dir, int L,
                                          const DMat<N>& Dm, double gm1, LineOut<N>& o) {
  using Cfg = EulerCartCfg<N>;
  constexpr int NN = Cfg::kNodes;
  constexpr int S = Cfg::kEPB * NN;  // record-plane stride
  const int u = L % N, w = L / N;
#pragma unroll
  for (int a = 0; a < N; ++a) {
    const int r0 = dir == 0 ? a : u;
    const int r1 = dir == 1 ? a : (dir == 0 ? u : w);
    const int r2 = dir == 2 ? a : w;
    o.pos[a] = swz<N>(r0, r1, r2);
  }
#pragma unroll
  for (int m = 0; m < 3; ++m) o.vplane[m] = (1 + (dir + m) % 3) * S;
  const double* re = rec + el * NN;
  auto load = [&](int a) {
    NodeRec q;
    const double* p = re + o.pos[a];
    q.hr = p[0];
    q.hv0 = p[o.vplane[0]];  // velocity rotated to (normal, t1, t2) of this direction
    q.hv1 = p[o.vplane[1]];
    q.hv2 = p[o.vplane[2]];
    q.hb = p[4 * S];
    q.hlr = p[5 * S];
    q.hlb = p[6 * S];  // unused: the energy flux uses 2 (v_a/2).(v_b/2)
    return q;
  };
#pragma unroll
  for (int a = 0; a < N; ++a)
#pragma unroll
    for (int v = 0; v < 5; ++v) o.acc[a][v] = 0.0;
  if constexpr ((N == 7 && SFB_LEAN_N7) || (N == 6 && SFB_LEAN_N6) || (N == 8 && SFB_LEAN_N8) ||
                (N == 5 && SFB_LEAN_N5)) {
    // register-lean loop: node a once per outer step, nodes b > a re-read with
    // volatile shared loads (no CSE keeps all n records live), so the kernel
    // fits 168 registers and 2 CTAs per SM
    const uint32_t rs = smem_u32(re);
    auto vl = [&](int a, int off) {
      double x;
      asm volatile("ld.shared.f64 %0, [%1];" : "=d"(x) : "r"(rs + 8u * (uint32_t)(o.pos[a] + off)));
      return x;
    };
    auto vload = [&](int a) {
      NodeRec q;
      q.hr = vl(a, 0);
      q.hv0 = vl(a, o.vplane[0]);
      q.hv1 = vl(a, o.vplane[1]);
      q.hv2 = vl(a, o.vplane[2]);
      q.hb = vl(a, 4 * S);
      q.hlr = vl(a, 5 * S);
      q.hlb = vl(a, 6 * S);
      return q;
    };
#pragma unroll
    for (int a = 0; a < N - 1; ++a) {
      const NodeRec qa = vload(a);
#pragma unroll
      for (int b = a + 1; b < N; ++b) {
        const NodeRec qb = vload(b);
        const NodeRec* A[1] = {&qa};
        const NodeRec* B[1] = {&qb};
        double f[1][5];
        chandrashekar_cart_v2<1>(A, B, gm1, f);
        const double dab = Dm.d[a * N + b], dba = Dm.d[b * N + a];
#pragma unroll
        for (int v = 0; v < 5; ++v) {
          o.acc[a][v] = fma(dab, f[0][v], o.acc[a][v]);
          o.acc[b][v] = fma(dba, f[0][v], o.acc[b][v]);
        }
      }
    }
    return;
  }
  constexpr PairOrder<N> po;
  constexpr int P = PairOrder<N>::kPairs;
  constexpr int K = kPairBatch<N>;
#if SFB_RECS_IN_REGS
  NodeRec nrec[N];
#pragma unroll
  for (int a = 0; a < N; ++a) nrec[a] = load(a);
#endif
#pragma unroll
  for (int k0 = 0; k0 < P; k0 += K) {
    const NodeRec* A[K];
    const NodeRec* B[K];
#if !SFB_RECS_IN_REGS
    NodeRec ra[K], rb[K];  // records loaded per pair batch (fewer live registers)
#endif
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const int kk = (k0 + k < P) ? k0 + k : P - 1;
#if SFB_RECS_IN_REGS
      A[k] = &nrec[po.a[kk]];
      B[k] = &nrec[po.b[kk]];
#else
      ra[k] = load(po.a[kk]);
      rb[k] = load(po.b[kk]);
      A[k] = &ra[k];
      B[k] = &rb[k];
#endif
    }
    double f[K][5];
    chandrashekar_cart_v2<K>(A, B, gm1, f);
#pragma unroll
    for (int k = 0; k < K; ++k) {
      if (k0 + k >= P) break;
      const int a = po.a[k0 + k], b = po.b[k0 + k];
      const double dab = Dm.d[a * N + b], dba = Dm.d[b * N + a];
#pragma unroll
      for (int v = 0; v < 5; ++v) {
        o.acc[a][v] = fma(dab, f[k][v], o.acc[a][v]);
        o.acc[b][v] = fma(dba, f[k][v], o.acc[b][v]);
      }
    }
  }
}

// Warp-specialised persistent kernel.  Line warps (the FP64-heavy pair work
// and the residual stores) and prep warps (bulk prefetch, node records and the
// diagonal term) run concurrently on consecutive element blocks, handing the
// double-buffered record sets over through named barriers:
//   REC_FULL[s]  prep -> line : records + diagonal of the block in set s ready
//   REC_EMPTY[s] line -> prep : record set s consumed
template <int N>
__global__ void __launch_bounds__(EulerCartCfg<N>::kThreads, EulerCartCfg<N>::kMinBlocks)
    euler_cartesian_kernel(int64_t E, const DMat<N> Dm, double gm1, double c_gamma,
                           double gam_ratio, const double* __restrict__ U,
                           double* __restrict__ R) {
  using Cfg = EulerCartCfg<N>;
  constexpr int NN = Cfg::kNodes;
  constexpr int EPB = Cfg::kEPB;
  constexpr int kVals = Cfg::kVals;
  constexpr int S = EPB * NN;
  constexpr int kLineT = 32 * Cfg::kLineWarps;
  constexpr int kPrepT = 32 * Cfg::kPrepWarps;
  constexpr int kAll = kLineT + kPrepT;
  constexpr int RS = Cfg::kRecSets;
  enum { REC_FULL = 1, REC_EMPTY = 4, LINE_ONLY = 7, PREP_ONLY = 8 };
  extern __shared__ __align__(16) double smem[];
  double* ibuf = smem;                      // [2][EPB][5][NN] bulk-copy target
  constexpr int kSlot = Cfg::kSlot;
  double* recb = smem + 2 * kSlot;          // [2][8][EPB*NN] swizzled records + p
  double* resb = recb + RS * Cfg::kRecVals;  // [3][EPB][5][NN] swizzled direction residuals
  double* ddiag = resb + 3 * kVals;         // [N] scale*D[i][i]
  __shared__ uint64_t full[2];

  const int tid = threadIdx.x;
  const int64_t nblocks = (E + EPB - 1) / EPB;
  if (tid == 0) {
#pragma unroll
    for (int i = 0; i < N; ++i) ddiag[i] = Dm.d[i * N + i];  // static indices: no local copy
    mbar_init(&full[0], 1);
    mbar_init(&full[1], 1);
    fence_mbar_init();
  }
  __syncthreads();
  const int niter = blockIdx.x < nblocks ? (int)((nblocks - 1 - blockIdx.x) / gridDim.x) + 1 : 0;

  if (tid < kLineT) {
    // =========================== line warps ==================================
    const int dir = tid / (EPB * Cfg::kLines);
    const int rem = tid - dir * EPB * Cfg::kLines;
    const int el = rem / Cfg::kLines;
    const int L = rem - el * Cfg::kLines;
    const bool active = tid < Cfg::kLineThreads;
    for (int it = 0; it < niter; ++it) {
      const int s = it % RS;
      const double* rec = recb + s * Cfg::kRecVals;
      nbar_sync(REC_FULL + s, kAll);
      LineOut<N> o;
#if SFB_EXP_NO_LINE
      if (active) { for (int a = 0; a < N; ++a) { o.pos[a] = a; for (int v = 0; v < 5; ++v) o.acc[a][v] = rec[a]; } }
#else
      if (active) line_work<N>(rec, el, dir, L, Dm, gm1, o);
#endif
      if (active) {
        double* rs = resb + dir * kVals + el * 5 * NN;
        // momentum components come back in the rotated frame: un-rotate by address
        const int mp0 = (1 + dir % 3) * NN, mp1 = (1 + (dir + 1) % 3) * NN,
                  mp2 = (1 + (dir + 2) % 3) * NN;
#pragma unroll
        for (int a = 0; a < N; ++a) {
          rs[o.pos[a]] = o.acc[a][0];
          rs[o.pos[a] + mp0] = o.acc[a][1];
          rs[o.pos[a] + mp1] = o.acc[a][2];
          rs[o.pos[a] + mp2] = o.acc[a][3];
          rs[o.pos[a] + 4 * NN] = o.acc[a][4];
        }
      }
      nbar_sync(LINE_ONLY, kLineT);  // all three direction residuals written
      // residual = diag + (R_0 + R_1) + R_2 per node; the diagonal term
      // sum_j D[r_j,r_j] f_j(u_r) is rebuilt here from the node record
      // (rho = 2hr, v = 2hv, p, E + p = p gamma/(gamma-1) + 4 hr q)
      {
        const int64_t blk = (int64_t)blockIdx.x + (int64_t)it * gridDim.x;
        const int64_t e0 = blk * EPB;
        const int nel = (E - e0) < EPB ? (int)(E - e0) : EPB;
        double* Rb = R + e0 * 5 * NN;
        const int nn = nel * NN;
        for (int i = tid; i < nn; i += kLineT) {
          const int e = i / NN;
          const int r = i - e * NN;
          const int c0 = r % N, c1 = (r / N) % N, c2 = r / (N * N);
          const int qn = swz<N>(c0, c1, c2);
          const double* rc = rec + e * NN + qn;
          const double hr = rc[0], h0 = rc[S], h1 = rc[2 * S], h2 = rc[3 * S];
          const double p = rc[7 * S];
          const double q = fma(h2, h2, fma(h1, h1, h0 * h0));  // |v|^2 / 4
          const double d0 = ddiag[c0], d1 = ddiag[c1], d2 = ddiag[c2];
          const double w = 2.0 * fma(d2, h2, fma(d1, h1, d0 * h0));  // sum_j d_j v_j
          const double rho = 2.0 * hr;
          const double rw = rho * w;
          const double ep = fma(gam_ratio, p, 4.0 * hr * q);  // E + p
          const double diag[5] = {rw, fma(2.0 * rw, h0, p * d0), fma(2.0 * rw, h1, p * d1),
                                  fma(2.0 * rw, h2, p * d2), ep * w};
          const double* r0 = resb + e * 5 * NN + qn;
          const double* r1 = r0 + kVals;
          const double* r2 = r1 + kVals;
#pragma unroll
          for (int v = 0; v < 5; ++v)
            __stcs(Rb + e * 5 * NN + v * NN + r,
                   ((diag[v] + r0[v * NN]) + r1[v * NN]) + r2[v * NN]);
        }
      }
      nbar_arrive(REC_EMPTY + s, kAll);  // records (incl. p) consumed
      nbar_sync(LINE_ONLY, kLineT);  // residual buffers free again
    }
  } else {
    // =========================== prep warps ==================================
    const int pt = tid - kLineT;
    // A block's states start at double offset blk*EPB*5*NN, which is odd for
    // odd 5*N^3*EPB: the bulk copy then starts one double early (16-byte
    // alignment) and the block is read at `shift` = 1.  Only a final block whose
    // aligned copy would run past the end of U falls back to plain loads.
    const int64_t total_vals = E * 5 * NN;
    auto block_shift = [&](int64_t blk) { return (int)((blk * EPB * 5 * NN) & 1); };
    auto block_vals = [&](int64_t blk) {
      const int64_t e0 = blk * EPB;
      const int nel = (E - e0) < EPB ? (int)(E - e0) : EPB;
      return nel * 5 * NN;
    };
    auto copy_doubles = [&](int64_t blk) { return (block_shift(blk) + block_vals(blk) + 1) & ~1; };
    auto bulk_ok = [&](int64_t blk) {
      return blk * EPB * 5 * NN - block_shift(blk) + copy_doubles(blk) <= total_vals;
    };
    auto issue = [&](int64_t blk, int slot) {
      const uint32_t bytes = (uint32_t)copy_doubles(blk) * 8;
      mbar_arrive_expect_tx(&full[slot], bytes);
      bulk_g2s(ibuf + slot * kSlot, U + blk * EPB * 5 * NN - block_shift(blk), bytes,
               &full[slot]);
    };
    int64_t blk = blockIdx.x;
    if (pt == 0 && niter > 0 && bulk_ok(blk)) issue(blk, 0);
    uint32_t parity_bits = 0;  // bit k = phase of input slot k (no local-memory array)
    for (int it = 0; it < niter; ++it, blk += gridDim.x) {
      const int slot = it & 1;
      const int s = it % RS;
      const int64_t e0 = blk * EPB;
      const int nel = (E - e0) < EPB ? (int)(E - e0) : EPB;
      double* in = ibuf + slot * kSlot;
      // all prep threads are done reading the other input slot (block it-1)
      nbar_sync(PREP_ONLY, kPrepT);
      const int64_t nxt = blk + gridDim.x;
      if (pt == 0 && it + 1 < niter && bulk_ok(nxt)) {
        fence_proxy_async_smem();
        issue(nxt, slot ^ 1);
      }
      if (bulk_ok(blk)) {
        mbar_wait_parity(&full[slot], (parity_bits >> slot) & 1u);
        parity_bits ^= 1u << slot;
        in += block_shift(blk);
      } else {  // final block that cannot be copied aligned: plain loads
        for (int i = pt; i < nel * 5 * NN; i += kPrepT) in[i] = __ldcs(U + e0 * 5 * NN + i);
        nbar_sync(PREP_ONLY, kPrepT);
      }
      if (it >= RS) nbar_sync(REC_EMPTY + s, kAll);  // record set s read for block it-RS
      double* rec = recb + s * Cfg::kRecVals;
      constexpr int kPer = (S + kPrepT - 1) / kPrepT;
#pragma unroll
      for (int k = 0; k < (SFB_EXP_NO_PREP ? 0 : kPer); ++k) {
        const int i = pt + k * kPrepT;
        if (kPer * kPrepT != S && i >= S) break;
        const int el = i / NN;
        const int r = i - el * NN;
        const double* u = in + el * 5 * NN + r;
        const double rho = u[0], m0 = u[NN], m1 = u[2 * NN], m2 = u[3 * NN], et = u[4 * NN];
        // two independent reciprocals (1/rho and 1/X, X = rho E - |m|^2/2 = rho p/(gamma-1))
        // instead of the chain 1/rho -> p -> 1/p; halvings folded into the factors
        const double hirho = 0.5 * rcp_refined(rho);
        const double mm = fma(m2, m2, fma(m1, m1, m0 * m0));
        const double X = fma(rho, et, -0.5 * mm);
        const double iX = rcp_refined(X);
        const double p = (2.0 * gm1) * X * hirho;
        const double hbeta = (rho * rho) * (0.5 * iX);  // (gamma-1) beta = rho^2 / (2X)
        const int c0 = r % N, c1 = (r / N) % N, c2 = r / (N * N);
        const int q = el * NN + swz<N>(c0, c1, c2);
        rec[q] = 0.5 * rho;
        rec[S + q] = m0 * hirho;
        rec[2 * S + q] = m1 * hirho;
        rec[3 * S + q] = m2 * hirho;
        rec[4 * S + q] = hbeta;
        rec[5 * S + q] = SFB_GENERIC_TABLOG ? log_half_tab(rho) : log_half(rho);
        rec[6 * S + q] = SFB_GENERIC_TABLOG ? log_half_tab(hbeta) : log_half(hbeta);
        rec[7 * S + q] = p;
      }
      nbar_arrive(REC_FULL + s, kAll);
    }
    // match the REC_EMPTY arrivals of the last (up to) RS blocks
    for (int k = niter - RS > 0 ? niter - RS : 0; k < niter; ++k) nbar_sync(REC_EMPTY + k % RS, kAll);
  }
}

template <int N>
static int launch_euler_cartesian(int64_t E, const double* Dh, double gamma, double scale,
                                  const double* U, double* R, cudaStream_t s) {
  using Cfg = EulerCartCfg<N>;
  DMat<N> Dm;
  for (int i = 0; i < N * N; ++i) Dm.d[i] = scale * Dh[i];
  static DeviceCache cache;
  const int per_sm = resident_ctas(euler_cartesian_kernel<N>, Cfg::kThreads, Cfg::kSmem, cache);
  const int64_t nblocks = (E + Cfg::kEPB - 1) / Cfg::kEPB;
  int64_t grid = (int64_t)num_sms() * per_sm;
  if (grid > nblocks) grid = nblocks;
  const double gm1 = gamma - 1.0;
  const double c_gamma = 1.0 / (2.0 * gm1);
  const double gam_ratio = gamma / gm1;  // (E + p) = p gamma/(gamma-1) + rho|v|^2/2
  euler_cartesian_kernel<N><<<(unsigned)grid, Cfg::kThreads, Cfg::kSmem, s>>>(
      E, Dm, gm1, c_gamma, gam_ratio, U, R);
  return check_launch("euler_volume_cartesian");
}


template <int N>
int launch_euler_cart_warp(int64_t E, const double* Dh, double gamma, double scale,
                           const double* U, double* R, cudaStream_t s);
template <int N>
int launch_euler_cart_sync(int64_t E, const double* Dh, double gamma, double scale,
                           const double* U, double* R, void* ws, cudaStream_t s);

int launch_euler_cart_n2(int64_t E, const double* Dh, double gamma, double scale,
                         const double* U, double* R, cudaStream_t s);
int launch_euler_cart_n3(int64_t E, const double* Dh, double gamma, double scale,
                         const double* U, double* R, cudaStream_t s);
template <int N>
int launch_euler_cart_node(int64_t E, const double* Dh, double gamma, double scale,
                           const double* U, double* R, void* ws, cudaStream_t s);

// ws: optional 8-byte device claim counter (dynamic element claims of the
// persistent CTA kernels; NULL = static split, the same results bitwise)
int euler_cartesian_dispatch(int64_t E, int64_t n, const double* D_host, double gamma,
                             double scale, const double* U, double* R, void* ws,
                             cudaStream_t s) {
  switch (n) {
    case 2:
      if (SFB_N2_REGS) return launch_euler_cart_n2(E, D_host, gamma, scale, U, R, s);
      return SFB_WARP_SMALL ? launch_euler_cart_warp<2>(E, D_host, gamma, scale, U, R, s)
                            : launch_euler_cartesian<2>(E, D_host, gamma, scale, U, R, s);
    case 3:  // own-line warp kernel 0.552 vs CTA kernel 0.663 ms (config 4)
      if (SFB_N3_REGS) return launch_euler_cart_n3(E, D_host, gamma, scale, U, R, s);
      return SFB_WARP_SMALL ? launch_euler_cart_warp<3>(E, D_host, gamma, scale, U, R, s)
                            : launch_euler_cartesian<3>(E, D_host, gamma, scale, U, R, s);
    case 4:
      if (SFB_WARP_N4) return launch_euler_cart_warp<4>(E, D_host, gamma, scale, U, R, s);
      return launch_euler_cartesian<4>(E, D_host, gamma, scale, U, R, s);
    case 5:  // warp kernel (25 of 32 lanes) measured 0.98 vs 0.84 ms: CTA kernel
      if (SFB_NODE_N5) return launch_euler_cart_node<5>(E, D_host, gamma, scale, U, R, ws, s);
      if (SFB_SYNC_N5) return launch_euler_cart_sync<5>(E, D_host, gamma, scale, U, R, ws, s);
      return SFB_WARP_SMALL > 1 ? launch_euler_cart_warp<5>(E, D_host, gamma, scale, U, R, s)
                                : launch_euler_cartesian<5>(E, D_host, gamma, scale, U, R, s);
    case 6:
      if (SFB_NODE_N6) return launch_euler_cart_node<6>(E, D_host, gamma, scale, U, R, ws, s);
      if (SFB_SYNC_N6) return launch_euler_cart_sync<6>(E, D_host, gamma, scale, U, R, ws, s);
      return launch_euler_cartesian<6>(E, D_host, gamma, scale, U, R, s);
    case 7:
      if (SFB_NODE_N7) return launch_euler_cart_node<7>(E, D_host, gamma, scale, U, R, ws, s);
      if (SFB_SYNC_N7) return launch_euler_cart_sync<7>(E, D_host, gamma, scale, U, R, ws, s);
      return launch_euler_cartesian<7>(E, D_host, gamma, scale, U, R, s);
    case 8:
      if (SFB_NODE_N8) return launch_euler_cart_node<8>(E, D_host, gamma, scale, U, R, ws, s);
      if (SFB_SYNC_N8) return launch_euler_cart_sync<8>(E, D_host, gamma, scale, U, R, ws, s);
      return launch_euler_cartesian<8>(E, D_host, gamma, scale, U, R, s);
    default: return fail(SFB_ENOTSUP, "euler_volume_cartesian: n must be in 2..8");
  }
}

}  // namespace sfb

using namespace sfb;

// D is a HOST pointer (n x n, folded into the kernel's parameter block); the
// Python layer passes the host-built operator exactly as the reference builds
// it (operators.py:136-152).
extern "C" int sfb_euler_volume_cartesian(int64_t E, int64_t n, const double* D, double gamma,
                                          double scale, const double* U, double* R,
                                          sfb_stream_t stream) {
  SFB_CHECK_ARG(E >= 0, "negative element count");
  SFB_CHECK_ARG(D != nullptr, "null D");
  SFB_CHECK_ARG(gamma > 1.0, "gamma must exceed 1");
  if (E == 0) return SFB_OK;
  SFB_CHECK_ARG(U && R, "null state pointer");
  SFB_CHECK_ARG(((uintptr_t)U % 16) == 0 && ((uintptr_t)R % 16) == 0,
                "U and R must be 16-byte aligned");
  return euler_cartesian_dispatch(E, n, D, gamma, scale, U, R, nullptr, (cudaStream_t)stream);
}

// The same with an 8-byte device workspace: the n >= 5 persistent kernels
// then claim elements from a counter the call zeroes on `stream` (a CTA on a
// slower SM takes fewer elements) instead of the static split; results are
// bitwise the same.  Concurrent calls need distinct workspaces.
extern "C" int sfb_euler_volume_cartesian_ws(int64_t E, int64_t n, const double* D, double gamma,
                                             double scale, const double* U, double* R,
                                             void* workspace, sfb_stream_t stream) {
  SFB_CHECK_ARG(E >= 0, "negative element count");
  SFB_CHECK_ARG(D != nullptr, "null D");
  SFB_CHECK_ARG(gamma > 1.0, "gamma must exceed 1");
  SFB_CHECK_ARG((uintptr_t)workspace % 8 == 0, "workspace must be 8-byte aligned");
  if (E == 0) return SFB_OK;
  SFB_CHECK_ARG(U && R, "null state pointer");
  SFB_CHECK_ARG(((uintptr_t)U % 16) == 0 && ((uintptr_t)R % 16) == 0,
                "U and R must be 16-byte aligned");
  return euler_cartesian_dispatch(E, n, D, gamma, scale, U, R, workspace, (cudaStream_t)stream);
}
