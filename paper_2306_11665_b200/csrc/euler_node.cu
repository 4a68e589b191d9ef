// K3 for n = 5..8, lane-per-node lines: the Cartesian Euler volume term
//
//   R[e,:,r] = scale * sum_j sum_l D[r_j,l] F#_j(U[e,:,r], U[e,:,r(j->l)])
//
// (burgers.py:117-131 generalised, as euler.cu / euler_sync.cu) with the pair
// stage laid out so that a thread holds ONE node's accumulators instead of a
// whole line's.  A line of n nodes is owned by a group of n consecutive lanes
// (floor(32/n) groups per warp); lane i keeps node i's record and its five
// accumulators in registers.  In round r lane i evaluates the pair
// (i, i+r mod n) - every unordered pair of the line exactly once over the
// rounds r = 1 .. (n-1)/2 for odd n - with the partner's record fetched by
// warp shuffles, and adds D[i][i+r] F to its own node; in the same round it
// receives (by a shuffle) the F of the pair (i-r, i) evaluated by lane i-r and
// adds D[i][i-r] F.  Per pair: ~54 FP64 operations,
// 7 + 5 64-bit shuffles (a 64-bit shuffle runs at one warp-instruction per
// clock per SM, twice the rate of a 64-bit shared load:
// tools/peaks/shfl_rate.cu), no shared-memory traffic.  For even n a task is
// TWO lines of the same direction: n/2 - 1 regular rounds per line, then one
// round in which lanes i < n/2 take line A's antipodal pair (i, i+n/2) and
// lanes i >= n/2 line B's (i-n/2, i), so no lane idles (n - 1 rounds for the
// task's n(n-1) pairs).  KB rounds are evaluated side by side (ILP).
//
// Per element (persistent CTAs, dynamic claims as in euler_sync.cu):
//   stage B  thread per node: node record (hr, hv, (gamma-1) beta, logs) into
//            shared memory, the diagonal term into the residual;
//   stage C  lane-group tasks (above); x0 results into the consumed state slot,
//            x1 results into their own buffer, x2 results added onto the
//            residual (every node on exactly one line per direction);
//   stage D  R = ((diag + x2) + x0) + x1, streaming stores.
//
// Measured (config 4, ncu at n = 6): the FP64 work per pair is the line
// kernels', but the shuffles (24 SHFL.32 per pair), the selects and the index
// arithmetic take ~58% of the issue slots, and the FP64 pipe stays at 44%;
// two rounds side by side (SFB_NODE_KB = 2) and more resident warps did not
// change the times.  It is the default at n = 7 only (1.27 vs 1.31 ms),
// where the line kernels spill.
#include "euler_common.cuh"

#ifndef SFB_NODE_KB
#define SFB_NODE_KB 1
#endif
#ifndef SFB_NODE_WARPS_N5
#define SFB_NODE_WARPS_N5 4
#endif
#ifndef SFB_NODE_WARPS_N6
#define SFB_NODE_WARPS_N6 4
#endif
#ifndef SFB_NODE_WARPS_N7
#define SFB_NODE_WARPS_N7 4
#endif
#ifndef SFB_NODE_WARPS_N8
#define SFB_NODE_WARPS_N8 6
#endif
#ifndef SFB_NODE_MB_N5
#define SFB_NODE_MB_N5 3
#endif
#ifndef SFB_NODE_MB_N6
#define SFB_NODE_MB_N6 3
#endif
#ifndef SFB_NODE_MB_N7
#define SFB_NODE_MB_N7 4  // 4 CTAs (16 warps) at 110 registers: 1.272 vs 1.280 ms with 3
#endif
#ifndef SFB_NODE_MB_N8
#define SFB_NODE_MB_N8 2
#endif

namespace sfb {

template <int N>
struct NodeCfg {
  static constexpr int kNodes = N * N * N;
  static constexpr int kLines = N * N;
  static constexpr int kGroups = 32 / N;              // lane groups per warp
  static constexpr int kLPT = (N % 2 == 0) ? 2 : 1;   // lines per task
  static constexpr int kTasks = 3 * kLines / kLPT;
  static constexpr int kReg = (N % 2) ? (N - 1) / 2 : N / 2 - 1;  // regular rounds per line
  static constexpr int kWarps = N == 5   ? SFB_NODE_WARPS_N5
                                : N == 6 ? SFB_NODE_WARPS_N6
                                : N == 7 ? SFB_NODE_WARPS_N7
                                         : SFB_NODE_WARPS_N8;
  static constexpr int kMinBlocks = N == 5   ? SFB_NODE_MB_N5
                                    : N == 6 ? SFB_NODE_MB_N6
                                    : N == 7 ? SFB_NODE_MB_N7
                                             : SFB_NODE_MB_N8;
  static constexpr int kThreads = 32 * kWarps;
  static constexpr int kU = 5 * kNodes;
  static constexpr int kSlot = ((kU + 1) + 1) / 2 * 2;  // + 1 for the 16-B alignment shift
  static constexpr size_t kSmem = (size_t)(2 * kSlot + 7 * kNodes + 2 * kU) * sizeof(double);
};

__device__ __forceinline__ NodeRec shfl_rec(const NodeRec& q, int src) {
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

__device__ __forceinline__ NodeRec sel_rec(bool p, const NodeRec& a, const NodeRec& b) {
  NodeRec r;
  r.hr = dsel(p, a.hr, b.hr);
  r.hv0 = dsel(p, a.hv0, b.hv0);
  r.hv1 = dsel(p, a.hv1, b.hv1);
  r.hv2 = dsel(p, a.hv2, b.hv2);
  r.hb = dsel(p, a.hb, b.hb);
  r.hlr = dsel(p, a.hlr, b.hlr);
  r.hlb = dsel(p, a.hlb, b.hlb);
  return r;
}

template <int NN>
__device__ __forceinline__ NodeRec load_rec(const double* rec, int k, int vp0, int vp1, int vp2) {
  NodeRec q;
  q.hr = rec[k];
  q.hv0 = rec[vp0 + k];
  q.hv1 = rec[vp1 + k];
  q.hv2 = rec[vp2 + k];
  q.hb = rec[4 * NN + k];
  q.hlr = rec[5 * NN + k];
  q.hlb = rec[6 * NN + k];
  return q;
}

// regular rounds r0 .. r0+KB-1 of one line: own record `me`, accumulators acc
template <int KB>
__device__ __forceinline__ void node_rounds(const NodeRec& me, const int (&srcP)[KB],
                                            const int (&srcF)[KB], const double (&dOwn)[KB],
                                            const double (&dRecv)[KB], double gm1,
                                            double (&acc)[5]) {
  NodeRec part[KB];
  const NodeRec* A[KB];
  const NodeRec* B[KB];
#pragma unroll
  for (int k = 0; k < KB; ++k) {
    part[k] = shfl_rec(me, srcP[k]);
    A[k] = &me;
    B[k] = &part[k];
  }
  double f[KB][5];
  chandrashekar_cart_v2<KB>(A, B, gm1, f);
#pragma unroll
  for (int k = 0; k < KB; ++k) {
#pragma unroll
    for (int v = 0; v < 5; ++v) {
      acc[v] = fma(dOwn[k], f[k][v], acc[v]);
      const double fr = __shfl_sync(0xffffffffu, f[k][v], srcF[k]);
      acc[v] = fma(dRecv[k], fr, acc[v]);
    }
  }
}

template <int N>
__global__ void __launch_bounds__(NodeCfg<N>::kThreads, NodeCfg<N>::kMinBlocks)
    euler_cart_node_kernel(int64_t E, const __grid_constant__ DMat<N> Dm, double gm1,
                           const double* __restrict__ U, double* __restrict__ R,
                           unsigned long long* claim_ctr) {
  using Cfg = NodeCfg<N>;
  constexpr int NN = Cfg::kNodes;
  constexpr int T = Cfg::kThreads;
  constexpr int KU = Cfg::kU;
  constexpr int KR = Cfg::kReg;
  constexpr int KB = SFB_NODE_KB < KR ? SFB_NODE_KB : KR;
  extern __shared__ __align__(16) double smem[];
  double* slots = smem;                 // [2][kSlot] element states (bulk-copy targets)
  double* rec = smem + 2 * Cfg::kSlot;  // [7][NN] node records
  double* res = rec + 7 * NN;           // [5][NN] diagonal term, then + x2 results
  double* buf1 = res + KU;              // [5][NN] x1 results
  __shared__ uint64_t full[2];
  __shared__ long long s_next[2];
  const int tid = threadIdx.x;
  const double hgm1 = 0.5 * gm1;
  if (tid == 0) {
    mbar_init(&full[0], 1);
    mbar_init(&full[1], 1);
    fence_mbar_init();
  }

  // ---- lane-group geometry and per-lane round constants (fixed) ------------
  const int lane = tid & 31, warp = tid >> 5;
  const int gl = lane / N;
  const bool lane_ok = gl < Cfg::kGroups;
  const int i = lane_ok ? lane - gl * N : 0;     // node position along the line
  const int gbase = lane_ok ? gl * N : 0;        // lane of the group's node 0
  const int gid = warp * Cfg::kGroups + (lane_ok ? gl : 0);
  constexpr int G = Cfg::kGroups * Cfg::kWarps;  // groups per CTA
  int srcP[KR], srcF[KR];
  double dOwn[KR], dRecv[KR];
#pragma unroll
  for (int r = 1; r <= KR; ++r) {
    const int p = (i + r) % N, q = (i - r + N) % N;
    srcP[r - 1] = gbase + p;
    srcF[r - 1] = gbase + q;
    dOwn[r - 1] = Dm.d[i * N + p];
    dRecv[r - 1] = Dm.d[i * N + q];
  }
  const int hN = N / 2;
  const int srcH = gbase + (i + hN) % N;
  const double dH = Dm.d[i * N + (i + hN) % N];
  const bool lowhalf = i < hN;

  // element states: offset e*KU is odd for odd n and odd e: copy one double
  // early (16-B alignment) and read at `shift` = 1; a final element whose
  // aligned copy would run past the end of U is read with plain loads
  const int64_t total = E * KU;
  auto shift_of = [](int64_t e) { return (int)((e * KU) & 1); };
  auto copy_doubles = [&](int64_t e) { return (shift_of(e) + KU + 1) & ~1; };
  auto bulk_ok = [&](int64_t e) { return e * KU - shift_of(e) + copy_doubles(e) <= total; };
  auto issue = [&](int64_t e, int slot) {
    const uint32_t bytes = (uint32_t)copy_doubles(e) * 8u;
    mbar_arrive_expect_tx(&full[slot], bytes);
    bulk_g2s(slots + slot * Cfg::kSlot, U + e * KU - shift_of(e), bytes, &full[slot]);
  };
  auto l2_prefetch = [&](int64_t e) {
    if (e < E && bulk_ok(e))
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(U + e * KU - shift_of(e)),
                   "r"((uint32_t)copy_doubles(e) * 8u)
                   : "memory");
  };
  const bool dyn = claim_ctr != nullptr;
  auto claim = [&](int k) -> int64_t {
    return dyn ? (int64_t)gridDim.x + (int64_t)atomicAdd(claim_ctr, 1ull)
               : (int64_t)blockIdx.x + (int64_t)k * gridDim.x;
  };
  __syncthreads();
  if (tid == 0 && (int64_t)blockIdx.x < E) {
    if (bulk_ok(blockIdx.x)) issue(blockIdx.x, 0);
    const int64_t e1 = claim(1);
    s_next[0] = e1;
    l2_prefetch(e1);
  }
  __syncthreads();
  uint32_t parity = 0;

  int it = 0;
  for (int64_t e = blockIdx.x; e < E; ++it) {
    if (tid == 0 && s_next[it & 1] < E) {
      const int64_t nn = claim(it + 2);
      s_next[(it + 1) & 1] = nn;
      l2_prefetch(nn);
    }
    const int slot = it & 1;
    double* in = slots + slot * Cfg::kSlot;
    if (bulk_ok(e)) {
      mbar_wait_parity(&full[slot], (parity >> slot) & 1u);
      parity ^= 1u << slot;
      in += shift_of(e);
    } else {
      for (int k = tid; k < KU; k += T) in[k] = __ldcs(U + e * KU + k);
      __syncthreads();
    }
    const int64_t nxt = tid == 0 ? s_next[it & 1] : E;
    if (tid == 0 && nxt < E && bulk_ok(nxt)) {
      fence_proxy_async_smem();  // the other slot was last read before the last barrier
      issue(nxt, slot ^ 1);
    }

    // ---- stage B: node records + diagonal term ------------------------------
    for (int r = tid; r < NN; r += T) {
      const double* u = in + r;
      const double rho = u[0], m0 = u[NN], m1 = u[2 * NN], m2 = u[3 * NN], et = u[4 * NN];
      const double irho = rcp_refined(rho);
      const double hirho = 0.5 * irho;
      const double mm = fma(m2, m2, fma(m1, m1, m0 * m0));
      const double X2 = fma(rho, et + et, -mm);
      const double iX2 = rcp_refined(X2);
      const double p = (hgm1 * X2) * irho;
      const double hbeta = (rho * rho) * iX2;
      rec[r] = 0.5 * rho;
      rec[NN + r] = m0 * hirho;
      rec[2 * NN + r] = m1 * hirho;
      rec[3 * NN + r] = m2 * hirho;
      rec[4 * NN + r] = hbeta;
      rec[5 * NN + r] = log_half(rho);
      rec[6 * NN + r] = log_half(hbeta);
      const int c0 = r % N, c1 = (r / N) % N, c2 = r / (N * N);
      const double d0 = Dm.d[c0 * (N + 1)], d1 = Dm.d[c1 * (N + 1)], d2 = Dm.d[c2 * (N + 1)];
      const double mass = fma(m2, d2, fma(m1, d1, m0 * d0));
      const double wv = mass * irho;
      res[r] = mass;
      res[NN + r] = fma(m0, wv, p * d0);
      res[2 * NN + r] = fma(m1, wv, p * d1);
      res[3 * NN + r] = fma(m2, wv, p * d2);
      res[4 * NN + r] = (et + p) * wv;
    }
    __syncthreads();  // records ready; the state slot is free for the x0 results

    // ---- stage C: lane-group line tasks (warp-uniform steps) -----------------
    constexpr int kSteps = (Cfg::kTasks + G - 1) / G;
#pragma unroll 1
    for (int st = 0; st < kSteps; ++st) {
      int task = st * G + gid;
      const bool valid = lane_ok && task < Cfg::kTasks;
      task = valid ? task : 0;  // idle lanes shadow a real task (shuffle partners), no writes
      const int line0 = task * Cfg::kLPT;
      const int dir = line0 / Cfg::kLines;
      const int L0 = line0 - dir * Cfg::kLines;
      const int stride = dir == 0 ? 1 : (dir == 1 ? N : N * N);
      const int vp0 = (1 + dir % 3) * NN, vp1 = (1 + (dir + 1) % 3) * NN,
                vp2 = (1 + (dir + 2) % 3) * NN;
      auto line_base = [&](int L) {
        const int u0 = L % N, u1 = L / N;
        return dir == 0 ? u0 * N + u1 * N * N : (dir == 1 ? u0 + u1 * N * N : u0 + u1 * N);
      };
      const int kA = line_base(L0) + i * stride;
      NodeRec A = load_rec<NN>(rec, kA, vp0, vp1, vp2);
      double accA[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
#pragma unroll
      for (int r0 = 0; r0 < KR; r0 += KB) {
        constexpr int kb = KB;
        int sp[kb], sf[kb];
        double dow[kb], drc[kb];
#pragma unroll
        for (int k = 0; k < kb; ++k) {
          const int rr = r0 + k < KR ? r0 + k : KR - 1;
          sp[k] = srcP[rr];
          sf[k] = srcF[rr];
          dow[k] = r0 + k < KR ? dOwn[rr] : 0.0;
          drc[k] = r0 + k < KR ? dRecv[rr] : 0.0;
        }
        node_rounds<kb>(A, sp, sf, dow, drc, gm1, accA);
      }
      if constexpr (Cfg::kLPT == 2) {
        const int kB = line_base(L0 + 1) + i * stride;
        NodeRec B = load_rec<NN>(rec, kB, vp0, vp1, vp2);
        double accB[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
#pragma unroll
        for (int r0 = 0; r0 < KR; r0 += KB) {
          constexpr int kb = KB;
          int sp[kb], sf[kb];
          double dow[kb], drc[kb];
#pragma unroll
          for (int k = 0; k < kb; ++k) {
            const int rr = r0 + k < KR ? r0 + k : KR - 1;
            sp[k] = srcP[rr];
            sf[k] = srcF[rr];
            dow[k] = r0 + k < KR ? dOwn[rr] : 0.0;
            drc[k] = r0 + k < KR ? dRecv[rr] : 0.0;
          }
          node_rounds<kb>(B, sp, sf, dow, drc, gm1, accB);
        }
        // antipodal round: lanes i < n/2 take line A's pair (i, i+n/2), lanes
        // i >= n/2 line B's pair (i-n/2, i); each sends the other line's record
        {
          const NodeRec me = sel_rec(lowhalf, A, B);
          const NodeRec send = sel_rec(lowhalf, B, A);
          const NodeRec part = shfl_rec(send, srcH);
          const NodeRec* PA[1] = {&me};
          const NodeRec* PB[1] = {&part};
          double f[1][5];
          chandrashekar_cart_v2<1>(PA, PB, gm1, f);
#pragma unroll
          for (int v = 0; v < 5; ++v) {
            const double own = dH * f[0][v];
            const double fr = dH * __shfl_sync(0xffffffffu, f[0][v], srcH);
            accA[v] += dsel(lowhalf, own, fr);
            accB[v] += dsel(lowhalf, fr, own);
          }
        }
        if (valid) {
          double* db = dir == 0 ? in : (dir == 1 ? buf1 : res);
          if (dir == 2) {
            res[kB] += accB[0];
            res[vp0 + kB] += accB[1];
            res[vp1 + kB] += accB[2];
            res[vp2 + kB] += accB[3];
            res[4 * NN + kB] += accB[4];
          } else {
            db[kB] = accB[0];
            db[vp0 + kB] = accB[1];
            db[vp1 + kB] = accB[2];
            db[vp2 + kB] = accB[3];
            db[4 * NN + kB] = accB[4];
          }
        }
      }
      if (valid) {
        double* db = dir == 0 ? in : (dir == 1 ? buf1 : res);
        if (dir == 2) {
          res[kA] += accA[0];
          res[vp0 + kA] += accA[1];
          res[vp1 + kA] += accA[2];
          res[vp2 + kA] += accA[3];
          res[4 * NN + kA] += accA[4];
        } else {
          db[kA] = accA[0];
          db[vp0 + kA] = accA[1];
          db[vp1 + kA] = accA[2];
          db[vp2 + kA] = accA[3];
          db[4 * NN + kA] = accA[4];
        }
      }
    }
    __syncthreads();

    // ---- stage D: R = ((diag + x2) + x0) + x1 --------------------------------
    double* Rg = R + e * KU;
    for (int k = tid; k < KU; k += T) __stcs(Rg + k, (res[k] + in[k]) + buf1[k]);
    const int64_t e_next = s_next[it & 1];
    __syncthreads();  // res / rec / buf1 / the slot are rewritten by the next element
    e = e_next;
  }
}

template <int N>
int launch_euler_cart_node(int64_t E, const double* Dh, double gamma, double scale,
                           const double* U, double* R, void* ws, cudaStream_t s) {
  using Cfg = NodeCfg<N>;
  DMat<N> Dm;
  for (int k = 0; k < N * N; ++k) Dm.d[k] = scale * Dh[k];
  static DeviceCache cache;
  const int ps = resident_ctas(euler_cart_node_kernel<N>, Cfg::kThreads, Cfg::kSmem, cache);
  int64_t grid = (int64_t)num_sms() * ps;
  if (grid > E) grid = E;
  unsigned long long* ctr = static_cast<unsigned long long*>(ws);
  if (ctr && cudaMemsetAsync(ctr, 0, sizeof(unsigned long long), s) != cudaSuccess)
    return fail(SFB_ECUDA, "claim counter reset failed");
  euler_cart_node_kernel<N><<<(unsigned)grid, Cfg::kThreads, Cfg::kSmem, s>>>(E, Dm, gamma - 1.0,
                                                                              U, R, ctr);
  return check_launch("euler_volume_cartesian");
}

template int launch_euler_cart_node<5>(int64_t, const double*, double, double, const double*,
                                       double*, void*, cudaStream_t);
template int launch_euler_cart_node<6>(int64_t, const double*, double, double, const double*,
                                       double*, void*, cudaStream_t);
template int launch_euler_cart_node<7>(int64_t, const double*, double, double, const double*,
                                       double*, void*, cudaStream_t);
template int launch_euler_cart_node<8>(int64_t, const double*, double, double, const double*,
                                       double*, void*, cudaStream_t);

}  // namespace sfb
