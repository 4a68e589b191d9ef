// K3 for n = 5..8 (config 4's upper points): the Cartesian Euler volume term
//
//   R[e,:,r] = scale * sum_j sum_l D[r_j,l] F#_j(U[e,:,r], U[e,:,r(j->l)])
//
// (burgers.py:117-131 generalised, as in euler.cu) with one CTA per element
// and every warp in every stage, separated by CTA barriers - the structure of
// the config-5 kernel (modal.cu) without its transforms and metric terms.
//
// Why not euler.cu's warp-specialised kernel: there one prep warp builds the
// node records of the next element while the line warps work, so a CTA needs
// two record sets and three direction buffers (71 KB at n = 6, 168 KB at
// n = 8) and 4-6 line warps + 1 prep warp: 10 warps per SM at n = 6, 7 at
// n = 8.  Here the element's state slot, records and residual are all the
// shared memory (22 n^3 doubles: 38 KB at n = 6, 90 KB at n = 8), so the SM
// holds 12 line-working warps at n = 5, 6, 8 (and 10 at n = 7) and a CTA's
// barrier wait is covered by the other CTAs.  Measured (config 4): faster at
// n = 6 only (0.95 vs 1.01 ms, the default there); at n = 5, 7, 8 the
// warp-specialised kernel stays ahead (0.79 / 1.34 / 1.27 vs 1.00 / 1.46 /
// 1.33 ms here): the lean pair loop has little ILP and the extra warps do not
// make up for the CTA barriers and the records stage's idle lanes.  (ncu:
// LDCU - the pair loop's D coefficients from the parameter bank - is 15% of
// the stall samples, but the coefficients from shared memory measured slower,
// 0.983 vs 0.953 ms.)
//
// Per element (persistent CTAs, grid = resident CTAs; the next element's
// states stream into the other slot by one 1-D bulk copy (UBLKCP) on an
// mbarrier, and the one after it into L2):
//   stage B  thread per node: primitives, node record (hr, hv, (gamma-1) beta,
//            ln rho / 2, ln hb / 2), the diagonal term sum_j D[r_j,r_j] f_j(u_r)
//            into the residual;
//   stage C  thread per (direction, line): each symmetric pair once in the
//            direction-rotated frame (chandrashekar_cart_v2), scattered to both
//            rows; register-lean loop (node b re-read from shared memory per
//            pair).  After a barrier the x0 results go to the consumed state
//            slot, the x1 results to the record planes and the x2 results are
//            added onto the residual (each node is on exactly one line per
//            direction: plain stores, no atomics);
//   stage D  R = ((diag + x2) + x0) + x1, streaming stores.
#include "euler_common.cuh"

#ifndef SFB_SYNC_MB_N5
#define SFB_SYNC_MB_N5 4
#endif
#ifndef SFB_SYNC_MB_N6
#define SFB_SYNC_MB_N6 3
#endif
#ifndef SFB_SYNC_MB_N7
#define SFB_SYNC_MB_N7 2
#endif
#ifndef SFB_SYNC_MB_N8
#define SFB_SYNC_MB_N8 2
#endif
#ifndef SFB_SYNC_K
#define SFB_SYNC_K 2  // pairs side by side in the lean loop (n = 6: 0.938 vs 0.950 ms with 1)
#endif
#ifndef SFB_SYNC_TABLOG
#define SFB_SYNC_TABLOG 0  // table-driven node logarithms: n = 6 0.973 vs 0.952 ms
#endif
#ifndef SFB_SYNC_L2PF
#define SFB_SYNC_L2PF 1  // L2 prefetch one element beyond the shared-memory copy
#endif

namespace sfb {

template <int N>
struct SyncCfg {
  static constexpr int kNodes = N * N * N;
  static constexpr int kLineThreads = 3 * N * N;
  static constexpr int kThreads = ((kLineThreads + 31) / 32) * 32;
  static constexpr int kU = 5 * kNodes;               // doubles of one element's states
  static constexpr int kSlot = ((kU + 1) + 1) / 2 * 2;  // + 1 for the 16-B alignment shift
  static constexpr int kRec = 7 * kNodes;
  static constexpr size_t kSmem = (size_t)(2 * kSlot + kRec + kU) * sizeof(double);
  static constexpr int kMinBlocks = N == 5   ? SFB_SYNC_MB_N5
                                    : N == 6 ? SFB_SYNC_MB_N6
                                    : N == 7 ? SFB_SYNC_MB_N7
                                             : SFB_SYNC_MB_N8;
  // register cap for kMinBlocks CTAs per SM (multiple of 8, at most 255)
  static constexpr int kRegCap = 65536 / (kMinBlocks * kThreads) / 8 * 8;
  static constexpr int kMaxRegs = kRegCap > 255 ? 255 : kRegCap;
};

__device__ __forceinline__ double vld_shared(uint32_t addr) {
  double x;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(x) : "r"(addr));
  return x;
}

// Node record k with the velocity planes permuted into the line's frame.
// Volatile loads: the compiler may not keep every record of the line live
// (that is what keeps the loop at ~168 registers).
template <int NN>
__device__ __forceinline__ NodeRec vload_rec(uint32_t rec, int k, int vp0, int vp1, int vp2) {
  NodeRec q;
  const uint32_t a = rec + 8u * (uint32_t)k;
  q.hr = vld_shared(a);
  q.hv0 = vld_shared(a + 8u * (uint32_t)vp0);
  q.hv1 = vld_shared(a + 8u * (uint32_t)vp1);
  q.hv2 = vld_shared(a + 8u * (uint32_t)vp2);
  q.hb = vld_shared(a + 8u * 4u * NN);
  q.hlr = vld_shared(a + 8u * 5u * NN);
  q.hlb = vld_shared(a + 8u * 6u * NN);
  return q;
}

template <int N, int KB>
__device__ __forceinline__ void sync_batch(uint32_t rec, int base, int stride, int vp0, int vp1,
                                           int vp2, int a, int b0, const NodeRec& qa,
                                           const DMat<N>& Dm, double gm1, double (&acc)[N][5]) {
  constexpr int NN = N * N * N;
  NodeRec qb[KB];
  const NodeRec* A[KB];
  const NodeRec* B[KB];
#pragma unroll
  for (int k = 0; k < KB; ++k) {
    qb[k] = vload_rec<NN>(rec, base + (b0 + k) * stride, vp0, vp1, vp2);
    A[k] = &qa;
    B[k] = &qb[k];
  }
  double f[KB][5];
  chandrashekar_cart_v2<KB>(A, B, gm1, f);
#pragma unroll
  for (int k = 0; k < KB; ++k) {
    const int b = b0 + k;
    const double dab = Dm.d[a * N + b], dba = Dm.d[b * N + a];
#pragma unroll
    for (int v = 0; v < 5; ++v) {
      acc[a][v] = fma(dab, f[k][v], acc[a][v]);
      acc[b][v] = fma(dba, f[k][v], acc[b][v]);
    }
  }
}

template <int N>
__global__ void __launch_bounds__(SyncCfg<N>::kThreads) __maxnreg__(SyncCfg<N>::kMaxRegs)
    euler_cart_sync_kernel(int64_t E, const __grid_constant__ DMat<N> Dm, double gm1,
                           const double* __restrict__ U, double* __restrict__ R,
                           unsigned long long* claim_ctr) {
  using Cfg = SyncCfg<N>;
  constexpr int NN = Cfg::kNodes;
  constexpr int T = Cfg::kThreads;
  constexpr int KU = Cfg::kU;
  extern __shared__ __align__(16) double smem[];
  double* slots = smem;                 // [2][kSlot] element states (bulk-copy targets)
  double* rec = smem + 2 * Cfg::kSlot;  // [7][NN] node records, natural node order
  double* res = rec + Cfg::kRec;        // [5][NN] diagonal term, then + x2 results
  __shared__ uint64_t full[2];
  const int tid = threadIdx.x;
  const double hgm1 = 0.5 * gm1;
  if (tid == 0) {
    mbar_init(&full[0], 1);
    mbar_init(&full[1], 1);
    fence_mbar_init();
  }
  __syncthreads();

  // An element's states start at double offset e*KU, odd for odd n and odd e:
  // the copy then starts one double early (16-B alignment) and the states are
  // read at `shift` = 1.  Only a final element whose aligned copy would run
  // past the end of U is read with plain loads.
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
  // Element order: e_0 = blockIdx.x, then (with a claim counter) elements
  // claimed one ahead from it - a CTA on a slower SM takes fewer - or
  // (static) e_0 + k gridDim.x.  s_next[it & 1] = the element after
  // iteration it's: written by thread 0 at the top of iteration it - 1 (the
  // prologue for it = 0), read by every thread before iteration it's final
  // barrier, rewritten only after it.
  __shared__ long long s_next[2];
  const bool dyn = claim_ctr != nullptr;
  auto claim = [&](int k) -> int64_t {
    return dyn ? (int64_t)gridDim.x + (int64_t)atomicAdd(claim_ctr, 1ull)
               : (int64_t)blockIdx.x + (int64_t)k * gridDim.x;
  };
  if (tid == 0 && (int64_t)blockIdx.x < E) {
    if (bulk_ok(blockIdx.x)) issue(blockIdx.x, 0);
    const int64_t e1 = claim(1);
    s_next[0] = e1;
    if (SFB_SYNC_L2PF > 0) l2_prefetch(e1);
  }
  __syncthreads();
  uint32_t parity = 0;  // bit s = phase of slot s

  // stage-C geometry of this thread's line (fixed for the whole kernel)
  const int dir = tid / (N * N);
  const int L = tid - dir * N * N;
  const bool active = tid < Cfg::kLineThreads;
  const int u0 = L % N, u1 = L / N;
  const int base = dir == 0 ? u0 * N + u1 * N * N : (dir == 1 ? u0 + u1 * N * N : u0 + u1 * N);
  const int stride = dir == 0 ? 1 : (dir == 1 ? N : N * N);
  // velocity planes in the line's frame: hv0 along the line
  const int vp0 = (1 + dir % 3) * NN, vp1 = (1 + (dir + 1) % 3) * NN,
            vp2 = (1 + (dir + 2) % 3) * NN;
  const uint32_t rec_s = smem_u32(rec);

  int it = 0;
  for (int64_t e = blockIdx.x; e < E; ++it) {
    if (tid == 0 && s_next[it & 1] < E) {
      const int64_t nn = claim(it + 2);
      s_next[(it + 1) & 1] = nn;
      if (SFB_SYNC_L2PF > 0) l2_prefetch(nn);
    }
    const int slot = it & 1;
    double* in = slots + slot * Cfg::kSlot;
    if (bulk_ok(e)) {
      mbar_wait_parity(&full[slot], (parity >> slot) & 1u);
      parity ^= 1u << slot;
      in += shift_of(e);
    } else {
      for (int i = tid; i < KU; i += T) in[i] = __ldcs(U + e * KU + i);
      __syncthreads();
    }
    const int64_t nxt = tid == 0 ? s_next[it & 1] : E;
    if (tid == 0 && nxt < E && bulk_ok(nxt)) {
      // the other slot was last read before the previous iteration's final barrier
      fence_proxy_async_smem();
      issue(nxt, slot ^ 1);
    }

    // ---- stage B: node records + diagonal term ------------------------------
    for (int r = tid; r < NN; r += T) {
      const double* u = in + r;
      const double rho = u[0], m0 = u[NN], m1 = u[2 * NN], m2 = u[3 * NN], et = u[4 * NN];
      const double irho = rcp_refined(rho);
      const double hirho = 0.5 * irho;
      const double mm = fma(m2, m2, fma(m1, m1, m0 * m0));
      const double X2 = fma(rho, et + et, -mm);  // 2 (rho E - |m|^2/2) = 2 rho p / (gamma-1)
      const double iX2 = rcp_refined(X2);
      const double p = (hgm1 * X2) * irho;
      const double hbeta = (rho * rho) * iX2;  // (gamma - 1) beta
      rec[r] = 0.5 * rho;
      rec[NN + r] = m0 * hirho;
      rec[2 * NN + r] = m1 * hirho;
      rec[3 * NN + r] = m2 * hirho;
      rec[4 * NN + r] = hbeta;
      rec[5 * NN + r] = SFB_SYNC_TABLOG ? log_half_tab(rho) : log_half(rho);
      rec[6 * NN + r] = SFB_SYNC_TABLOG ? log_half_tab(hbeta) : log_half(hbeta);
      // sum_j D[r_j,r_j] f_j(u): mass = sum_j d_j m_j, w = mass / rho:
      // (mass, w m + p d, (E + p) w)
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
    __syncthreads();

    // ---- stage C: one thread per (direction, line) -------------------------
    double acc[N][5];
#pragma unroll
    for (int a = 0; a < N; ++a)
#pragma unroll
      for (int v = 0; v < 5; ++v) acc[a][v] = 0.0;
    if (active) {
#pragma unroll
      for (int a = 0; a < N - 1; ++a) {
        const NodeRec qa = vload_rec<NN>(rec_s, base + a * stride, vp0, vp1, vp2);
#pragma unroll
        for (int b0 = a + 1; b0 < N; b0 += SFB_SYNC_K) {
          if (SFB_SYNC_K == 2 && b0 + 1 < N)
            sync_batch<N, 2>(rec_s, base, stride, vp0, vp1, vp2, a, b0, qa, Dm, gm1, acc);
          else
            sync_batch<N, 1>(rec_s, base, stride, vp0, vp1, vp2, a, b0, qa, Dm, gm1, acc);
        }
      }
    }
    __syncthreads();  // every line has read the records; the state slot is free
    if (active) {
      // momentum results come back in the line's frame: un-rotate by address
#pragma unroll
      for (int a = 0; a < N; ++a) {
        const int k = base + a * stride;
        if (dir == 2) {
          res[k] += acc[a][0];
          res[vp0 + k] += acc[a][1];
          res[vp1 + k] += acc[a][2];
          res[vp2 + k] += acc[a][3];
          res[4 * NN + k] += acc[a][4];
        } else {
          double* dst = dir == 0 ? in : rec;
          dst[k] = acc[a][0];
          dst[vp0 + k] = acc[a][1];
          dst[vp1 + k] = acc[a][2];
          dst[vp2 + k] = acc[a][3];
          dst[4 * NN + k] = acc[a][4];
        }
      }
    }
    __syncthreads();

    // ---- stage D: R = ((diag + x2) + x0) + x1 --------------------------------
    double* Rg = R + e * KU;
    for (int i = tid; i < KU; i += T) __stcs(Rg + i, (res[i] + in[i]) + rec[i]);
    const int64_t e_next = s_next[it & 1];
    __syncthreads();  // res / rec / the slot are rewritten by the next element
    e = e_next;
  }
}

template <int N>
int launch_euler_cart_sync(int64_t E, const double* Dh, double gamma, double scale,
                           const double* U, double* R, void* ws, cudaStream_t s) {
  using Cfg = SyncCfg<N>;
  DMat<N> Dm;
  for (int i = 0; i < N * N; ++i) Dm.d[i] = scale * Dh[i];
  static DeviceCache cache;
  const int ps = resident_ctas(euler_cart_sync_kernel<N>, Cfg::kThreads, Cfg::kSmem, cache);
  int64_t grid = (int64_t)num_sms() * ps;
  if (grid > E) grid = E;
  unsigned long long* ctr = static_cast<unsigned long long*>(ws);
  if (ctr && cudaMemsetAsync(ctr, 0, sizeof(unsigned long long), s) != cudaSuccess)
    return fail(SFB_ECUDA, "claim counter reset failed");
  euler_cart_sync_kernel<N><<<(unsigned)grid, Cfg::kThreads, Cfg::kSmem, s>>>(E, Dm, gamma - 1.0,
                                                                              U, R, ctr);
  return check_launch("euler_volume_cartesian");
}

template int launch_euler_cart_sync<5>(int64_t, const double*, double, double, const double*,
                                       double*, void*, cudaStream_t);
template int launch_euler_cart_sync<6>(int64_t, const double*, double, double, const double*,
                                       double*, void*, cudaStream_t);
template int launch_euler_cart_sync<7>(int64_t, const double*, double, double, const double*,
                                       double*, void*, cudaStream_t);
template int launch_euler_cart_sync<8>(int64_t, const double*, double, double, const double*,
                                       double*, void*, cudaStream_t);

}  // namespace sfb
