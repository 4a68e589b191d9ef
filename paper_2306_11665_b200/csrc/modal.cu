// K4: curvilinear, modal Euler volume term (BASELINE config 5).
//
//   u    = (V x V x V) Uhat                      modal -> GLL nodal (kronecker_apply,
//                                                 operators.py:274-318)
//   r    = scale sum_i sum_l D[r_i,l] Ft_i(u_r, u_r(i->l))
//          Ft_i(a,b) = F#(a, b; n = (Ja^i(a) + Ja^i(b))/2)   contravariant flux
//                                                 differencing (burgers.py:117-131
//                                                 generalised; Hadamard + row sum)
//   Rhat = (Pi x Pi x Pi) r                      nodal -> modal projection
//   sumsq[e] = sum Rhat[e]^2                     (fixed-order partial of the norm)
//
// One persistent CTA processes one element per iteration, taking its elements
// from a per-call claim counter (workspace) when one is given: with the static
// split e = blockIdx.x + k gridDim.x the CTAs on slower SMs set the end of the
// kernel (40.5 -> 38.6 ms at config 5 with the claims).  The next element's
// Uhat and Ja (8.6 KB + 15.6 KB at n = 6) are prefetched with two 1-D bulk
// copies (cp.async.bulk, UBLKCP) into the other half of a double buffer (and
// the one after it into L2, cp.async.bulk.prefetch) while the current
// element is transformed, differenced and projected - all in
// shared memory, so HBM sees exactly Uhat + Ja in and Rhat (+ 8 B) out.
//   stage A  three sum-factorised passes of V (one per direction), thread per
//            (variable, line), ping-ponging between the input slot and the residual buffer;
//   stage B  thread per node: primitives, per-node logs, node record; the
//            diagonal term sum_i D[r_i,r_i] F#(u_r,u_r; Ja^i(r)) into the
//            residual (consistency: F#(u,u;n) = f(u).n);
//   stage C  thread per (direction, line): each symmetric pair once, scattered
//            to both rows (register-lean loop, SFB_MODAL_LEAN); then, after a
//            barrier, the x0 residuals into the slot's free Uhat region, the x1
//            residuals into the record planes and the x2 residuals added into
//            the diagonal term (SFB_MODAL_COMPACT: 69 KB, 3 CTAs per SM);
//   stage D  three passes of Pi, the first summing the three buffers on the
//            fly, the last storing Rhat straight to HBM; per-thread squares
//            summed in a fixed order, xor-butterfly per warp, warps in
//            order -> sumsq[e].
// The metric averaging 1/2 is folded into D (Ft is linear in n).
#include "bulk.cuh"
#include "common.cuh"
#include "euler_flux.cuh"

#ifndef SFB_MODAL_MINBLOCKS_N6
#define SFB_MODAL_MINBLOCKS_N6 3
#endif
#ifndef SFB_MODAL_LEAN
#define SFB_MODAL_LEAN 1  // register-lean line loop (3 CTAs/SM at n = 6)
#endif
#ifndef SFB_MODAL_LEAN_K
#define SFB_MODAL_LEAN_K 1
#endif
#ifndef SFB_MODAL_CAP_CTAS
#define SFB_MODAL_CAP_CTAS 0  // experiments: cap the CTAs per SM
#endif
#ifndef SFB_MODAL_PARITY
#define SFB_MODAL_PARITY 1  // even/odd transforms when the operators have the parity
#endif
#ifndef SFB_MODAL_TABLOG
#define SFB_MODAL_TABLOG 0  // table log measured 47.6 vs 47.0 ms here
#endif
#ifndef SFB_MODAL_COMPACT
#define SFB_MODAL_COMPACT 1  // 69 KB smem (3 CTAs/SM with the lean line loop: 43.3 -> 41.5 ms)
#endif
#ifndef SFB_MODAL_EXP_SKIP
#define SFB_MODAL_EXP_SKIP 0  // experiments only (wrong results): skip stages A=1 B=2 C=4 D=8
#endif
#ifndef SFB_MODAL_L2PF
#define SFB_MODAL_L2PF 1  // L2 prefetch one element beyond the smem copy (40.8 -> 40.5 ms; 0 or 1)
#endif
#ifndef SFB_MODAL_SLOTS
#define SFB_MODAL_SLOTS 1  // input slots: 1 = one slot, the next copy issued after the element (37.0 vs 38.0 ms with 2)
#endif
#ifndef SFB_MODAL_PAIRITEMS
#define SFB_MODAL_PAIRITEMS 0  // two transform items per thread side by side: 37.0 vs 36.6 ms (spills 72 -> 144 B)
#endif
#ifndef SFB_MODAL_BATCH_N6
#define SFB_MODAL_BATCH_N6 2
#endif

namespace sfb {

template <int N>
struct ModalOps {
  double D[N * N];   // scale * D / 2 (the 1/2 of the metric average folded in)
  double V[N * N];   // Vandermonde (interpolation)
  double P[N * N];   // projection
  double Dd[N];      // scale * D[i][i] (diagonal term, full metric at the node)
};

template <int N>
struct ModalCfg {
  static constexpr int kNodes = N * N * N;
  static constexpr int kLines = N * N;
  static constexpr int kLineThreads = 3 * kLines;
  static constexpr int kThreads = ((kLineThreads + 31) / 32) * 32 < 128 ? 128
                                  : ((kLineThreads + 31) / 32) * 32;
  static constexpr int kU = 5 * kNodes;   // doubles of Uhat / u / r per element
  static constexpr int kJ = 9 * kNodes;   // doubles of Ja per element
  static constexpr int kSlot = kU + kJ;   // one input slot
  static constexpr int kRec = 7 * kNodes; // node records: 7 planes
  // residual (+ 2 direction buffers unless SFB_MODAL_COMPACT reuses the
  // record planes and the residual itself for them)
  static constexpr size_t kSmem =
      (size_t)(SFB_MODAL_SLOTS * kSlot + kRec + (SFB_MODAL_COMPACT ? 1 : 3) * kU) * sizeof(double);
  static constexpr int kMinBlocks = (N == 6) ? SFB_MODAL_MINBLOCKS_N6 : 1;
};

// y = A x along one line, dense or exploiting the parity of the Legendre /
// GLL operators (x_{n-1-i} = -x_i, P_k(-x) = (-1)^k P_k(x)):
//   MODE 1, V (modal -> nodal): V[n-1-i][k] = (-1)^k V[i][k], so with the even
//     and odd modal sums e_i, o_i over the first n/2 nodes y_i = e_i + o_i and
//     y_{n-1-i} = e_i - o_i (n/2 rows of n FMAs instead of n rows);
//   MODE 2, Pi = V^-1 (nodal -> modal): Pi[k][n-1-i] = (-1)^k Pi[k][i], so the
//     nodal sums s_i = x_i + x_{n-1-i} feed the even modes and the differences
//     t_i = x_i - x_{n-1-i} the odd ones (n rows of n/2 FMAs).
// At n = 6: 18 FMAs + 6 adds per line instead of 36 FMAs.  The host takes the
// symmetric path only when the given operators have the parity to 1e-13
// (they do when built by the reference's constructors, operators.py:96-232).
template <int N, int MODE>
__device__ __forceinline__ void apply_line(const double (&A)[N * N], const double (&x)[N],
                                           double (&y)[N]) {
  constexpr int H = N / 2;
  if constexpr (MODE == 1) {
#pragma unroll
    for (int i = 0; i < H; ++i) {
      double e = 0.0, o = 0.0;
#pragma unroll
      for (int k = 0; k < N; k += 2) e = fma(A[i * N + k], x[k], e);
#pragma unroll
      for (int k = 1; k < N; k += 2) o = fma(A[i * N + k], x[k], o);
      y[i] = e + o;
      y[N - 1 - i] = e - o;
    }
    if constexpr (N % 2 == 1) {
      double e = 0.0;
#pragma unroll
      for (int k = 0; k < N; k += 2) e = fma(A[H * N + k], x[k], e);
      y[H] = e;
    }
  } else if constexpr (MODE == 2) {
    double sm[H > 0 ? H : 1], df[H > 0 ? H : 1];
#pragma unroll
    for (int i = 0; i < H; ++i) {
      sm[i] = x[i] + x[N - 1 - i];
      df[i] = x[i] - x[N - 1 - i];
    }
#pragma unroll
    for (int k = 0; k < N; ++k) {
      double acc = 0.0;
#pragma unroll
      for (int i = 0; i < H; ++i) acc = fma(A[k * N + i], (k % 2 == 0) ? sm[i] : df[i], acc);
      if constexpr (N % 2 == 1) {
        if (k % 2 == 0) acc = fma(A[k * N + H], x[H], acc);
      }
      y[k] = acc;
    }
  } else {
#pragma unroll
    for (int a = 0; a < N; ++a) {
      double acc = 0.0;
#pragma unroll
      for (int c = 0; c < N; ++c) acc = fma(A[a * N + c], x[c], acc);
      y[a] = acc;
    }
  }
}

// One sum-factorised pass along direction j: out[.., a_j, ..] = (A x)_a over
// each line, the input being the sum of NIN buffers ((a + b) + c) + d at each
// node (NIN = 1: a plain pass; 3/4: diagonal term + the direction residuals).
// A is a reference into the __grid_constant__ parameter block, so with the
// loops unrolled every coefficient is a constant-bank operand of its DFMA (no
// shared-memory load per multiply: 56 -> 52.5 ms at config 5).  One work item
// per (variable, line); each line is read completely before it is written and
// lines are disjoint, so out may alias an input.  (Splitting a line's outputs
// over two items to fill the CTA more evenly measured slower: 58.8 ms.)
template <int N, int MODE, int NIN = 1, int J = 0>
__device__ __forceinline__ void kron_pass(const double (&A)[N * N], const double* in0,
                                          double* out, int tid, int nthreads,
                                          const double* in1 = nullptr,
                                          const double* in2 = nullptr,
                                          const double* in3 = nullptr) {
  constexpr int NN = N * N * N;
  constexpr int NI = 5 * N * N;  // (variable, line) items
  constexpr int stride = J == 0 ? 1 : (J == 1 ? N : N * N);
  // x0 lines are contiguous: 16-byte accesses (a stride-n line per lane with
  // 8-byte accesses is an n-way bank conflict pattern; 48-byte strided 16-byte
  // accesses at n = 6 cover the 32 banks once per quarter warp)
  constexpr bool kVec = (J == 0) && (N % 2 == 0);
  auto offset = [&](int t) {
    const int v = t / (N * N);
    const int L = t - v * N * N;
    const int u0 = L % N, u1 = L / N;
    int base;
    if constexpr (J == 0) base = u0 * N + u1 * N * N;
    else if constexpr (J == 1) base = u0 + u1 * N * N;
    else base = u0 + u1 * N;
    return v * NN + base;
  };
  auto load = [&](int o, double (&x)[N]) {
    if constexpr (kVec) {
#pragma unroll
      for (int c = 0; c < N; c += 2) {
        double2 q = *reinterpret_cast<const double2*>(in0 + o + c);
        if constexpr (NIN > 1) {
          const double2 q1 = *reinterpret_cast<const double2*>(in1 + o + c);
          const double2 q2 = *reinterpret_cast<const double2*>(in2 + o + c);
          q.x = (q.x + q1.x) + q2.x;
          q.y = (q.y + q1.y) + q2.y;
          if constexpr (NIN == 4) {
            const double2 q3 = *reinterpret_cast<const double2*>(in3 + o + c);
            q.x = q.x + q3.x;
            q.y = q.y + q3.y;
          }
        }
        x[c] = q.x;
        x[c + 1] = q.y;
      }
    } else {
#pragma unroll
      for (int c = 0; c < N; ++c) {
        const int k = o + c * stride;
        if constexpr (NIN == 1) {
          x[c] = in0[k];
        } else {
          x[c] = (in0[k] + in1[k]) + in2[k];
          if constexpr (NIN == 4) x[c] = x[c] + in3[k];
        }
      }
    }
  };
  auto store = [&](int o, const double (&y)[N]) {
    if constexpr (kVec) {
#pragma unroll
      for (int a = 0; a < N; a += 2)
        *reinterpret_cast<double2*>(out + o + a) = make_double2(y[a], y[a + 1]);
    } else {
#pragma unroll
      for (int a = 0; a < N; ++a) out[o + a * stride] = y[a];
    }
  };
  if (SFB_MODAL_PAIRITEMS) {
    // items t and t + nthreads side by side (two independent lines per thread:
    // ILP for the threads that have two; each line is read completely before
    // any line is written, and lines are disjoint, so out may alias an input)
    for (int t = tid; t < NI; t += 2 * nthreads) {
      const int t1 = t + nthreads;
      const bool two = t1 < NI;
      const int o0 = offset(t), o1 = offset(two ? t1 : t);
      double x0[N], x1[N], y0[N], y1[N];
      load(o0, x0);
      load(o1, x1);
      apply_line<N, MODE>(A, x0, y0);
      apply_line<N, MODE>(A, x1, y1);
      store(o0, y0);
      if (two) store(o1, y1);
    }
  } else {
    for (int t = tid; t < NI; t += nthreads) {
      const int o = offset(t);
      double x[N], y[N];
      load(o, x);
      apply_line<N, MODE>(A, x, y);
      store(o, y);
    }
  }
}

// The last pass (x2 lines) of Pi^3 with its lines written straight to HBM
// (evict-first; at a given node offset the lanes of a warp cover consecutive
// lines, so every store instruction is coalesced) and the squares of the
// written values summed per thread in item order: no shared round trip and
// no barrier between the last pass and the store.
template <int N, int MODE>
__device__ __forceinline__ double kron_pass_out(const double (&A)[N * N], const double* in,
                                                double* __restrict__ gout, int tid,
                                                int nthreads) {
  constexpr int NN = N * N * N;
  double ss = 0.0;
  for (int t = tid; t < 5 * N * N; t += nthreads) {
    const int v = t / (N * N);
    const int L = t - v * N * N;
    const int o = v * NN + L;  // x2 line (u0, u1): base u0 + u1 N = L, stride N^2
    double x[N], y[N];
#pragma unroll
    for (int c = 0; c < N; ++c) x[c] = in[o + c * N * N];
    apply_line<N, MODE>(A, x, y);
#pragma unroll
    for (int a = 0; a < N; ++a) {
      __stcs(gout + o + a * N * N, y[a]);
      ss = fma(y[a], y[a], ss);
    }
  }
  return ss;
}

// Contravariant Chandrashekar flux for K pairs at once (normals n = Ja_a + Ja_b,
// the 1/2 being folded into D).  Records carry hb = (gamma-1) beta (see
// chandrashekar_cart_v2 in euler_flux.cuh): the beta log mean's reciprocal is
// then c_gamma / beta_ln directly and p_hat = gm1 rhobar / sb.
template <int K>
__device__ __forceinline__ void chandrashekar_curv_k(const NodeRec (&A)[K],
                                                     const NodeRec (&B)[K],
                                                     const double (&nx)[K], const double (&ny)[K],
                                                     const double (&nz)[K], double gm1,
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
    const double sr = A[k].hr + B[k].hr;
    const double sb = A[k].hb + B[k].hb;
    const double p1 = dr[k] * nb[k];
    const double rr = rcp_refined(p1 * sb);
    const double inv_sb = rr * p1;
    const double t = rr * sb;
    const double rho_ln = nr[k] * (t * nb[k]);
    const double cibeta = db[k] * (t * dr[k]);  // c_gamma / beta_ln
    const double phat = (gm1 * sr) * inv_sb;
    const double vn = fma(vb2[k], nz[k], fma(vb1[k], ny[k], vb0[k] * nx[k]));
    const double f1 = rho_ln * vn;
    f[k][0] = f1;
    f[k][1] = fma(f1, vb0[k], phat * nx[k]);
    f[k][2] = fma(f1, vb1[k], phat * ny[k]);
    f[k][3] = fma(f1, vb2[k], phat * nz[k]);
    const double dot = fma(A[k].hv2, B[k].hv2, fma(A[k].hv1, B[k].hv1, A[k].hv0 * B[k].hv0));
    f[k][4] = fma(f1, fma(2.0, dot, cibeta), phat * vn);
  }
}

// Register-lean pair loop for one line (SFB_MODAL_LEAN): node a is loaded once
// per outer step, the nodes b > a are reloaded for each pair with volatile
// shared loads (so the compiler cannot keep all n records of the line live),
// which keeps the line stage under ~170 registers for 3 CTAs per SM.
__device__ __forceinline__ double vlds(const double* p) {
  double x;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(x) : "r"(smem_u32(p)));
  return x;
}
template <int NN>
__device__ __forceinline__ void vload_node(const double* rec, const double* jd, int k, NodeRec& q,
                                           double& jx, double& jy, double& jz) {
  q.hr = vlds(rec + k);
  q.hv0 = vlds(rec + NN + k);
  q.hv1 = vlds(rec + 2 * NN + k);
  q.hv2 = vlds(rec + 3 * NN + k);
  q.hb = vlds(rec + 4 * NN + k);
  q.hlr = vlds(rec + 5 * NN + k);
  q.hlb = vlds(rec + 6 * NN + k);
  jx = vlds(jd + k);
  jy = vlds(jd + NN + k);
  jz = vlds(jd + 2 * NN + k);
}
template <int N, int KB>
__device__ __forceinline__ void lean_batch(const double* rec, const double* jd, int base, int stride,
                                           int a, int b0, const NodeRec& qa, double ax, double ay,
                                           double az, const double (&Dm)[N * N], double gm1,
                                           double (&acc)[N][5]) {
  constexpr int NN = N * N * N;
  NodeRec A[KB], B[KB];
  double nx[KB], ny[KB], nz[KB];
#pragma unroll
  for (int k = 0; k < KB; ++k) {
    double bx, by, bz;
    vload_node<NN>(rec, jd, base + (b0 + k) * stride, B[k], bx, by, bz);
    A[k] = qa;
    nx[k] = ax + bx;
    ny[k] = ay + by;
    nz[k] = az + bz;
  }
  double f[KB][5];
  chandrashekar_curv_k<KB>(A, B, nx, ny, nz, gm1, f);
#pragma unroll
  for (int k = 0; k < KB; ++k) {
    const int b = b0 + k;
    const double dab = Dm[a * N + b], dba = Dm[b * N + a];
#pragma unroll
    for (int v = 0; v < 5; ++v) {
      acc[a][v] = fma(dab, f[k][v], acc[a][v]);
      acc[b][v] = fma(dba, f[k][v], acc[b][v]);
    }
  }
}

template <int N>
struct ModalPairs {
  static constexpr int kPairs = N * (N - 1) / 2;
  int a[kPairs > 0 ? kPairs : 1], b[kPairs > 0 ? kPairs : 1];
  constexpr ModalPairs() : a{}, b{} {
    const int M = (N % 2 == 0) ? N : N + 1;
    int k = 0;
    for (int round = 0; round < M - 1; ++round) {
      for (int i = 0; i < M / 2; ++i) {
        int x = (i == 0) ? M - 1 : (round + i) % (M - 1);
        int y = (i == 0) ? round : (round - i + (M - 1)) % (M - 1);
        if (x >= N || y >= N) continue;
        a[k] = x < y ? x : y;
        b[k] = x < y ? y : x;
        ++k;
      }
    }
  }
};

template <int N>
constexpr int kModalBatch = (N >= 7) ? 1 : (N == 6 ? SFB_MODAL_BATCH_N6 : (N >= 4 ? 2 : 1));

template <int N, bool EO>
__global__ void __launch_bounds__(ModalCfg<N>::kThreads, ModalCfg<N>::kMinBlocks)
    euler_modal_kernel(int64_t E, const __grid_constant__ ModalOps<N> ops, double gm1, double c_gamma,
                       double gam_ratio, const double* __restrict__ Uhat,
                       const double* __restrict__ Ja, double* __restrict__ Rhat,
                       double* __restrict__ sumsq, unsigned long long* claim_ctr) {
  using Cfg = ModalCfg<N>;
  constexpr int NN = Cfg::kNodes;
  constexpr int T = Cfg::kThreads;
  extern __shared__ __align__(16) double smem[];
  // smem: 2 input slots [Uhat | Ja], node records, residual.  The slot's Uhat
  // region doubles as the transform ping-pong buffer: V^3 runs slot -> res ->
  // slot -> res (u ends in res), Pi^3 runs res -> slot -> res -> slot.
  double* slots = smem;                    // [2][Uhat | Ja]
  double* rec = smem + SFB_MODAL_SLOTS * Cfg::kSlot;  // [7][NN] node records (natural layout)
  double* res = rec + Cfg::kRec;           // [5][NN] u, then the nodal residual r
  // x1-line residuals: the record planes once every line has read them
  // (compact), else a buffer of their own; x2-line residuals: added into the
  // residual in place (compact; each node is on exactly one x2 line), else a
  // buffer of their own
  double* dbuf1 = SFB_MODAL_COMPACT ? rec : res + Cfg::kU;
  double* dbuf2 = SFB_MODAL_COMPACT ? nullptr : res + 2 * Cfg::kU;
  __shared__ double wsum[T / 32];
  __shared__ uint64_t full[2];
  const int tid = threadIdx.x;
  const double hgm1 = 0.5 * gm1;
  if (tid == 0) {
    mbar_init(&full[0], 1);
    mbar_init(&full[1], 1);
    fence_mbar_init();
  }
  __syncthreads();
  // operators straight from the __grid_constant__ parameter block (constant bank)
  const double(&sV)[N * N] = ops.V;
  const double(&sP)[N * N] = ops.P;

  constexpr uint32_t kUB = (uint32_t)(Cfg::kU * 8), kJB = (uint32_t)(Cfg::kJ * 8);
  constexpr bool kBulk = (kUB % 16) == 0 && (kJB % 16) == 0;
  auto issue = [&](int64_t e, int slot) {
    double* dst = slots + slot * Cfg::kSlot;
    mbar_arrive_expect_tx(&full[slot], kUB + kJB);
    bulk_g2s(dst, Uhat + e * Cfg::kU, kUB, &full[slot]);
    bulk_g2s(dst + Cfg::kU, Ja + e * Cfg::kJ, kJB, &full[slot]);
  };
  auto l2_prefetch = [&](int64_t e) {  // bytes multiple of 16 (kBulk)
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(Uhat + e * Cfg::kU), "r"(kUB)
                 : "memory");
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(Ja + e * Cfg::kJ), "r"(kJB)
                 : "memory");
  };
  // Element order: e_0 = blockIdx.x; with a claim counter (dynamic) every
  // further element is claimed from it, one element ahead (the bulk copy of
  // the next element and the L2 prefetch of the one after need them early),
  // so a CTA on a slower SM simply takes fewer elements; without one
  // (static) the CTA takes e_0 + k gridDim.x.
  __shared__ long long s_next[2];
  const bool dyn = claim_ctr != nullptr;
  auto claim = [&](int k) -> int64_t {  // k-th element of this CTA, k >= 1
    return dyn ? (int64_t)gridDim.x + (int64_t)atomicAdd(claim_ctr, 1ull)
               : (int64_t)blockIdx.x + (int64_t)k * gridDim.x;
  };
  if (tid == 0 && (int64_t)blockIdx.x < E) {
    if (kBulk) issue(blockIdx.x, 0);
    const int64_t e1 = claim(1);
    s_next[0] = e1;
    if (kBulk && SFB_MODAL_L2PF > 0 && e1 < E) l2_prefetch(e1);
  }
  __syncthreads();
  uint32_t parity[2] = {0, 0};

  int it = 0;
  // s_next[it & 1] = the element after iteration it's: written by thread 0 at
  // the top of iteration it - 1 (the prologue for it = 0), read by every
  // thread just before iteration it's final barrier, rewritten (for it + 2)
  // only after that barrier
  for (int64_t e = blockIdx.x; e < E; ++it) {
    if (tid == 0 && s_next[it & 1] < E) {
      const int64_t nn = claim(it + 2);
      s_next[(it + 1) & 1] = nn;
      if (kBulk && SFB_MODAL_L2PF > 0 && nn < E) l2_prefetch(nn);
    }
    const int slot = SFB_MODAL_SLOTS == 2 ? (it & 1) : 0;
    double* in = slots + slot * Cfg::kSlot;
    const double* jin = in + Cfg::kU;
    if (kBulk) {
      mbar_wait_parity(&full[slot], parity[slot]);
      parity[slot] ^= 1;
      const int64_t nxt = tid == 0 ? s_next[it & 1] : E;
      if (SFB_MODAL_SLOTS == 2 && tid == 0 && nxt < E) {
        fence_proxy_async_smem();
        issue(nxt, slot ^ 1);
      }
    } else {
      for (int i = tid; i < Cfg::kU; i += T) in[i] = __ldcs(Uhat + e * Cfg::kU + i);
      for (int i = tid; i < Cfg::kJ; i += T) in[Cfg::kU + i] = __ldcs(Ja + e * Cfg::kJ + i);
      __syncthreads();
    }

    // ---- stage A: u = V^3 Uhat ------------------------------------------------
    constexpr int MV = EO ? 1 : 0, MP = EO ? 2 : 0;
    if (!(SFB_MODAL_EXP_SKIP & 1)) {
    kron_pass<N, MV, 1, 0>(sV, in, res, tid, T);
    __syncthreads();
    kron_pass<N, MV, 1, 1>(sV, res, in, tid, T);
    __syncthreads();
    kron_pass<N, MV, 1, 2>(sV, in, res, tid, T);  // u in res
    __syncthreads();
    }

    // ---- stage B: node records + diagonal term ----------------------------------
    for (int r = tid; r < ((SFB_MODAL_EXP_SKIP & 2) ? 0 : NN); r += T) {
      const double* u = res + r;  // read this node's u, then overwrite it with its diagonal term
      const double rho = u[0], m0 = u[NN], m1 = u[2 * NN], m2 = u[3 * NN], et = u[4 * NN];
      const double irho = rcp_refined(rho);
      const double hirho = 0.5 * irho;
      const double mm = fma(m2, m2, fma(m1, m1, m0 * m0));
      const double X2 = fma(rho, et + et, -mm);  // 2 (rho E - |m|^2/2)
      const double iX2 = rcp_refined(X2);
      const double p = (hgm1 * X2) * irho;
      const double hbeta = (rho * rho) * iX2;  // (gamma - 1) beta
      rec[r] = 0.5 * rho;
      rec[NN + r] = m0 * hirho;
      rec[2 * NN + r] = m1 * hirho;
      rec[3 * NN + r] = m2 * hirho;
      rec[4 * NN + r] = hbeta;
      rec[5 * NN + r] = SFB_MODAL_TABLOG ? log_half_tab(rho) : log_half(rho);
      rec[6 * NN + r] = SFB_MODAL_TABLOG ? log_half_tab(hbeta) : log_half(hbeta);
      // n_diag = sum_i D[r_i,r_i] Ja^i(r); diagonal term f(u).n_diag with
      // mass = m.n_diag, w = mass / rho:  (mass, w m + p n_diag, (E + p) w)
      const int c0 = r % N, c1 = (r / N) % N, c2 = r / (N * N);
      const double d0 = ops.Dd[c0], d1 = ops.Dd[c1], d2 = ops.Dd[c2];
      double nd[3];
#pragma unroll
      for (int m = 0; m < 3; ++m)
        nd[m] = fma(d2, jin[(2 * 3 + m) * NN + r],
                    fma(d1, jin[(1 * 3 + m) * NN + r], d0 * jin[(0 * 3 + m) * NN + r]));
      const double mass = fma(m2, nd[2], fma(m1, nd[1], m0 * nd[0]));
      const double wv = mass * irho;
      res[r] = mass;
      res[NN + r] = fma(m0, wv, p * nd[0]);
      res[2 * NN + r] = fma(m1, wv, p * nd[1]);
      res[3 * NN + r] = fma(m2, wv, p * nd[2]);
      res[4 * NN + r] = (et + p) * wv;
    }
    __syncthreads();

    // ---- stage C: line threads --------------------------------------------------
    {
      const int dir = tid / Cfg::kLines;
      const int L = tid - dir * Cfg::kLines;
      const bool active = tid < Cfg::kLineThreads;
      const int u0 = L % N, u1 = L / N;
      int base, stride;
      if (dir == 0) { base = u0 * N + u1 * N * N; stride = 1; }
      else if (dir == 1) { base = u0 + u1 * N * N; stride = N; }
      else { base = u0 + u1 * N; stride = N * N; }
      double acc[N][5];
#pragma unroll
      for (int a = 0; a < N; ++a)
#pragma unroll
        for (int v = 0; v < 5; ++v) acc[a][v] = 0.0;
      if ((SFB_MODAL_EXP_SKIP & 4)) {
      } else if (SFB_MODAL_LEAN && active) {
        const double* jd = jin + (dir * 3) * NN;  // Ja^dir_m planes
#pragma unroll
        for (int a = 0; a < N - 1; ++a) {
          NodeRec qa;
          double ax, ay, az;
          vload_node<NN>(rec, jd, base + a * stride, qa, ax, ay, az);
#pragma unroll
          for (int b0 = a + 1; b0 < N; b0 += SFB_MODAL_LEAN_K) {
            if (SFB_MODAL_LEAN_K == 2 && b0 + 1 < N)
              lean_batch<N, 2>(rec, jd, base, stride, a, b0, qa, ax, ay, az, ops.D, gm1, acc);
            else
              lean_batch<N, 1>(rec, jd, base, stride, a, b0, qa, ax, ay, az, ops.D, gm1, acc);
          }
        }
      } else if (active) {
        constexpr ModalPairs<N> po;
        constexpr int P = ModalPairs<N>::kPairs;
        constexpr int K = kModalBatch<N>;
        const double* jd = jin + (dir * 3) * NN;  // Ja^dir_m planes
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
          chandrashekar_curv_k<K>(A, B, nx, ny, nz, gm1, f);
#pragma unroll
          for (int k = 0; k < K; ++k) {
            if (k0 + k >= P) break;
            const int a = po.a[k0 + k], b = po.b[k0 + k];
            const double dab = ops.D[a * N + b], dba = ops.D[b * N + a];
#pragma unroll
            for (int v = 0; v < 5; ++v) {
              acc[a][v] = fma(dab, f[k][v], acc[a][v]);
              acc[b][v] = fma(dba, f[k][v], acc[b][v]);
            }
          }
        }
      }
      if (SFB_MODAL_COMPACT) __syncthreads();  // all lines have read the records
      if (active) {  // every node is on exactly one line per direction: plain stores
        if (SFB_MODAL_COMPACT && dir == 2) {
#pragma unroll
          for (int a = 0; a < N; ++a)
#pragma unroll
            for (int v = 0; v < 5; ++v) res[v * NN + base + a * stride] += acc[a][v];
        } else {
          double* db = dir == 0 ? in : (dir == 1 ? dbuf1 : dbuf2);
#pragma unroll
          for (int a = 0; a < N; ++a)
#pragma unroll
            for (int v = 0; v < 5; ++v) db[v * NN + base + a * stride] = acc[a][v];
        }
      }
      __syncthreads();
    }

    // ---- stage D: Rhat = Pi^3 r, store, sum of squares -------------------------
    if (!(SFB_MODAL_EXP_SKIP & 8)) {
    if (SFB_MODAL_COMPACT)  // r = (diag + x2) + x0 + x1
      kron_pass<N, MP, 3, 0>(sP, res, res, tid, T, in, dbuf1);
    else  // r = diag + x0 + x1 + x2
      kron_pass<N, MP, 4, 0>(sP, res, res, tid, T, in, dbuf1, dbuf2);
    __syncthreads();
    kron_pass<N, MP, 1, 1>(sP, res, in, tid, T);
    __syncthreads();
    }
    double* Rg = Rhat + e * Cfg::kU;
    double ss = 0.0;
    if (!(SFB_MODAL_EXP_SKIP & 8)) {
      ss = kron_pass_out<N, MP>(sP, in, Rg, tid, T);  // last pass straight to HBM
    } else {
      for (int i = tid; i < Cfg::kU; i += T) __stcs(Rg + i, res[i]);
    }
    const int64_t e_next = s_next[it & 1];
    if (sumsq) {  // fixed order: xor-butterfly in each warp, then the warps in order
#pragma unroll
      for (int o = 16; o >= 1; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
      if ((tid & 31) == 0) wsum[tid >> 5] = ss;
      __syncthreads();  // also the end of this element's shared-memory use
      if (tid == 0) {
        double t = wsum[0];
#pragma unroll
        for (int w = 1; w < T / 32; ++w) t += wsum[w];
        sumsq[e] = t;
      }
    } else {
      __syncthreads();
    }
    if (SFB_MODAL_SLOTS == 1 && kBulk && tid == 0 && e_next < E) {
      fence_proxy_async_smem();  // the slot's last generic reads were before the barrier
      issue(e_next, 0);
    }
    e = e_next;
  }
}

template <int N>
static int launch_modal(int64_t E, const double* V, const double* Pi, const double* D,
                        double gamma, double scale, const double* Uhat, const double* Ja,
                        double* Rhat, double* sumsq, void* workspace, cudaStream_t s) {
  using Cfg = ModalCfg<N>;
  ModalOps<N> ops;
  for (int i = 0; i < N * N; ++i) {
    ops.D[i] = 0.5 * scale * D[i];
    ops.V[i] = V[i];
    ops.P[i] = Pi[i];
  }
  for (int i = 0; i < N; ++i) ops.Dd[i] = scale * D[i * N + i];
  // the parity of the operators (Legendre modes on symmetric GLL nodes)
  double vmax = 0.0, pmax = 0.0;
  for (int i = 0; i < N * N; ++i) {
    vmax = fmax(vmax, fabs(V[i]));
    pmax = fmax(pmax, fabs(Pi[i]));
  }
  bool eo = SFB_MODAL_PARITY != 0;
  for (int i = 0; i < N && eo; ++i)
    for (int k = 0; k < N; ++k) {
      const double sg = (k % 2 == 0) ? 1.0 : -1.0;
      if (fabs(V[(N - 1 - i) * N + k] - sg * V[i * N + k]) > 1e-13 * vmax ||
          fabs(Pi[k * N + (N - 1 - i)] - sg * Pi[k * N + i]) > 1e-13 * pmax)
        eo = false;
    }
  auto kern = eo ? euler_modal_kernel<N, true> : euler_modal_kernel<N, false>;
  static DeviceCache cache[2];  // parity / dense kernel
  int ps = resident_ctas(kern, Cfg::kThreads, Cfg::kSmem, cache[eo ? 1 : 0]);
  if (SFB_MODAL_CAP_CTAS > 0 && ps > SFB_MODAL_CAP_CTAS) ps = SFB_MODAL_CAP_CTAS;
  int64_t grid = (int64_t)num_sms() * ps;
  if (grid > E) grid = E;
  const double gm1 = gamma - 1.0;
  unsigned long long* ctr = static_cast<unsigned long long*>(workspace);
  if (ctr && cudaMemsetAsync(ctr, 0, sizeof(unsigned long long), s) != cudaSuccess)
    return fail(SFB_ECUDA, "claim counter reset failed");
  kern<<<(unsigned)grid, Cfg::kThreads, Cfg::kSmem, s>>>(E, ops, gm1, 1.0 / (2.0 * gm1),
                                                         gamma / gm1, Uhat, Ja, Rhat, sumsq, ctr);
  return check_launch("euler_volume_curvilinear_modal");
}


}  // namespace sfb


using namespace sfb;

// V, Pi, D are HOST pointers (n x n operators folded into the parameter block).
extern "C" int sfb_euler_volume_curvilinear_modal(int64_t E, int64_t n, const double* V,
                                                  const double* Pi, const double* D, double gamma,
                                                  double scale, const double* Uhat,
                                                  const double* Ja, double* Rhat, double* sumsq,
                                                  void* workspace, sfb_stream_t stream) {
  SFB_CHECK_ARG(E >= 0, "negative element count");
  SFB_CHECK_ARG(V && Pi && D, "null operator (host n x n arrays)");
  SFB_CHECK_ARG(gamma > 1.0, "gamma must exceed 1");
  if (E == 0) return SFB_OK;
  SFB_CHECK_ARG(Uhat && Ja && Rhat, "null state / metric / output pointer");
  SFB_CHECK_ARG(((uintptr_t)Uhat | (uintptr_t)Ja | (uintptr_t)Rhat) % 16 == 0,
                "Uhat, Ja, Rhat must be 16-byte aligned");
  SFB_CHECK_ARG((uintptr_t)workspace % 8 == 0, "workspace must be 8-byte aligned");
  cudaStream_t s = (cudaStream_t)stream;
  switch (n) {
    case 2: return launch_modal<2>(E, V, Pi, D, gamma, scale, Uhat, Ja, Rhat, sumsq, workspace, s);
    case 3: return launch_modal<3>(E, V, Pi, D, gamma, scale, Uhat, Ja, Rhat, sumsq, workspace, s);
    case 4:
      return launch_modal<4>(E, V, Pi, D, gamma, scale, Uhat, Ja, Rhat, sumsq, workspace, s);
    case 5: return launch_modal<5>(E, V, Pi, D, gamma, scale, Uhat, Ja, Rhat, sumsq, workspace, s);
    case 6:
      return launch_modal<6>(E, V, Pi, D, gamma, scale, Uhat, Ja, Rhat, sumsq, workspace, s);
    case 7: return launch_modal<7>(E, V, Pi, D, gamma, scale, Uhat, Ja, Rhat, sumsq, workspace, s);
    case 8: return launch_modal<8>(E, V, Pi, D, gamma, scale, Uhat, Ja, Rhat, sumsq, workspace, s);
    default: return fail(SFB_ENOTSUP, "euler_volume_curvilinear_modal: n must be in 2..8");
  }
}
