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
// whole chain is one kernel and nothing but U and R touches HBM:
//
//   stage 0  the CTA's EPB elements (EPB*5*N^3 doubles, contiguous) are
//            streamed into shared memory with 16-byte coalesced loads;
//   stage 1  one thread per node: primitives, per-node logarithms (ln rho,
//            ln beta), the node record of euler_flux.cuh, and the diagonal
//            term sum_j D[r_j,r_j] f_j(u_r) (written as the initial residual);
//   stage 2  one thread per (element, direction, line): the line's N node
//            records in registers, each symmetric pair (a<b) evaluated ONCE
//            and scattered to both rows (D[a,b] and D[b,a]) - the
//            n(n-1)/2-per-line sum factorization of Theorem 1, halved again by
//            symmetry; warps are direction-uniform by construction;
//   stage 3  direction-ordered accumulation into the shared residual (three
//            barrier-separated phases; deterministic order, no atomics);
//   stage 4  coalesced 16-byte stores of the residual.
#include "common.cuh"
#include "euler_flux.cuh"

namespace sfb {

template <int N>
struct DMat {
  double d[N * N];  // scale * D, row-major
};

template <int N>
struct EulerCartCfg {
  static constexpr int kNodes = N * N * N;
  static constexpr int kLines = N * N;
  // elements per CTA: keep EPB*N^2 a multiple of 32 where affordable so that
  // every warp works on one direction
  static constexpr int kEPB = (N == 2) ? 16 : (N == 3) ? 8 : (N == 4) ? 4 : (N == 5) ? 2 : 1;
  static constexpr int kThreads = 3 * kLines * kEPB;
  static constexpr int kRecs = 8;
  static constexpr size_t kSmem =
      (size_t)kEPB * kNodes * (kRecs + 5) * sizeof(double);
};

template <int N>
__global__ void __launch_bounds__(EulerCartCfg<N>::kThreads)
    euler_cartesian_kernel(int64_t E, const DMat<N> Dm, double gm1, double c_gamma,
                           const double* __restrict__ U, double* __restrict__ R) {
  using Cfg = EulerCartCfg<N>;
  constexpr int NN = Cfg::kNodes;
  constexpr int EPB = Cfg::kEPB;
  constexpr int kVals = EPB * 5 * NN;
  extern __shared__ double smem[];
  double* Rs = smem;             // [EPB][5][NN]  (stages U in, R out)
  double* nd = smem + kVals;     // [8][EPB*NN]   node records, SoA

  const int tid = threadIdx.x;
  const int64_t e0 = (int64_t)blockIdx.x * EPB;
  const int nel = (E - e0) < EPB ? (int)(E - e0) : EPB;
  const int nvals = nel * 5 * NN;
  const double* Ub = U + e0 * 5 * NN;

  // ---- stage 0: stream the element block in -------------------------------
  if constexpr ((kVals % 2) == 0) {
    for (int i = 2 * tid; i < nvals; i += 2 * Cfg::kThreads) {
      double2 v = ld_stream_d2(Ub + i);
      Rs[i] = v.x;
      Rs[i + 1] = v.y;
    }
  } else {
    for (int i = tid; i < nvals; i += Cfg::kThreads) Rs[i] = __ldcs(Ub + i);
  }
  __syncthreads();

  // ---- stage 1: node records + diagonal term --------------------------------
  for (int i = tid; i < EPB * NN; i += Cfg::kThreads) {
    const int el = i / NN;
    const int r = i - el * NN;
    double* u = Rs + el * 5 * NN + r;
    const double rho = u[0], m0 = u[NN], m1 = u[2 * NN], m2 = u[3 * NN], et = u[4 * NN];
    const double irho = rcp_refined(rho);
    const double v0 = m0 * irho, v1 = m1 * irho, v2 = m2 * irho;
    const double vv = fma(v2, v2, fma(v1, v1, v0 * v0));
    const double p = gm1 * fma(-0.5 * rho, vv, et);
    const double beta = 0.5 * rho * rcp_refined(p);
    nd[0 * EPB * NN + i] = 0.5 * rho;
    nd[1 * EPB * NN + i] = 0.5 * v0;
    nd[2 * EPB * NN + i] = 0.5 * v1;
    nd[3 * EPB * NN + i] = 0.5 * v2;
    nd[4 * EPB * NN + i] = 0.5 * beta;
    nd[5 * EPB * NN + i] = 0.5 * log(rho);
    nd[6 * EPB * NN + i] = 0.5 * log(beta);
    nd[7 * EPB * NN + i] = 0.25 * vv;
    const int r0 = r % N, r1 = (r / N) % N, r2 = r / (N * N);
    const double d0 = Dm.d[r0 * N + r0], d1 = Dm.d[r1 * N + r1], d2 = Dm.d[r2 * N + r2];
    const double w = fma(d2, v2, fma(d1, v1, d0 * v0));
    u[0] = rho * w;
    u[NN] = fma(m0, w, p * d0);
    u[2 * NN] = fma(m1, w, p * d1);
    u[3 * NN] = fma(m2, w, p * d2);
    u[4 * NN] = (et + p) * w;
  }
  __syncthreads();

  // ---- stage 2: line threads -------------------------------------------------
  const int dir = tid / (EPB * Cfg::kLines);  // warp-uniform when EPB*N^2 % 32 == 0
  const int rem = tid - dir * EPB * Cfg::kLines;
  const int el = rem / Cfg::kLines;
  const int L = rem - el * Cfg::kLines;
  int base, stride;
  if (dir == 0) {
    base = L * N;
    stride = 1;
  } else if (dir == 1) {
    base = (L % N) + (L / N) * N * N;
    stride = N;
  } else {
    base = L;
    stride = N * N;
  }
  const int nb = el * NN + base;  // node index of line point 0 in nd

  double acc[N][5];
#pragma unroll
  for (int a = 0; a < N; ++a)
#pragma unroll
    for (int v = 0; v < 5; ++v) acc[a][v] = 0.0;

  auto load_rec = [&](int a) {
    NodeRec q;
    const int k = nb + a * stride;
    q.hr = nd[0 * EPB * NN + k];
    q.hv0 = nd[1 * EPB * NN + k];
    q.hv1 = nd[2 * EPB * NN + k];
    q.hv2 = nd[3 * EPB * NN + k];
    q.hb = nd[4 * EPB * NN + k];
    q.hlr = nd[5 * EPB * NN + k];
    q.hlb = nd[6 * EPB * NN + k];
    q.q = nd[7 * EPB * NN + k];
    return q;
  };
  const double n0 = dir == 0 ? 1.0 : 0.0;
  const double n1 = dir == 1 ? 1.0 : 0.0;
  const double n2 = dir == 2 ? 1.0 : 0.0;

#pragma unroll
  for (int a = 0; a < N - 1; ++a) {
    const NodeRec ra = load_rec(a);
#pragma unroll
    for (int b = a + 1; b < N; ++b) {
      const NodeRec rb = load_rec(b);
      double f[5];
      chandrashekar(ra, rb, n0, n1, n2, c_gamma, f);
      const double dab = Dm.d[a * N + b], dba = Dm.d[b * N + a];
#pragma unroll
      for (int v = 0; v < 5; ++v) {
        acc[a][v] = fma(dab, f[v], acc[a][v]);
        acc[b][v] = fma(dba, f[v], acc[b][v]);
      }
    }
  }

  // ---- stage 3: direction-ordered accumulation ------------------------------
#pragma unroll
  for (int phase = 0; phase < 3; ++phase) {
    if (dir == phase) {
#pragma unroll
      for (int a = 0; a < N; ++a) {
        double* rr = Rs + el * 5 * NN + base + a * stride;
#pragma unroll
        for (int v = 0; v < 5; ++v) rr[v * NN] += acc[a][v];
      }
    }
    __syncthreads();
  }

  // ---- stage 4: stream the residual out --------------------------------------
  double* Rb = R + e0 * 5 * NN;
  if constexpr ((kVals % 2) == 0) {
    for (int i = 2 * tid; i < nvals; i += 2 * Cfg::kThreads)
      st_stream_d2(Rb + i, make_double2(Rs[i], Rs[i + 1]));
  } else {
    for (int i = tid; i < nvals; i += Cfg::kThreads) __stcs(Rb + i, Rs[i]);
  }
}

template <int N>
static int launch_euler_cartesian(int64_t E, const double* Dh, double gamma, double scale,
                                  const double* U, double* R, cudaStream_t s) {
  using Cfg = EulerCartCfg<N>;
  DMat<N> Dm;
  for (int i = 0; i < N * N; ++i) Dm.d[i] = scale * Dh[i];
  static bool attr_done = false;
  if (!attr_done) {
    cudaFuncSetAttribute(euler_cartesian_kernel<N>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)Cfg::kSmem);
    attr_done = true;
  }
  const int64_t blocks = (E + Cfg::kEPB - 1) / Cfg::kEPB;
  if (blocks > 0x7fffffff) return fail(SFB_EINVAL, "too many elements for one launch");
  const double gm1 = gamma - 1.0;
  const double c_gamma = 1.0 / (2.0 * gm1);
  euler_cartesian_kernel<N><<<(unsigned)blocks, Cfg::kThreads, Cfg::kSmem, s>>>(E, Dm, gm1, c_gamma,
                                                                                U, R);
  return check_launch("euler_volume_cartesian");
}

int euler_cartesian_dispatch(int64_t E, int64_t n, const double* D_host, double gamma,
                             double scale, const double* U, double* R, cudaStream_t s) {
  switch (n) {
    case 2: return launch_euler_cartesian<2>(E, D_host, gamma, scale, U, R, s);
    case 3: return launch_euler_cartesian<3>(E, D_host, gamma, scale, U, R, s);
    case 4: return launch_euler_cartesian<4>(E, D_host, gamma, scale, U, R, s);
    case 5: return launch_euler_cartesian<5>(E, D_host, gamma, scale, U, R, s);
    case 6: return launch_euler_cartesian<6>(E, D_host, gamma, scale, U, R, s);
    case 7: return launch_euler_cartesian<7>(E, D_host, gamma, scale, U, R, s);
    case 8: return launch_euler_cartesian<8>(E, D_host, gamma, scale, U, R, s);
    default: return fail(SFB_ENOTSUP, "euler_volume_cartesian: n must be in 2..8");
  }
}

}  // namespace sfb

using namespace sfb;

// D is read on the host (it is folded into the kernel's parameter block); the
// Python layer passes the host-built operator exactly as the reference builds
// it (operators.py:136-152).  Here D must be a HOST pointer.
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
  return euler_cartesian_dispatch(E, n, D, gamma, scale, U, R, (cudaStream_t)stream);
}
