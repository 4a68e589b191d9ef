// Pieces shared by the Cartesian Euler kernels (euler.cu, euler_fused.cu, euler_warp.cu).
#pragma once

#include "bulk.cuh"
#include "common.cuh"
#include "euler_flux.cuh"

namespace sfb {

template <int N>
struct DMat {
  double d[N * N];  // scale * D, row-major
};

template <int N>
__device__ __forceinline__ int swz(int r0, int r1, int r2) {
  int a = r0 + r2;
  a = a >= N ? a - N : a;
  int b = r1 + r2;
  b = b >= N ? b - N : b;
  return r2 * N * N + a + N * b;
}


// Cartesian Chandrashekar flux for K independent pairs at once, in the
// direction-rotated frame: the callers load the velocity components permuted
// so that hv0 is the component along the line's direction (and write the
// momentum results back un-permuted by address), so the flux itself never
// branches or selects on the direction.  Every statement is written across the K pairs so
// the instruction stream carries K independent dependency chains: the FP64
// pipe needs ~4 independent DFMAs in flight per warp to approach its peak
// (DFMA latency ~9 cycles; tools/peaks/fp64_latency.cu), which warps alone
// cannot supply.  The direction only selects operands (ALU selects).
template <int K>
__device__ __forceinline__ void chandrashekar_cart_k(const NodeRec* const (&A)[K],
                                                     const NodeRec* const (&B)[K],
                                                     double c_gamma, double (&f)[K][5]) {
  double vb0[K], vb1[K], vb2[K], nr[K], dr[K], nb[K], db[K];
#pragma unroll
  for (int k = 0; k < K; ++k) {
    vb0[k] = A[k]->hv0 + B[k]->hv0;
    vb1[k] = A[k]->hv1 + B[k]->hv1;
    vb2[k] = A[k]->hv2 + B[k]->hv2;
  }
#pragma unroll
  for (int k = 0; k < K; ++k) {
    logmean_parts(A[k]->hr, B[k]->hr, A[k]->hlr, B[k]->hlr, nr[k], dr[k]);  // rho_ln
    logmean_parts(A[k]->hb, B[k]->hb, A[k]->hlb, B[k]->hlb, nb[k], db[k]);  // beta_ln
  }
  double sr[K], sb[K], p1[K], rr[K];
#pragma unroll
  for (int k = 0; k < K; ++k) {
    sr[k] = __dadd_rn(A[k]->hr, B[k]->hr);  // rhobar (same op as the log mean's s: CSE)
    sb[k] = __dadd_rn(A[k]->hb, B[k]->hb);  // betabar
    p1[k] = dr[k] * nb[k];
    rr[k] = rcp_refined(p1[k] * sb[k]);
  }
#pragma unroll
  for (int k = 0; k < K; ++k) {
    const double inv_sb = rr[k] * p1[k];
    const double t = rr[k] * sb[k];
    const double rho_ln = nr[k] * (t * nb[k]);
    const double ibeta = db[k] * (t * dr[k]);
    const double phat = 0.5 * sr[k] * inv_sb;
    const double vn = vb0[k];  // rotated frame: component 0 is normal to the face
    const double f1 = rho_ln * vn;
    f[k][0] = f1;
    f[k][1] = fma(f1, vb0[k], phat);
    f[k][2] = f1 * vb1[k];
    f[k][3] = f1 * vb2[k];
    // |vbar|^2 - (|v_a|^2 + |v_b|^2)/4 = 2 (v_a/2).(v_b/2): no cancellation, no q plane
    const double dot = fma(A[k]->hv2, B[k]->hv2, fma(A[k]->hv1, B[k]->hv1, A[k]->hv0 * B[k]->hv0));
    const double g = fma(2.0, dot, c_gamma * ibeta);
    f[k][4] = fma(f1, g, phat * vn);
  }
}

// Pair order of one line: the circle-method round robin, so consecutive pairs
// are disjoint (independent dependency chains and accumulators) - for N = 4:
// (0,3)(1,2) (1,3)(0,2) (2,3)(0,1).
template <int N>
struct PairOrder {
  static constexpr int kPairs = N * (N - 1) / 2;
  int a[kPairs > 0 ? kPairs : 1], b[kPairs > 0 ? kPairs : 1];
  constexpr PairOrder() : a{}, b{} {
    const int M = (N % 2 == 0) ? N : N + 1;  // odd N: dummy node M-1
    int k = 0;
    for (int round = 0; round < M - 1; ++round) {
      for (int i = 0; i < M / 2; ++i) {
        int x = (i == 0) ? M - 1 : (round + i) % (M - 1);
        int y = (round - i + (M - 1)) % (M - 1);
        if (i == 0) y = round;
        if (x >= N || y >= N) continue;
        a[k] = x < y ? x : y;
        b[k] = x < y ? y : x;
        ++k;
      }
    }
  }
};

// named barriers (id 0 is __syncthreads)
__device__ __forceinline__ void nbar_sync(int id, int count) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}
__device__ __forceinline__ void nbar_arrive(int id, int count) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(count) : "memory");
}

}  // namespace sfb
