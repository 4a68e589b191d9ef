// Chandrashekar entropy-conservative two-point flux for the 3-D compressible
// Euler equations, in the node-record form used by the sm_100a kernels.
//
// Definition (oracle/euler_oracle.py:chandrashekar_flux is
// the CPU restatement it must match to 1e-12):
//   rho_ln = L(rho_a, rho_b),  beta = rho / (2 p),  beta_ln = L(beta_a, beta_b)
//   vbar = (v_a + v_b)/2,  p_hat = rhobar / (2 betabar)
//   F1 = rho_ln vbar.n ;  F_{1+m} = F1 vbar_m + p_hat n_m
//   F5 = F1 (1/(2(gamma-1) beta_ln) - (|v_a|^2 + |v_b|^2)/4) + sum_m vbar_m F_{1+m}
// with L the logarithmic mean:
//   d = y - x, s = x + y, u = d^2/s^2;
//   if hi(d^2) - hi(s^2) < -(hi(1) - hi(1e-5)):  L = s / (2 + u(2/3 + ...))
//   else:                                        L = d / (ln y - ln x)
// The branch test is the same integer comparison of IEEE high words as the
// oracle's (oracle/euler_oracle.py:series_branch), so both take the same
// branch.  The kernels work on rescaled quantities (x/2, or (gamma-1) beta),
// use per-node logarithms and fold the three per-pair reciprocals
// (1/L_rho, L_beta, 1/(2 betabar)) into one refined reciprocal; these change
// rounding only (few ulps).
#pragma once

#include "common.cuh"
#include "log_table.cuh"

namespace sfb {


// Per-node record, all entries pre-scaled so that pair sums are exact means.
struct NodeRec {
  double hr;             // rho / 2
  double hv0, hv1, hv2;  // v / 2
  double hb;             // (gamma-1) beta (see chandrashekar_cart_v2)
  double hlr;            // ln(rho) / 2
  double hlb;            // ln(hb) / 2 (only differences of the logs are used)
};

// Coefficients of ln(m)/2 = atanh(f) = f + f^3 (1/3 + f^2/5 + ...), f = (m-1)/(m+1),
// plus ln2/2 split hi/lo (log_half returns ln(x)/2).
__constant__ double kLogPolyHalf[11] = {
    1.0 / 3.0,  1.0 / 5.0,  1.0 / 7.0,  1.0 / 9.0,  1.0 / 11.0, 1.0 / 13.0,
    1.0 / 15.0, 1.0 / 17.0, 1.0 / 19.0, 3.46573590184561908245e-01, 9.54107464635293850010e-11};

// Half natural log ln(x)/2 (the node records store halved logs) for positive
// normal x: x = 2^e m, m in [sqrt(1/2), sqrt(2)), ln m = 2 atanh(f),
// f = (m-1)/(m+1), |f| <= 0.1716, series to f^19 (truncation < 2.5e-17
// relative), Estrin-evaluated; the 1/2 is folded into the constants.  About
// 18 FP64 operations, within ~2 ulp.  Branch-free: the validity test is an
// integer range check on the high word (no FP64 compare); non-positive /
// non-finite / subnormal inputs - non-physical states - return NaN.
__device__ __forceinline__ double log_half(double x) {
  const int hi = __double2hiint(x), lo = __double2loint(x);
  const bool ok = (unsigned)(hi - 0x00100000) < 0x7fe00000u;
  int e = (hi >> 20) - 1023;
  int mh = (hi & 0x000fffff) | 0x3ff00000;
  const bool big = mh > 0x3ff6a09e;  // m > sqrt(2)
  mh = big ? mh - 0x00100000 : mh;
  e = big ? e + 1 : e;
  const double m = __hiloint2double(mh, lo);
  const double num = m - 1.0;  // exact (Sterbenz)
  const double f = num * rcp_refined(m + 1.0);
  const double f2 = f * f;
  const double f4 = f2 * f2;
  const double f8 = f4 * f4;
  const double q01 = fma(kLogPolyHalf[1], f2, kLogPolyHalf[0]);
  const double q23 = fma(kLogPolyHalf[3], f2, kLogPolyHalf[2]);
  const double q45 = fma(kLogPolyHalf[5], f2, kLogPolyHalf[4]);
  const double q67 = fma(kLogPolyHalf[7], f2, kLogPolyHalf[6]);
  const double q03 = fma(q23, f4, q01);
  const double q47 = fma(q67, f4, q45);
  const double p = fma(fma(kLogPolyHalf[8], f8, q47), f8, q03);
  const double lnm_half = fma(f * f2, p, f);
  const double de = (double)e;
  const double res = fma(de, kLogPolyHalf[9], fma(de, kLogPolyHalf[10], lnm_half));
  return dsel(ok, res, __longlong_as_double(0x7ff8000000000000ll));
}

// Table-driven ln(x)/2 for the warp kernels' node records (~10 FP64
// operations instead of log_half's ~22 and no reciprocal): after the same
// reduction x = 2^e m, m in [sqrt(1/2), sqrt(2)), the top mantissa bits pick
// c ~ 1/m from a 257-entry table (tools/gen_log_table.py; c = 1 next to
// m = 1), r = m c - 1 is formed by one FMA (|r| <= 2^-8), and
// ln(x)/2 = e ln2/2 + (-ln c)/2 + log1p(r)/2 with the series to r^6
// (truncation < 2e-18).  Absolute error ~1e-17 (the log mean only uses
// differences of these).  Non-positive / non-finite / subnormal -> NaN.
static __device__ __align__(16) const double kLogTab[2 * SFB_LOG_TABLE_N] = {SFB_LOG_TABLE_VALUES};
__device__ __forceinline__ double log_half_tab(double x) {
  const int hi = __double2hiint(x), lo = __double2loint(x);
  const bool ok = (unsigned)(hi - 0x00100000) < 0x7fe00000u;
  int e = (hi >> 20) - 1023;
  int mh = (hi & 0x000fffff) | 0x3ff00000;
  const bool big = mh > 0x3ff6a09e;  // m > sqrt(2)
  mh = big ? mh - 0x00100000 : mh;
  e = big ? e + 1 : e;
  int idx = (mh - SFB_LOG_TABLE_BASE) >> SFB_LOG_TABLE_SHIFT;
  idx = min(max(idx, 0), SFB_LOG_TABLE_N - 1);
  const double2 t = __ldg(reinterpret_cast<const double2*>(kLogTab) + idx);
  const double rh = fma(__hiloint2double(mh, lo), 0.5 * t.x, -0.5);  // r/2, one rounding
  const double r2 = rh * rh;
  // log1p(2 rh)/2 = rh - rh^2 + 4/3 rh^3 - 2 rh^4 + 16/5 rh^5 - 16/3 rh^6
  double p = fma(rh, -16.0 / 3.0, 16.0 / 5.0);
  p = fma(rh, p, -2.0);
  p = fma(rh, p, 4.0 / 3.0);
  p = fma(rh, p, -1.0);
  const double l1p = fma(r2, p, rh);
  // e ln2/2 with ln2/2 rounded to one double: the log mean only uses differences
  // of these logs, in which the rounding of ln2/2 cancels exactly for equal
  // exponents and contributes ~1e-17 per unit of exponent difference otherwise
  const double res = fma((double)e, 3.46573590279972654709e-01, l1p + t.y);
  return dsel(ok, res, __longlong_as_double(0x7ff8000000000000ll));
}

// Numerator / denominator of the log mean of (x, y) = (2 hx, 2 hy) (or any
// exact rescaling): L = num / den.
//   series branch:  num = s (s^2 - 3/5 d^2),  den = s^2 - 4/15 d^2
//   log branch:     num = d,                  den = (ln y - ln x)/2  (per-node logs)
// The series branch is the [1/1] Pade approximant in u = d^2/s^2 of
// L/s = 1 / (1 + u/3 + u^2/5 + u^3/7 + ...): (1 - 3u/5) / (1 - 4u/15), exact
// through u^2 with an O(u^3) remainder below 2e-16 relative for u <= 2e-5
// (checked against 50-digit logarithms) - no reciprocal, no MUFU in the chain.
// Branch test: integer comparison of the IEEE high words of d^2 and s^2,
// series iff hi(d^2) - hi(s^2) < -(hi(1.0) - hi(1e-5)), i.e. u below ~1e-5 -
// the test of the oracle (oracle/euler_oracle.py:series_branch, euler_oracle.c)
// verbatim, on the ALU (no FP64 compare).  Above it the per-node log
// difference loses at most ~|ln x| 1e-16 / (2|d/s|), |d/s| >= 3e-3 -> < 4e-14
// relative.  The final division happens in the caller's combined reciprocal.
__device__ __forceinline__ void logmean_parts(double hx, double hy, double hlx, double hly,
                                              double& num, double& den) {
  const double d = __dsub_rn(hy, hx);
  const double s = __dadd_rn(hx, hy);
  const double d2 = __dmul_rn(d, d);
  const double s2 = __dmul_rn(s, s);
  const bool series = (__double2hiint(d2) - __double2hiint(s2)) < -(int)(0x3ff00000 - 0x3ee4f8b5);
  num = dsel(series, s * fma(d2, -0.6, s2), d);
  den = dsel(series, fma(d2, -4.0 / 15.0, s2), __dsub_rn(hly, hlx));
}

// Cartesian Chandrashekar flux for K independent pairs at once, in the
// direction-rotated frame: the callers load the velocity components permuted
// so that hv0 is the component along the line's direction (and write the
// momentum results back un-permuted by address), so the flux never branches
// or selects on the direction.  Every statement is written across the K pairs
// so the instruction stream carries K independent dependency chains (DFMA
// latency ~9 cycles; tools/peaks/fp64_latency.cu).
// Records carry hb = (gamma - 1) beta and hlb = ln(hb)/2: the beta log mean
// then returns beta_ln / c_gamma (c_gamma = 1/(2(gamma-1))), so its reciprocal
// is already c_gamma / beta_ln, and betabar carries the same factor, absorbed
// into the p_hat constant (gm1 = gamma - 1): p_hat = rhobar / (2 betabar) =
// gm1 rhobar / sb.
template <int K>
__device__ __forceinline__ void chandrashekar_cart_v2(const NodeRec* const (&A)[K],
                                                      const NodeRec* const (&B)[K], double gm1,
                                                      double (&f)[K][5]) {
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
    logmean_parts(A[k]->hb, B[k]->hb, A[k]->hlb, B[k]->hlb, nb[k], db[k]);  // beta_ln/c
  }
  double sr[K], sb[K], p1[K], rr[K];
#pragma unroll
  for (int k = 0; k < K; ++k) {
    sr[k] = __dadd_rn(A[k]->hr, B[k]->hr);  // rhobar (CSE with the log mean's s)
    sb[k] = __dadd_rn(A[k]->hb, B[k]->hb);  // betabar / c_gamma
    p1[k] = dr[k] * nb[k];
    rr[k] = rcp_refined(p1[k] * sb[k]);
  }
#pragma unroll
  for (int k = 0; k < K; ++k) {
    const double inv_sb = rr[k] * p1[k];
    const double t = rr[k] * sb[k];
    const double rho_ln = nr[k] * (t * nb[k]);
    const double cibeta = db[k] * (t * dr[k]);  // c_gamma / beta_ln
    const double phat = (gm1 * sr[k]) * inv_sb;
    const double vn = vb0[k];
    const double f1 = rho_ln * vn;
    f[k][0] = f1;
    f[k][1] = fma(f1, vb0[k], phat);
    f[k][2] = f1 * vb1[k];
    f[k][3] = f1 * vb2[k];
    const double dot = fma(A[k]->hv2, B[k]->hv2, fma(A[k]->hv1, B[k]->hv1, A[k]->hv0 * B[k]->hv0));
    f[k][4] = fma(f1, fma(2.0, dot, cibeta), phat * vn);
  }
}

}  // namespace sfb
