// Device restatements of the reference's numpy / Python floating-point order,
// shared by the bitwise kernels (pattern.cu, burgers_time.cu): separately
// rounded products (no FMA contraction: __dmul_rn / __dadd_rn / __ddiv_rn) and
// numpy's summation order.
#pragma once

#include "common.cuh"

namespace sfb {

__device__ __forceinline__ double two_point(int flux, double a, double b) {
  switch (flux) {
    case SFB_FLUX_BURGERS_EC:  // (a*a + a*b + b*b) / 6.0, burgers.py:36-43
      return __ddiv_rn(__dadd_rn(__dadd_rn(__dmul_rn(a, a), __dmul_rn(a, b)), __dmul_rn(b, b)),
                       6.0);
    case SFB_FLUX_BURGERS_AVG:  // (a*a/2.0 + b*b/2.0) / 2.0, burgers.py:46-49
      return __ddiv_rn(
          __dadd_rn(__ddiv_rn(__dmul_rn(a, a), 2.0), __ddiv_rn(__dmul_rn(b, b), 2.0)), 2.0);
    default:  // rank one, _kernels.py:86-88
      return __dmul_rn(a, b);
  }
}

// numpy's pairwise_sum (numpy/_core/src/umath/loops_utils.h.src): sequential
// below 8, eight running lanes up to 128, recursive split at a multiple of 8
// above.  Recursion depth is log2(n / 128).
template <typename Load>
__device__ double numpy_pairwise_sum(Load x, int64_t lo, int64_t n) {
  if (n <= 128) {
    if (n < 8) {
      double res = 0.0;
      for (int64_t i = 0; i < n; ++i) res = __dadd_rn(res, x(lo + i));
      return res;
    }
    double r[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) r[q] = x(lo + q);
    int64_t i = 8;
    for (; i < n - (n % 8); i += 8) {
#pragma unroll
      for (int q = 0; q < 8; ++q) r[q] = __dadd_rn(r[q], x(lo + i + q));
    }
    double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                           __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
    for (; i < n; ++i) res = __dadd_rn(res, x(lo + i));
    return res;
  }
  int64_t n2 = n / 2;
  n2 -= n2 % 8;
  double left = numpy_pairwise_sum(x, lo, n2);
  return __dadd_rn(left, numpy_pairwise_sum(x, lo + n2, n - n2));
}

// Fast path for the common n <= 16 sizes (no recursion needed below 129).
template <typename Load>
__device__ __forceinline__ double numpy_sum_small(Load x, int n) {
  if (n < 8) {
    double res = 0.0;
    for (int i = 0; i < n; ++i) res = __dadd_rn(res, x(i));
    return res;
  }
  double r[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) r[q] = x(q);
  int i = 8;
  for (; i < n - (n % 8); i += 8) {
#pragma unroll
    for (int q = 0; q < 8; ++q) r[q] = __dadd_rn(r[q], x(i + q));
  }
  double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                         __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
  for (; i < n; ++i) res = __dadd_rn(res, x(i));
  return res;
}

}  // namespace sfb
