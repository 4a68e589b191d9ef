// Pieces shared by the Cartesian Euler kernels (euler.cu, euler_warp.cu).
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

#ifndef SFB_PAIR_LEX
#define SFB_PAIR_LEX 1
#endif
#ifndef SFB_PAIR_LEX_N4
#define SFB_PAIR_LEX_N4 0
#endif
#ifndef SFB_PAIR_ORDER_N4
#define SFB_PAIR_ORDER_N4 2  // n = 4: the three perfect matchings one after another
#endif
// Pair order of one line: lexicographic, so a batch of K pairs shares its
// first node (at n = 4, K = 3: (0,1)(0,2)(0,3) | (1,2)(1,3)(2,3)), or the
// circle-method round robin (consecutive pairs disjoint, e.g. (0,3)(1,2)
// (1,3)(0,2) (2,3)(0,1)).  The compiler's schedule of the pair batches is
// sensitive to it: at n = 4 lexicographic measured 1.5% faster with the
// static block split and round robin 2.5% faster (0.401 -> 0.391 ms) since
// the dynamic block claims; at n = 3 lexicographic stays 2% ahead; n = 5..8
// do not care.  At n = 4 (K = 3) ten explicit orders were timed
// (SFB_PAIR_ORDER_N4, config 3 ms): the perfect matchings 01 23 | 02 13 |
// 03 12 one after another 0.387, round robin 0.390, other matching orders
// 0.389-0.395, reverse lexicographic 0.400, node-3 pairs last 0.401; the
// matchings order with K = 2 or 6 pairs per batch 0.397-0.399.
template <int N>
struct PairOrder {
  static constexpr int kPairs = N * (N - 1) / 2;
  int a[kPairs > 0 ? kPairs : 1], b[kPairs > 0 ? kPairs : 1];
  constexpr PairOrder() : a{}, b{} {
    int k = 0;
    if (N == 4 && SFB_PAIR_ORDER_N4 > 0) {  // explicit n = 4 orders (0: the macros below)
      constexpr int tab[10][12] = {
          {0, 3, 1, 2, 1, 3, 0, 2, 2, 3, 0, 1},  // 1: the round robin, written out
          {0, 1, 2, 3, 0, 2, 1, 3, 0, 3, 1, 2},  // 2: matchings, one after another
          {0, 1, 2, 3, 0, 3, 1, 2, 0, 2, 1, 3},
          {0, 2, 1, 3, 0, 1, 2, 3, 0, 3, 1, 2},
          {1, 2, 0, 3, 1, 3, 0, 2, 2, 3, 0, 1},
          {2, 3, 1, 3, 1, 2, 0, 3, 0, 2, 0, 1},  // 6: reverse lexicographic
          {0, 3, 1, 3, 2, 3, 0, 2, 1, 2, 0, 1},  // 7: last node shared per batch
          {0, 1, 0, 2, 1, 2, 0, 3, 1, 3, 2, 3},  // 8: triangle then the node 3 pairs
          {1, 2, 0, 3, 0, 2, 1, 3, 0, 1, 2, 3},
          {2, 3, 0, 1, 1, 3, 0, 2, 1, 2, 0, 3}};
      for (int i = 0; i < 6 && i < kPairs; ++i) {
        a[i] = tab[SFB_PAIR_ORDER_N4 - 1][2 * i];
        b[i] = tab[SFB_PAIR_ORDER_N4 - 1][2 * i + 1];
      }
      return;
    }
    if (N == 4 ? SFB_PAIR_LEX_N4 : SFB_PAIR_LEX) {  // lexicographic: (0,1) (0,2) .. (0,n-1) (1,2) ..
      for (int x = 0; x < N; ++x)
        for (int y = x + 1; y < N; ++y) {
          a[k] = x;
          b[k] = y;
          ++k;
        }
      return;
    }
    const int M = (N % 2 == 0) ? N : N + 1;  // odd N: dummy node M-1
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
