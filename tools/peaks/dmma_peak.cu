// FP64 tensor-core (DMMA m8n8k4) throughput on this B200, alone and
// interleaved with DFMA, to decide whether the sum-factorised transforms
// should run on DMMA.  nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

template <int MODE>  // 0: DMMA only, 1: DFMA only, 2: both interleaved
__global__ void k(double* out, int iters, double x) {
  double c[8][2];
  double f[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    c[i][0] = c[i][1] = x * i;
    f[i] = x + i;
  }
  const double a = x * 1.0001, b = x * 0.9999;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (MODE != 1) dmma(c[i], a, b);
      if (MODE != 0) {
        f[i] = fma(f[i], a, b);
        f[i] = fma(f[i], a, b);
      }
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1] + f[i];
  if (s == 12345.678) out[0] = s;
}

int main() {
  double* out;
  cudaMalloc(&out, 8);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int iters = 20000, threads = 256, blocks = sms * 4;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int mode = 0; mode < 3; ++mode) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      if (mode == 0) k<0><<<blocks, threads>>>(out, iters, 1.0);
      if (mode == 1) k<1><<<blocks, threads>>>(out, iters, 1.0);
      if (mode == 2) k<2><<<blocks, threads>>>(out, iters, 1.0);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      const double warps = (double)blocks * threads / 32;
      const double mma_fl = mode != 1 ? warps * iters * 8 * 512.0 : 0;  // m8n8k4: 256 FMA
      const double fma_fl = mode != 0 ? (double)blocks * threads * iters * 8 * 2 * 2 : 0;
      if (rep == 1)
        printf("mode %d: %.3f ms  DMMA %.2f TF  DFMA %.2f TF  total %.2f TF\n", mode, ms,
               mma_fl / ms / 1e9, fma_fl / ms / 1e9, (mma_fl + fma_fl) / ms / 1e9);
    }
  }
  return 0;
}
