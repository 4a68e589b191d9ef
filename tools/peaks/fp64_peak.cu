// FP64 pipe microbenchmarks for the roofline denominator (MEASURED_PEAKS.json
// carries no FP64 entry).  Each kernel runs a long chain of independent DFMA /
// log / division streams per thread; timed with CUDA events, best of 5.
#include <cstdio>
#include <cuda_runtime.h>
#include <cmath>

#define CHK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); return 1; } } while (0)

constexpr int ILP = 8;

__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double x[ILP];
#pragma unroll
  for (int i = 0; i < ILP; ++i) x[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
#pragma unroll
      for (int i = 0; i < ILP; ++i) x[i] = fma(x[i], a, b);
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < ILP; ++i) s += x[i];
  if (s == 123.456) out[0] = s;
}

__global__ void log_kernel(double* out, int iters) {
  double x[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) x[i] = 1.0 + threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 4; ++i) x[i] = log(x[i]) + 2.5;
  }
  double s = 0;
  for (int i = 0; i < 4; ++i) s += x[i];
  if (s == 123.456) out[0] = s;
}

__global__ void div_kernel(double* out, int iters) {
  double x[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) x[i] = 1.0 + threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 4; ++i) x[i] = 1.5 / x[i] + 1.0;
  }
  double s = 0;
  for (int i = 0; i < 4; ++i) s += x[i];
  if (s == 123.456) out[0] = s;
}

__global__ void rcpapprox_kernel(double* out, int iters) {
  double x[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) x[i] = 1.0 + threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      double r;
      asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x[i]));
      x[i] = r + 1.0;
    }
  }
  double s = 0;
  for (int i = 0; i < 4; ++i) s += x[i];
  if (s == 123.456) out[0] = s;
}

template <typename K, typename... A>
float time_kernel(K k, int blocks, int threads, A... args) {
  cudaEvent_t s, e;
  cudaEventCreate(&s); cudaEventCreate(&e);
  k<<<blocks, threads>>>(args...);
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(s);
    k<<<blocks, threads>>>(args...);
    cudaEventRecord(e);
    cudaEventSynchronize(e);
    float ms; cudaEventElapsedTime(&ms, s, e);
    if (ms < best) best = ms;
  }
  return best;
}

int main() {
  cudaDeviceProp p; CHK(cudaGetDeviceProperties(&p, 0));
  int sms = p.multiProcessorCount;
  double* out; CHK(cudaMalloc(&out, 8));
  int threads = 512, blocks = sms * 4;
  int iters = 4096;
  float ms = time_kernel(dfma_kernel, blocks, threads, out, iters, 0.999999, 1e-7);
  double flops = 2.0 * ILP * 16.0 * iters * (double)blocks * threads;
  printf("{\"sms\": %d, \"dfma_tflops\": %.3f, \"dfma_ms\": %.3f", sms, flops / ms / 1e9, ms);
  int li = 512;
  ms = time_kernel(log_kernel, blocks, threads, out, li);
  double n = 4.0 * li * (double)blocks * threads;
  printf(", \"log_per_s\": %.4e", n / ms * 1e3);
  ms = time_kernel(div_kernel, blocks, threads, out, li);
  printf(", \"div_per_s\": %.4e", n / ms * 1e3);
  ms = time_kernel(rcpapprox_kernel, blocks, threads, out, li);
  printf(", \"rcp_approx_per_s\": %.4e", n / ms * 1e3);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf(", \"clock_khz_attr\": %d}\n", clk);
  CHK(cudaGetLastError());
  return 0;
}
