// FP64 pipe latency / throughput vs ILP and warps per SM (design input for
// the flux kernel's occupancy/ILP trade-off).
#include <cstdio>
#include <cuda_runtime.h>

template <int ILP>
__global__ void chain(double* out, int iters, double a, double b) {
  double x[ILP];
#pragma unroll
  for (int i = 0; i < ILP; ++i) x[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 8; ++k)
#pragma unroll
      for (int i = 0; i < ILP; ++i) x[i] = fma(x[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < ILP; ++i) s += x[i];
  if (s == 1.2345) out[0] = s;
}

template <int ILP>
void run(double* out, int warps_per_sm, int sms) {
  int threads = 32 * warps_per_sm;
  if (threads > 1024) return;
  int iters = 2000;
  cudaEvent_t s, e;
  cudaEventCreate(&s); cudaEventCreate(&e);
  chain<ILP><<<sms, threads>>>(out, iters, 0.9999999, 1e-9);
  cudaEventRecord(s);
  chain<ILP><<<sms, threads>>>(out, iters, 0.9999999, 1e-9);
  cudaEventRecord(e);
  cudaEventSynchronize(e);
  float ms; cudaEventElapsedTime(&ms, s, e);
  double warp_instr_per_sm = (double)warps_per_sm * iters * 8 * ILP;
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  double cycles = ms * 1e-3 * clk * 1e3;
  printf("ILP=%d warps/SM=%2d : %.3f warp-DFMA/clk/SM (peak 2.0), latency est %.1f cyc\n", ILP,
         warps_per_sm, warp_instr_per_sm / cycles,
         cycles / (iters * 8.0));
}

int main() {
  double* out; cudaMalloc(&out, 8);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int ws[] = {4, 8, 12, 16, 24, 32};
  for (int w : ws) run<1>(out, w, sms);
  for (int w : ws) run<2>(out, w, sms);
  for (int w : ws) run<4>(out, w, sms);
  return 0;
}
