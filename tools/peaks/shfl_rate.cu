// Warp shuffle (SHFL.IDX / BFLY on 64-bit values) and shared-load throughput per
// SM on this GPU: warp-instructions per clock per SM, all SMs busy.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void shfl_kernel(double* out, int iters) {
  double x = threadIdx.x * 1.0, y = 0.5;
  const int lane = threadIdx.x & 31;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      x = __shfl_sync(0xffffffffu, x, (lane + k + 1) & 31);
      y = __shfl_xor_sync(0xffffffffu, y, 1 + (k & 7));
    }
  }
  if (x + y == 123.456) out[0] = x;
}

__global__ void lds_kernel(double* out, int iters) {
  __shared__ double s[2048];
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) s[i] = i;
  __syncthreads();
  double acc = 0;
  int idx = threadIdx.x;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 32; ++k) {
      acc += s[(idx + k * 37) & 2047];
    }
    idx = (idx + 1) & 2047;
  }
  if (acc == 123.456) out[0] = acc;
}

int main() {
  int sms, clk;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  double* d;
  cudaMalloc(&d, 8);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int iters = 4096;
  for (int warps = 8; warps <= 32; warps *= 2) {
    shfl_kernel<<<sms, warps * 32>>>(d, 16);
    cudaEventRecord(a);
    shfl_kernel<<<sms, warps * 32>>>(d, iters);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    double instr = (double)warps * iters * 32;  // per SM, 32 SHFL per iteration
    printf("SHFL.64 (2 x 32-bit each): warps/SM %d: %.3f warp-SHFL64/clk/SM\n", warps,
           instr / (ms * 1e-3 * clk * 1e3));
    lds_kernel<<<sms, warps * 32>>>(d, 16);
    cudaEventRecord(a);
    lds_kernel<<<sms, warps * 32>>>(d, iters);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    printf("LDS.64: warps/SM %d: %.3f warp-LDS64/clk/SM\n", warps, instr / (ms * 1e-3 * clk * 1e3));
  }
  return 0;
}
