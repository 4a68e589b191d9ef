// Batched sum-factorized Kronecker apply (operators.py:274-318 kronecker_apply):
// y = (A_{d-1} x ... x A_0) x, one direction at a time, direction 0 fastest.
// One CTA per vector; the intermediate tensor ping-pongs through shared memory
// and each pass is a small dense contraction along one axis (d n^{d+1} FMAs
// for square n x n factors, the count the reference tallies).
#include "common.cuh"

namespace sfb {

struct KronDesc {
  int d;
  int rows[3], cols[3];
  int off[3];  // offset of factor j in the packed factor array
};

__global__ void kron_apply_kernel(int64_t B, KronDesc kd, const double* __restrict__ factors,
                                  const double* __restrict__ x, double* __restrict__ y,
                                  int in_size, int out_size, int buf) {
  extern __shared__ double s[];
  double* fa = s;                 // packed factors
  double* t0 = s + kd.off[2] + kd.rows[2] * kd.cols[2];
  double* t1 = t0 + buf;
  const int nf = kd.off[kd.d - 1] + kd.rows[kd.d - 1] * kd.cols[kd.d - 1];
  for (int i = threadIdx.x; i < nf; i += blockDim.x) fa[i] = factors[i];
  for (int64_t b = blockIdx.x; b < B; b += gridDim.x) {
    __syncthreads();
    for (int i = threadIdx.x; i < in_size; i += blockDim.x) t0[i] = x[b * in_size + i];
    __syncthreads();
    // current extents, direction 0 fastest
    int ext[3] = {kd.cols[0], kd.d > 1 ? kd.cols[1] : 1, kd.d > 2 ? kd.cols[2] : 1};
    double* src = t0;
    double* dst = t1;
    for (int j = 0; j < kd.d; ++j) {
      int lo = 1;
      for (int i = 0; i < j; ++i) lo *= ext[i];
      int hi = 1;
      for (int i = j + 1; i < kd.d; ++i) hi *= ext[i];
      const int rj = kd.rows[j], cj = kd.cols[j];
      const double* A = fa + kd.off[j];
      const int total = lo * rj * hi;
      for (int o = threadIdx.x; o < total; o += blockDim.x) {
        const int a = o % lo;
        const int r = (o / lo) % rj;
        const int h = o / (lo * rj);
        const double* in = src + a + h * lo * cj;
        double acc = 0.0;
        for (int c = 0; c < cj; ++c) acc = fma(A[r * cj + c], in[c * lo], acc);
        dst[o] = acc;
      }
      ext[j] = rj;
      __syncthreads();
      double* t = src;
      src = dst;
      dst = t;
    }
    for (int i = threadIdx.x; i < out_size; i += blockDim.x) y[b * out_size + i] = src[i];
  }
}

}  // namespace sfb

using namespace sfb;

extern "C" int sfb_kronecker_apply(int64_t B, int64_t d, const int64_t* rows_1d,
                                   const int64_t* cols_1d, const double* factors, const double* x,
                                   double* y, sfb_stream_t stream) {
  SFB_CHECK_ARG(d >= 1 && d <= 3, "kronecker_apply: d must be 1..3");
  SFB_CHECK_ARG(rows_1d && cols_1d, "null extents (host arrays)");
  SFB_CHECK_ARG(B >= 0, "negative batch");
  KronDesc kd{};
  kd.d = (int)d;
  int off = 0, in_size = 1, out_size = 1, buf = 1;
  for (int j = 0; j < 3; ++j) {
    int r = j < d ? (int)rows_1d[j] : 1, c = j < d ? (int)cols_1d[j] : 1;
    SFB_CHECK_ARG(r >= 1 && r <= 16 && c >= 1 && c <= 16, "factor extents must be in 1..16");
    kd.rows[j] = r;
    kd.cols[j] = c;
    kd.off[j] = off;
    if (j < d) off += r * c;
  }
  // pad unused directions so the smem carve-out arithmetic stays uniform
  for (int j = (int)d; j < 3; ++j) kd.off[j] = off, kd.rows[j] = 0, kd.cols[j] = 0;
  {
    int ext[3] = {kd.cols[0], d > 1 ? kd.cols[1] : 1, d > 2 ? kd.cols[2] : 1};
    for (int j = 0; j < d; ++j) in_size *= ext[j];
    for (int j = 0; j < d; ++j) {
      ext[j] = kd.rows[j];
      int sz = 1;
      for (int i = 0; i < d; ++i) sz *= ext[i];
      if (sz > buf) buf = sz;
    }
    if (in_size > buf) buf = in_size;
    out_size = 1;
    for (int j = 0; j < d; ++j) out_size *= kd.rows[j];
  }
  if (B == 0) return SFB_OK;
  SFB_CHECK_ARG(factors && x && y, "null pointer");
  size_t smem = (size_t)(off + 2 * buf) * sizeof(double);
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(kron_apply_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
  int64_t grid = B < (int64_t)num_sms() * 16 ? B : (int64_t)num_sms() * 16;
  kron_apply_kernel<<<(unsigned)grid, 256, smem, (cudaStream_t)stream>>>(B, kd, factors, x, y,
                                                                         in_size, out_size, buf);
  return check_launch("kronecker_apply");
}
