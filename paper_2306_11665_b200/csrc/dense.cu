// The reference's dense route (sumfac/oracle.py) and the general
// sum-factorized Kronecker apply (operators.py:274-318) on the device.
//
// The dense matrices are the O(n^{2d}) baseline the paper compares against:
// every entry is formed, zeros included, exactly as the reference forms it,
// so results are bitwise equal (products taken in the reference's order):
//
//   sfb_dense_direction_factor  oracle.py:54-92   weight product in ascending
//                               direction order, the basis value applied last
//   sfb_dense_kronecker         oracle.py:39-51   reduce(np.kron, reversed):
//                               ((f_{d-1} f_{d-2}) ...) f_0 per entry
//   sfb_dense_rank_one          oracle.py:111-124 (_kernels.rank_one_matrix)
//   sfb_scatter_direction /     oracle.py:127-160 one direction's compressed
//   sfb_gather_direction        factor to / from its dense matrix
//   sfb_kronecker_pass          one direction of kronecker_apply, any extents
//
// One thread per output entry, grid-stride; these are API-tier helpers (the
// batched hot paths live in euler*.cu / modal.cu / pattern.cu).
#include "common.cuh"

namespace sfb {
namespace {

unsigned grid_of(int64_t total, int threads) {
  int64_t g = (total + threads - 1) / threads;
  const int64_t cap = (int64_t)num_sms() * 32;
  return (unsigned)(g < 1 ? 1 : (g > cap ? cap : g));
}

constexpr int kMaxDims = 16;

struct DenseDesc {
  int d;
  int64_t rstride[kMaxDims], cstride[kMaxDims];  // x-fastest strides per direction
  int rows[kMaxDims], cols[kMaxDims];
  int64_t off[kMaxDims];  // factor j in the packed array (row-major rows x cols)
};

__global__ void dense_kronecker_kernel(DenseDesc dd, const double* __restrict__ packed,
                                       int64_t R, int64_t C, double* __restrict__ out) {
  const int64_t total = R * C;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = t / C, c = t % C;
    // reduce(np.kron, reversed(mats)): the slowest direction's value first
    double v = 0.0;
    for (int j = dd.d - 1; j >= 0; --j) {
      const int rj = (int)((r / dd.rstride[j]) % dd.rows[j]);
      const int cj = (int)((c / dd.cstride[j]) % dd.cols[j]);
      const double f = packed[dd.off[j] + (int64_t)rj * dd.cols[j] + cj];
      v = (j == dd.d - 1) ? f : __dmul_rn(v, f);
    }
    out[t] = v;
  }
}

// out (R x C) is zeroed by the caller; thread per (row, slot l)
__global__ void dense_direction_factor_kernel(int64_t R, int m, int n, int d, int dir,
                                              const double* __restrict__ basis,
                                              const double* __restrict__ weights, int64_t C,
                                              double* __restrict__ out) {
  const int64_t total = R * n;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = t / n;
    const int l = (int)(t % n);
    // digits of r: extent m in slot dir, n elsewhere (x fastest)
    int64_t rem = r, base = 0, cstride = 1, dstride = 1;
    int rdir = 0;
    double w = 1.0;
    bool have = false;
    for (int i = 0; i < d; ++i) {
      const int ext = (i == dir) ? m : n;
      const int digit = (int)(rem % ext);
      rem /= ext;
      if (i == dir) {
        rdir = digit;
        dstride = cstride;
      } else {
        base += (int64_t)digit * cstride;
        w = have ? __dmul_rn(w, weights[digit]) : weights[digit];
        have = true;
      }
      cstride *= n;
    }
    const double b = basis[(int64_t)rdir * n + l];
    out[r * C + base + (int64_t)l * dstride] = have ? __dmul_rn(b, w) : b;
  }
}

__global__ void dense_rank_one_kernel(const double* __restrict__ rv, const double* __restrict__ cv,
                                      int64_t R, int64_t C, double* __restrict__ out) {
  const int64_t total = R * C;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x)
    out[t] = __dmul_rn(rv[t / C], cv[t % C]);
}

__global__ void scatter_direction_kernel(const int64_t* __restrict__ rows,
                                         const int64_t* __restrict__ cols, int d, int dir,
                                         int64_t entries, const double* __restrict__ values,
                                         int64_t C, double* __restrict__ out) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < entries;
       k += (int64_t)gridDim.x * blockDim.x)
    out[rows[k * d + dir] * C + cols[k * d + dir]] = values[k];
}

__global__ void gather_direction_kernel(const int64_t* __restrict__ rows,
                                        const int64_t* __restrict__ cols, int d, int dir,
                                        int64_t entries, const double* __restrict__ dense,
                                        int64_t C, double* __restrict__ values) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < entries;
       k += (int64_t)gridDim.x * blockDim.x)
    values[k] = dense[rows[k * d + dir] * C + cols[k * d + dir]];
}

// y[b][h][r][a] = sum_c A[r][c] x[b][h][c][a]  (a < lo, h < hi), sequential
// sum over c; diag: y[b][h][r][a] = A[r] x[b][h][r][a]
__global__ void kron_pass_kernel(int64_t B, int64_t lo, int rj, int cj, int64_t hi, int diag,
                                 const double* __restrict__ A, const double* __restrict__ x,
                                 double* __restrict__ y) {
  const int64_t total = B * hi * rj * lo;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t a = t % lo;
    const int r = (int)((t / lo) % rj);
    const int64_t bh = t / (lo * rj);  // b * hi + h
    const double* in = x + bh * cj * lo + a;
    if (diag) {
      y[t] = __dmul_rn(A[r], in[(int64_t)r * lo]);
    } else {
      double acc = 0.0;
      for (int c = 0; c < cj; ++c) acc = fma(A[(int64_t)r * cj + c], in[(int64_t)c * lo], acc);
      y[t] = acc;
    }
  }
}

}  // namespace
}  // namespace sfb

using namespace sfb;

extern "C" int sfb_dense_kronecker(int64_t d, const int64_t* rows_1d, const int64_t* cols_1d,
                                   const double* packed, double* out, sfb_stream_t stream) {
  SFB_CHECK_ARG(d >= 1 && d <= kMaxDims, "dense_kronecker: d must be 1..16");
  SFB_CHECK_ARG(rows_1d && cols_1d, "null extents (host arrays)");
  DenseDesc dd{};
  dd.d = (int)d;
  int64_t R = 1, C = 1, off = 0;
  for (int j = 0; j < d; ++j) {
    SFB_CHECK_ARG(rows_1d[j] >= 1 && cols_1d[j] >= 1, "factor extents must be positive");
    dd.rows[j] = (int)rows_1d[j];
    dd.cols[j] = (int)cols_1d[j];
    dd.rstride[j] = R;
    dd.cstride[j] = C;
    dd.off[j] = off;
    R *= rows_1d[j];
    C *= cols_1d[j];
    off += rows_1d[j] * cols_1d[j];
  }
  if (R * C == 0) return SFB_OK;
  SFB_CHECK_ARG(packed && out, "null pointer");
  dense_kronecker_kernel<<<grid_of(R * C, 256), 256, 0, (cudaStream_t)stream>>>(dd, packed, R, C,
                                                                               out);
  return check_launch("dense_kronecker");
}

extern "C" int sfb_dense_direction_factor(int64_t m, int64_t n, int64_t d, int64_t direction,
                                          const double* basis, const double* weights, double* out,
                                          sfb_stream_t stream) {
  SFB_CHECK_ARG(m >= 1 && n >= 1 && d >= 1, "extents must be positive");
  SFB_CHECK_ARG(direction >= 0 && direction < d, "direction out of range");
  SFB_CHECK_ARG(basis && weights && out, "null pointer");
  int64_t R = m, C = n;
  for (int64_t i = 1; i < d; ++i) {
    R *= n;
    C *= n;
  }
  cudaStream_t s = (cudaStream_t)stream;
  if (cudaMemsetAsync(out, 0, (size_t)(R * C) * sizeof(double), s) != cudaSuccess)
    return fail(SFB_ECUDA, "dense_direction_factor: memset failed");
  dense_direction_factor_kernel<<<grid_of(R * n, 256), 256, 0, s>>>(
      R, (int)m, (int)n, (int)d, (int)direction, basis, weights, C, out);
  return check_launch("dense_direction_factor");
}

extern "C" int sfb_dense_rank_one(const double* row_values, int64_t R, const double* col_values,
                                  int64_t C, double* out, sfb_stream_t stream) {
  SFB_CHECK_ARG(R >= 0 && C >= 0, "negative extent");
  if (R * C == 0) return SFB_OK;
  SFB_CHECK_ARG(row_values && col_values && out, "null pointer");
  dense_rank_one_kernel<<<grid_of(R * C, 256), 256, 0, (cudaStream_t)stream>>>(
      row_values, col_values, R, C, out);
  return check_launch("dense_rank_one");
}

extern "C" int sfb_scatter_direction(const int64_t* rows, const int64_t* columns, int64_t d,
                                     int64_t direction, int64_t entries, const double* values,
                                     int64_t row_space, int64_t column_space, double* out,
                                     sfb_stream_t stream) {
  SFB_CHECK_ARG(d >= 1 && direction >= 0 && direction < d, "direction out of range");
  SFB_CHECK_ARG(entries >= 0 && row_space >= 0 && column_space >= 0, "negative extent");
  SFB_CHECK_ARG(out, "null pointer");
  cudaStream_t s = (cudaStream_t)stream;
  if (row_space * column_space > 0 &&
      cudaMemsetAsync(out, 0, (size_t)(row_space * column_space) * sizeof(double), s) !=
          cudaSuccess)
    return fail(SFB_ECUDA, "scatter: memset failed");
  if (entries == 0) return SFB_OK;
  SFB_CHECK_ARG(rows && columns && values, "null pointer");
  scatter_direction_kernel<<<grid_of(entries, 256), 256, 0, s>>>(
      rows, columns, (int)d, (int)direction, entries, values, column_space, out);
  return check_launch("scatter_direction");
}

extern "C" int sfb_gather_direction(const int64_t* rows, const int64_t* columns, int64_t d,
                                    int64_t direction, int64_t entries, const double* dense,
                                    int64_t column_space, double* values, sfb_stream_t stream) {
  SFB_CHECK_ARG(d >= 1 && direction >= 0 && direction < d, "direction out of range");
  SFB_CHECK_ARG(entries >= 0 && column_space >= 0, "negative extent");
  if (entries == 0) return SFB_OK;
  SFB_CHECK_ARG(rows && columns && dense && values, "null pointer");
  gather_direction_kernel<<<grid_of(entries, 256), 256, 0, (cudaStream_t)stream>>>(
      rows, columns, (int)d, (int)direction, entries, dense, column_space, values);
  return check_launch("gather_direction");
}

extern "C" int sfb_kronecker_pass(int64_t B, int64_t lo, int64_t rows, int64_t cols, int64_t hi,
                                  int diag, const double* A, const double* x, double* y,
                                  sfb_stream_t stream) {
  SFB_CHECK_ARG(B >= 0 && lo >= 1 && rows >= 1 && cols >= 1 && hi >= 1, "bad extents");
  SFB_CHECK_ARG(!diag || rows == cols, "a diagonal factor is square");
  if (B == 0) return SFB_OK;
  SFB_CHECK_ARG(A && x && y, "null pointer");
  SFB_CHECK_ARG(x != y, "kronecker_pass cannot run in place");
  const int64_t total = B * hi * rows * lo;
  kron_pass_kernel<<<grid_of(total, 256), 256, 0, (cudaStream_t)stream>>>(
      B, lo, (int)rows, (int)cols, hi, diag, A, x, y);
  return check_launch("kronecker_pass");
}
