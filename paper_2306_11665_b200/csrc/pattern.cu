// Unfused sum-factorization stages on the device: Algorithm 1 (pattern),
// Algorithm 2 (basis assembly), operand assembly, Hadamard evaluation and the
// row sum, plus the fused batched Hadamard + row-sum + direction-sum (K2).
//
// Every kernel reproduces the reference's floating-point operation order
// (products rounded separately - no FMA contraction - and numpy's summation
// order), so outputs are bitwise equal to the reference pipeline:
//   fill_pattern      <- _kernels.py:15-40
//   assemble_basis    <- _kernels.py:43-76
//   assemble_rank_one <- _kernels.py:79-88 (and the func path, kernel.py:226-229)
//   hadamard_evaluate <- kernel.py:233-248
//   hadamard_row_sum  <- kernel.py:251-266 (numpy pairwise_sum order)
#include "common.cuh"
#include "numpy_order.cuh"

namespace sfb {

// --------------------------------------------------------------------------
// K1: Algorithm 1.  One thread per (entry, direction); output (entries, d)
// row-major, so consecutive threads write consecutive int64s.
// --------------------------------------------------------------------------
__global__ void fill_pattern_kernel(int64_t m, int64_t n, int64_t d, int64_t entries,
                                    int64_t* __restrict__ rows, int64_t* __restrict__ columns) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t total = entries * d;
  for (; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    int64_t k = t / d;
    int64_t j = t - k * d;
    int64_t glob = k / n;
    int64_t l = k - glob * n;
    int64_t rem = glob, colflat = 0, colstride = 1;
    for (int64_t i = 0; i < d; ++i) {
      int64_t ext = (i == j) ? m : n;
      int64_t digit = rem % ext;
      rem /= ext;
      colflat += ((i == j) ? l : digit) * colstride;
      colstride *= n;
    }
    rows[t] = glob;
    columns[t] = colflat;
  }
}

// --------------------------------------------------------------------------
// K5: Algorithm 2.  Weight product in ascending direction, basis value last.
// --------------------------------------------------------------------------
__global__ void assemble_basis_kernel(const int64_t* __restrict__ rows,
                                      const int64_t* __restrict__ columns,
                                      const double* __restrict__ basis,
                                      const double* __restrict__ weights, int64_t m, int64_t n,
                                      int64_t d, int64_t entries, double* __restrict__ out) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t total = entries * d;
  int64_t R = entries / n;
  for (; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    int64_t j = t / entries;
    int64_t k = t - j * entries;
    int64_t colstride_j = 1;
    for (int64_t i = 0; i < j; ++i) colstride_j *= n;
    int64_t row = rows[k * d + j];
    int64_t counter = k - (k / n) * n;
    int64_t cj = (columns[k * d + j] / colstride_j) % n;
    int64_t rem = row, rj = 0;
    double wprod = 1.0;
    bool have_weight = false;
    for (int64_t i = 0; i < d; ++i) {
      int64_t ext = (i == j) ? m : n;
      int64_t digit = rem % ext;
      rem /= ext;
      if (i == j) {
        rj = digit;
      } else if (have_weight) {
        wprod = __dmul_rn(wprod, weights[digit]);
      } else {
        wprod = weights[digit];
        have_weight = true;
      }
    }
    double value = basis[rj * n + cj];
    out[(j * R + row) * n + counter] = have_weight ? __dmul_rn(value, wprod) : value;
  }
}

// --------------------------------------------------------------------------
// K6: operand assembly at the pattern positions (rank one or built-in flux).
// --------------------------------------------------------------------------
__global__ void assemble_two_point_kernel(const int64_t* __restrict__ rows,
                                          const int64_t* __restrict__ columns,
                                          const double* __restrict__ rv,
                                          const double* __restrict__ cv, int64_t n, int64_t d,
                                          int64_t entries, int flux, double* __restrict__ out) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t total = entries * d;
  int64_t R = entries / n;
  for (; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    int64_t j = t / entries;
    int64_t k = t - j * entries;
    int64_t row = rows[k * d + j];
    int64_t counter = k - (k / n) * n;
    out[(j * R + row) * n + counter] = two_point(flux, rv[row], cv[columns[k * d + j]]);
  }
}

__global__ void gather_dense_kernel(const int64_t* __restrict__ rows,
                                    const int64_t* __restrict__ columns,
                                    const double* __restrict__ dense, int64_t ncols, int64_t n,
                                    int64_t d, int64_t entries, double* __restrict__ out) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t total = entries * d;
  int64_t R = entries / n;
  for (; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    int64_t j = t / entries;
    int64_t k = t - j * entries;
    int64_t row = rows[k * d + j];
    int64_t counter = k - (k / n) * n;
    out[(j * R + row) * n + counter] = dense[row * ncols + columns[k * d + j]];
  }
}

__global__ void hadamard_evaluate_kernel(const double* __restrict__ a,
                                         const double* __restrict__ b, int64_t count,
                                         double* __restrict__ out) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  for (; t < count; t += (int64_t)gridDim.x * blockDim.x) out[t] = __dmul_rn(a[t], b[t]);
}

template <bool LARGE>  // n > 128: numpy's recursive split (the other has no stack)
__global__ void row_sum_kernel(const double* __restrict__ p, int64_t rows, int64_t n,
                               double* __restrict__ out) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  for (; t < rows; t += (int64_t)gridDim.x * blockDim.x) {
    const double* row = p + t * n;
    auto ld = [row](int64_t i) { return row[i]; };
    if constexpr (LARGE) out[t] = numpy_pairwise_sum(ld, 0, n);
    else out[t] = numpy_sum_small(ld, (int)n);
  }
}

// --------------------------------------------------------------------------
// K2: fused batched Hadamard + row sum + direction sum (configs 1-2).
// One thread per (element, row R).  For direction j the thread reads the n
// contiguous F entries of its row (consecutive threads -> consecutive rows,
// so a warp streams 32*n*8 contiguous bytes per direction), multiplies by the
// element-independent basis factor (L1/L2 resident) with separately rounded
// products, sums in numpy order, then accumulates over j sequentially.
// --------------------------------------------------------------------------
template <int N, int D>
__global__ void __launch_bounds__(256) hadamard_rowsum_fixed_kernel(
    int64_t E, int64_t R, const double* __restrict__ basis, const double* __restrict__ F,
    double* __restrict__ out_dir, double* __restrict__ out_sum) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t total = E * R;
  for (; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = t / R;
    const int64_t row = t - e * R;
    // issue every direction's loads before any arithmetic: D*N*8 bytes in
    // flight per thread (memory-level parallelism for an HBM-bound stream)
    double fv[D][N], bv[D][N];
#pragma unroll
    for (int j = 0; j < D; ++j) {
      const double* f = F + ((e * D + j) * R + row) * N;
      const double* b = basis + ((int64_t)j * R + row) * N;
      if constexpr (N % 4 == 0) {
#pragma unroll
        for (int l = 0; l < N; l += 4) {
          const d4 v = ld_stream_d4(f + l);
          const d4 w = ld_ro_d4(b + l);
          fv[j][l] = v.x; fv[j][l + 1] = v.y; fv[j][l + 2] = v.z; fv[j][l + 3] = v.w;
          bv[j][l] = w.x; bv[j][l + 1] = w.y; bv[j][l + 2] = w.z; bv[j][l + 3] = w.w;
        }
      } else if constexpr (N % 2 == 0) {
#pragma unroll
        for (int l = 0; l < N; l += 2) {
          const double2 v = ld_stream_d2(f + l);
          const double2 w = __ldg(reinterpret_cast<const double2*>(b + l));
          fv[j][l] = v.x; fv[j][l + 1] = v.y;
          bv[j][l] = w.x; bv[j][l + 1] = w.y;
        }
      } else {
#pragma unroll
        for (int l = 0; l < N; ++l) {
          fv[j][l] = __ldcs(f + l);
          bv[j][l] = __ldg(b + l);
        }
      }
    }
    double acc = 0.0;
#pragma unroll
    for (int j = 0; j < D; ++j) {
      double p[N];
#pragma unroll
      for (int l = 0; l < N; ++l) p[l] = __dmul_rn(bv[j][l], fv[j][l]);
      const double s = numpy_sum_small([&p](int i) { return p[i]; }, N);
      if (out_dir) out_dir[(e * D + j) * R + row] = s;
      acc = (j == 0) ? s : __dadd_rn(acc, s);
    }
    if (out_sum) out_sum[t] = acc;
  }
}

// LARGE: rows longer than 128 need numpy's recursive split; the n <= 128
// instantiation carries no recursion (and so no stack / spills)
template <bool LARGE>
__global__ void hadamard_rowsum_generic_kernel(int64_t E, int64_t R, int64_t n, int d,
                                               const double* __restrict__ basis,
                                               const double* __restrict__ F,
                                               double* __restrict__ out_dir,
                                               double* __restrict__ out_sum) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t total = E * R;
  for (; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    int64_t e = t / R;
    int64_t row = t - e * R;
    double acc = 0.0;
    for (int j = 0; j < d; ++j) {
      const double* f = F + ((e * d + j) * R + row) * n;
      const double* b = basis + ((int64_t)j * R + row) * n;
      auto ld = [f, b](int64_t i) { return __dmul_rn(b[i], f[i]); };
      double s;
      if constexpr (LARGE) s = numpy_pairwise_sum(ld, 0, n);
      else s = numpy_sum_small(ld, (int)n);
      if (out_dir) out_dir[(e * d + j) * R + row] = s;
      acc = (j == 0) ? s : __dadd_rn(acc, s);
    }
    if (out_sum) out_sum[t] = acc;
  }
}

// --------------------------------------------------------------------------
// Scalar Burgers flux differencing, fused (burgers.py:117-131):
// out[e,r] = (-2.0 * sum_j rowsum_j[r]) / omega[r]
// --------------------------------------------------------------------------
template <bool LARGE>
__global__ void burgers_volume_kernel(int64_t E, int64_t n, int d, int64_t nodes,
                                      const double* __restrict__ qf,
                                      const double* __restrict__ omega, int flux,
                                      const double* __restrict__ u, double* __restrict__ out) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t total = E * nodes;
  for (; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    int64_t e = t / nodes;
    int64_t r = t - e * nodes;
    const double* ue = u + e * nodes;
    double ur = ue[r];
    double acc = 0.0;
    int64_t stride = 1;
    for (int j = 0; j < d; ++j) {
      int64_t digit = (r / stride) % n;
      int64_t base = r - digit * stride;
      const double* q = qf + ((int64_t)j * nodes + r) * n;
      auto ld = [&](int64_t l) { return __dmul_rn(q[l], two_point(flux, ur, ue[base + l * stride])); };
      double s;
      if constexpr (LARGE) s = numpy_pairwise_sum(ld, 0, n);
      else s = numpy_sum_small(ld, (int)n);
      acc = (j == 0) ? s : __dadd_rn(acc, s);
      stride *= n;
    }
    out[t] = __ddiv_rn(__dmul_rn(-2.0, acc), omega[r]);
  }
}

static int grid_for(int64_t work, int threads) {
  int64_t blocks = (work + threads - 1) / threads;
  int64_t cap = (int64_t)num_sms() * 32;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  return (int)blocks;
}

}  // namespace sfb

using namespace sfb;

extern "C" int sfb_fill_pattern(int64_t m, int64_t n, int64_t d, int64_t* rows, int64_t* columns,
                                sfb_stream_t stream) {
  SFB_CHECK_ARG(m >= 1 && n >= 1 && d >= 1, "extents must be positive");
  SFB_CHECK_ARG(rows && columns, "null output pointer");
  int64_t entries = m;
  for (int64_t i = 0; i < d; ++i) entries *= n;
  int64_t total = entries * d;
  if (total == 0) return SFB_OK;
  fill_pattern_kernel<<<grid_for(total, 256), 256, 0, (cudaStream_t)stream>>>(m, n, d, entries,
                                                                              rows, columns);
  return check_launch("fill_pattern");
}

extern "C" int sfb_assemble_basis(const int64_t* rows, const int64_t* columns, const double* basis,
                                  const double* weights, int64_t m, int64_t n, int64_t d,
                                  double* out, sfb_stream_t stream) {
  SFB_CHECK_ARG(m >= 1 && n >= 1 && d >= 1, "extents must be positive");
  SFB_CHECK_ARG(rows && columns && basis && weights && out, "null pointer");
  int64_t entries = m;
  for (int64_t i = 0; i < d; ++i) entries *= n;
  int64_t total = entries * d;
  assemble_basis_kernel<<<grid_for(total, 256), 256, 0, (cudaStream_t)stream>>>(
      rows, columns, basis, weights, m, n, d, entries, out);
  return check_launch("assemble_basis");
}

extern "C" int sfb_assemble_two_point(const int64_t* rows, const int64_t* columns,
                                      const double* row_values, const double* col_values,
                                      int64_t m, int64_t n, int64_t d, int flux, double* out,
                                      sfb_stream_t stream) {
  SFB_CHECK_ARG(m >= 1 && n >= 1 && d >= 1, "extents must be positive");
  SFB_CHECK_ARG(flux >= SFB_FLUX_PRODUCT && flux <= SFB_FLUX_BURGERS_AVG, "unknown flux id");
  SFB_CHECK_ARG(rows && columns && row_values && col_values && out, "null pointer");
  int64_t entries = m;
  for (int64_t i = 0; i < d; ++i) entries *= n;
  int64_t total = entries * d;
  assemble_two_point_kernel<<<grid_for(total, 256), 256, 0, (cudaStream_t)stream>>>(
      rows, columns, row_values, col_values, n, d, entries, flux, out);
  return check_launch("assemble_two_point");
}

extern "C" int sfb_gather_dense(const int64_t* rows, const int64_t* columns, const double* dense,
                                int64_t m, int64_t n, int64_t d, double* out,
                                sfb_stream_t stream) {
  SFB_CHECK_ARG(m >= 1 && n >= 1 && d >= 1, "extents must be positive");
  SFB_CHECK_ARG(rows && columns && dense && out, "null pointer");
  int64_t entries = m, ncols = 1;
  for (int64_t i = 0; i < d; ++i) {
    entries *= n;
    ncols *= n;
  }
  int64_t total = entries * d;
  gather_dense_kernel<<<grid_for(total, 256), 256, 0, (cudaStream_t)stream>>>(
      rows, columns, dense, ncols, n, d, entries, out);
  return check_launch("gather_dense");
}

extern "C" int sfb_hadamard_evaluate(const double* a, const double* b, int64_t count, double* out,
                                     sfb_stream_t stream) {
  SFB_CHECK_ARG(count >= 0, "negative count");
  if (count == 0) return SFB_OK;
  SFB_CHECK_ARG(a && b && out, "null pointer");
  hadamard_evaluate_kernel<<<grid_for(count, 256), 256, 0, (cudaStream_t)stream>>>(a, b, count,
                                                                                   out);
  return check_launch("hadamard_evaluate");
}

extern "C" int sfb_hadamard_row_sum(const double* product, int64_t rows, int64_t n, double* out,
                                    sfb_stream_t stream) {
  SFB_CHECK_ARG(rows >= 0 && n >= 1, "bad extents");
  if (rows == 0) return SFB_OK;
  SFB_CHECK_ARG(product && out, "null pointer");
  auto kern = n <= 128 ? row_sum_kernel<false> : row_sum_kernel<true>;
  kern<<<grid_for(rows, 256), 256, 0, (cudaStream_t)stream>>>(product, rows, n, out);
  return check_launch("hadamard_row_sum");
}

extern "C" int sfb_hadamard_rowsum_batched(int64_t E, int64_t m, int64_t n, int64_t d,
                                           const double* basis, const double* F, double* out_dir,
                                           double* out_sum, sfb_stream_t stream) {
  SFB_CHECK_ARG(E >= 0 && m >= 1 && n >= 1 && d >= 1 && d <= 16, "bad extents");
  SFB_CHECK_ARG(basis && F, "null input pointer");
  if (E == 0 || (!out_dir && !out_sum)) return SFB_OK;
  int64_t R = m;
  for (int64_t i = 1; i < d; ++i) R *= n;
  int64_t total = E * R;
  cudaStream_t s = (cudaStream_t)stream;
  int threads = 256;
  int64_t blocks64 = (total + threads - 1) / threads;
  int blocks = (int)(blocks64 > (1 << 30) ? (1 << 30) : blocks64);
  bool aligned = (((uintptr_t)F | (uintptr_t)basis) % 32) == 0;
  // fixed-size kernels where they beat the generic one (n-sweep of bench.py
  // --config 2: n = 5, 7, 9, 12 at d = 3 gain; 10, 11, 13 lose to it)
  const int key = aligned ? (int)(n * 10 + d) : 0;
  switch (key) {
    case 23: hadamard_rowsum_fixed_kernel<2, 3><<<blocks, threads, 0, s>>>(E, R, basis, F, out_dir, out_sum); break;
    case 33: hadamard_rowsum_fixed_kernel<3, 3><<<blocks, threads, 0, s>>>(E, R, basis, F, out_dir, out_sum); break;
    case 43: hadamard_rowsum_fixed_kernel<4, 3><<<blocks, threads, 0, s>>>(E, R, basis, F, out_dir, out_sum); break;
    case 42: hadamard_rowsum_fixed_kernel<4, 2><<<blocks, threads, 0, s>>>(E, R, basis, F, out_dir, out_sum); break;
    case 52: hadamard_rowsum_fixed_kernel<5, 2><<<blocks, threads, 0, s>>>(E, R, basis, F, out_dir, out_sum); break;
    case 63: hadamard_rowsum_fixed_kernel<6, 3><<<blocks, threads, 0, s>>>(E, R, basis, F, out_dir, out_sum); break;
    case 83: hadamard_rowsum_fixed_kernel<8, 3><<<blocks, threads, 0, s>>>(E, R, basis, F, out_dir, out_sum); break;
    case 53: hadamard_rowsum_fixed_kernel<5, 3><<<blocks, threads, 0, s>>>(E, R, basis, F, out_dir, out_sum); break;
    case 73: hadamard_rowsum_fixed_kernel<7, 3><<<blocks, threads, 0, s>>>(E, R, basis, F, out_dir, out_sum); break;
    case 93: hadamard_rowsum_fixed_kernel<9, 3><<<blocks, threads, 0, s>>>(E, R, basis, F, out_dir, out_sum); break;
    case 123: hadamard_rowsum_fixed_kernel<12, 3><<<blocks, threads, 0, s>>>(E, R, basis, F, out_dir, out_sum); break;
    default:
      if (n <= 128)
        hadamard_rowsum_generic_kernel<false><<<grid_for(total, threads), threads, 0, s>>>(
            E, R, n, (int)d, basis, F, out_dir, out_sum);
      else
        hadamard_rowsum_generic_kernel<true><<<grid_for(total, threads), threads, 0, s>>>(
            E, R, n, (int)d, basis, F, out_dir, out_sum);
  }
  return check_launch("hadamard_rowsum_batched");
}

extern "C" int sfb_burgers_volume(int64_t E, int64_t n, int64_t d, const double* qfactors,
                                  const double* omega, int flux, const double* u, double* out,
                                  sfb_stream_t stream) {
  SFB_CHECK_ARG(E >= 0 && n >= 1 && d >= 1 && d <= 16, "bad extents");
  SFB_CHECK_ARG(flux >= SFB_FLUX_PRODUCT && flux <= SFB_FLUX_BURGERS_AVG, "unknown flux id");
  if (E == 0) return SFB_OK;
  SFB_CHECK_ARG(qfactors && omega && u && out, "null pointer");
  int64_t nodes = 1;
  for (int64_t i = 0; i < d; ++i) nodes *= n;
  int64_t total = E * nodes;
  auto kern = n <= 128 ? burgers_volume_kernel<false> : burgers_volume_kernel<true>;
  kern<<<grid_for(total, 256), 256, 0, (cudaStream_t)stream>>>(
      E, n, (int)d, nodes, qfactors, omega, flux, u, out);
  return check_launch("burgers_volume");
}
