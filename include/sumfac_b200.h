/*
 * sumfac_b200.h - C ABI of the B200-native (sm_100a) sum-factorized Hadamard /
 * flux-differencing path.
 *
 * This is the drop-in boundary for the reference package `sumfac` 0.1.0
 * (/root/reference/pkg).  The reference's native seam is `sumfac._kernels`:
 * numba loops over caller-preallocated, C-contiguous numpy arrays (int64
 * indices, float64 values) that return nothing and leave validation,
 * accounting and object plumbing to the Python wrappers
 * (_kernels.py:1-9).  Each function below replaces one of those loops, or one
 * numpy stage of kernel.py / burgers.py / operators.py, with the same argument
 * meaning.  Differences that follow from the device boundary:
 *
 *   - pointers are DEVICE pointers (cudaMalloc / torch CUDA tensors), except
 *     the small n x n operators of the Euler entries (D, V, Pi: HOST pointers,
 *     copied into the launch parameters) and the *_host entry points, which
 *     take host buffers (pinned or pageable) and do the copies themselves;
 *   - every call is stream-ordered on `stream` (a cudaStream_t; NULL = legacy
 *     default stream), does not synchronise, and does not allocate device
 *     memory (the *_host entry points keep one cached staging arena per
 *     device; calls on one device serialise on it);
 *   - errors: the return value is SFB_OK (0) or a nonzero SFB_E* code, and
 *     sfb_last_error() returns a thread-local message.  No C++ exception
 *     crosses the ABI.  The Python layer maps SFB_EINVAL to ValueError like the
 *     reference's wrappers do (kernel.py:84-92,185-188,200-217,239-243,258-263).
 *
 * Layouts (all C-contiguous, FP64 unless noted):
 *   node flat index   r = r_0 + r_1 n + r_2 n^2 ...   (indexing.py:1-10)
 *   pattern           rows/columns (entries, d) int64, entry k = R n + l
 *                     (kernel.py:25-72, _kernels.py:15-40)
 *   factor set        (d, R, n) with R = m n^(d-1)          (kernel.py:99-125)
 *   element batch     leading element axis E: F (E, d, R, n); states
 *                     U (E, 5, n^d) = [rho, rho v_x, rho v_y, rho v_z, E_tot]
 *                     per element, node axis fastest (structure of arrays)
 *   metric cofactors  Ja (E, 3, 3, n^3): Ja[e][i][m][r] = J dxi^i/dx_m at r
 */
#ifndef SUMFAC_B200_H
#define SUMFAC_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif
#if defined(__GNUC__)
#pragma GCC visibility push(default)
#endif

typedef struct CUstream_st* sfb_stream_t; /* == cudaStream_t */

#define SFB_OK 0
#define SFB_EINVAL 1 /* bad extents / shapes / arguments */
#define SFB_ECUDA 2  /* CUDA launch or runtime failure */
#define SFB_ENOTSUP 3 /* configuration not compiled (e.g. n outside 2..8) */

/* Two-point flux selectors for the scalar (Burgers) operand path. */
#define SFB_FLUX_PRODUCT 0 /* C[i,j] = rv[i] * cv[j]          (kernel.py:138-164, rank one) */
#define SFB_FLUX_BURGERS_EC 1 /* (a^2 + a b + b^2) / 6       (burgers.py:36-43) */
#define SFB_FLUX_BURGERS_AVG 2 /* (a^2/2 + b^2/2) / 2         (burgers.py:46-49) */

/* ---- library ---------------------------------------------------------- */
const char* sfb_last_error(void);
int sfb_version(void); /* 100 * major + minor */
/* Number of kernel launches issued by this library since load (all entry
 * points); used by bench.py to report gpu_launches. */
int64_t sfb_launch_count(void);

/* ---- Algorithm 1: sparsity pattern ------------------------------------
 * Replaces _kernels.fill_pattern (_kernels.py:15-40) called from
 * build_sparsity_pattern (kernel.py:75-96).  rows/columns: (m n^d, d) int64.
 * rows[k,j] = k / n; columns[k,j] = row multi-index (extent m in slot j, n
 * elsewhere) with digit j replaced by l = k % n, flattened over extents n. */
int sfb_fill_pattern(int64_t m, int64_t n, int64_t d, int64_t* rows, int64_t* columns,
                     sfb_stream_t stream);

/* ---- Algorithm 2: basis assembly --------------------------------------
 * Replaces _kernels.assemble_basis (_kernels.py:43-76) called from
 * assemble_basis_factors (kernel.py:172-192).  out[j,R,l] =
 * basis[r_j, c_j] * prod_{i!=j} weights[r_i], weights multiplied in ascending
 * i, basis value last (bitwise order of the reference).  basis (m,n),
 * weights (n), out (d, m n^(d-1), n). */
int sfb_assemble_basis(const int64_t* rows, const int64_t* columns, const double* basis,
                       const double* weights, int64_t m, int64_t n, int64_t d, double* out,
                       sfb_stream_t stream);

/* ---- operand assembly -------------------------------------------------
 * Replaces _kernels.assemble_rank_one (_kernels.py:79-88) for
 * flux == SFB_FLUX_PRODUCT and the func path of assemble_operand_factors
 * (kernel.py:226-229) for the built-in Burgers fluxes.  out[j,R,l] =
 * f(row_values[rows[k,j]], col_values[columns[k,j]]) with k = R n + l.
 * m is the row extent of the pattern (R = m n^(d-1)). */
int sfb_assemble_two_point(const int64_t* rows, const int64_t* columns,
                           const double* row_values, const double* col_values, int64_t m,
                           int64_t n, int64_t d, int flux, double* out, sfb_stream_t stream);

/* Gather of a dense operand matrix at the pattern (oracle.gather,
 * oracle.py:158-167): out[j,R,l] = dense[rows[k,j], columns[k,j]].
 * dense (m n^(d-1), n^d). */
int sfb_gather_dense(const int64_t* rows, const int64_t* columns, const double* dense,
                     int64_t m, int64_t n, int64_t d, double* out, sfb_stream_t stream);

/* ---- evaluation -------------------------------------------------------
 * hadamard_evaluate (kernel.py:233-248): out = a * b entrywise, count entries. */
int sfb_hadamard_evaluate(const double* a, const double* b, int64_t count, double* out,
                          sfb_stream_t stream);

/* hadamard_row_sum (kernel.py:251-266): product (rows, n) -> out (rows),
 * summed in numpy's order (sequential for n < 8, 8-lane pairwise for n >= 8),
 * so the result is bitwise equal to ndarray.sum(axis=-1). */
int sfb_hadamard_row_sum(const double* product, int64_t rows, int64_t n, double* out,
                         sfb_stream_t stream);

/* ---- fused batched Hadamard + row-sum + direction-sum (configs 1-2) ----
 * out_dir[e,j,R] = sum_l basis[j,R,l] * F[e,j,R,l]   (hadamard_evaluate +
 *                  hadamard_row_sum, kernel.py:244,264)
 * out_sum[e,R]   = sum_j out_dir[e,j,R]              (burgers.py:131 sum(axis=0))
 * Products rounded separately and summed in the reference's order, so both
 * outputs are bitwise equal to the reference's numpy pipeline.  basis
 * (d,R,n) shared by all elements, F (E,d,R,n).  Either output may be NULL. */
int sfb_hadamard_rowsum_batched(int64_t E, int64_t m, int64_t n, int64_t d, const double* basis,
                                const double* F, double* out_dir, double* out_sum,
                                sfb_stream_t stream);

/* ---- scalar Burgers flux differencing (burgers.py:117-131) -------------
 * out[e,r] = -(2/omega_r) sum_j sum_k Q_j[r,k] f(u_r, u_k), evaluated as
 * -(2/omega_r) * sum_j (hadamard row sum of direction j); qfactors is the
 * assembled (d, n^d, n) basis factor set of Q = W D (burgers.py:87-97),
 * omega (n^d) the tensor-product weights.  u (E, n^d) -> out (E, n^d). */
int sfb_burgers_volume(int64_t E, int64_t n, int64_t d, const double* qfactors,
                       const double* omega, int flux, const double* u, double* out,
                       sfb_stream_t stream);

/* ---- periodic Burgers time derivative (burgers.py:134-162) -------------
 * dudt = volume term (as sfb_burgers_volume) + the periodic interface term of
 * _surface_residual (burgers.py:134-156): per direction, in order, right-face
 * nodes -= (f*(u_R,u_L) - u_R^2/2)/w[n-1], left-face nodes
 * += (f*(u_R,u_L) - u_L^2/2)/w[0]; w0 = w[0], wn = w[n-1] of the GLL rule.
 * Bitwise equal to the reference's time_derivative.  flux: BURGERS_EC/AVG. */
int sfb_burgers_time_derivative(int64_t E, int64_t n, int64_t d, const double* qfactors,
                                const double* omega, double w0, double wn, int flux,
                                const double* u, double* dudt, sfb_stream_t stream);

/* ---- RK4 time integration of a batch of periodic Burgers elements ------
 * (demos/burgers_entropy.py:25-33, classic RK4 on time_derivative), `steps`
 * steps of size dt, all in ONE launch (one CTA per element, n^d <= 1024);
 * u (E, n^d) is advanced in place, bitwise equal to the reference's
 * trajectory.  Monitors every `every` steps, before the step (step 0, every,
 * ..., incl. `steps` when divisible): entropy[e, k] = 0.5 sum_r omega_r u_r^2
 * (burgers.py:165-169) and mass[e, k] = sum_r omega_r u_r, each
 * (E, steps/every + 1), fixed-order sums; either may be NULL (every = 0: no
 * monitors). */
int sfb_burgers_rk4(int64_t E, int64_t n, int64_t d, const double* qfactors, const double* omega,
                    double w0, double wn, int flux, double dt, int64_t steps, int64_t every,
                    double* u, double* entropy, double* mass, sfb_stream_t stream);

/* ---- sum-factorized Kronecker apply (operators.py:274-318) -------------
 * y[b] = (A_{d-1} x ... x A_0) x[b] for a batch of B vectors; factors is a
 * packed array of d dense (rows_j, cols_j) matrices (direction 0 first);
 * a diagonal factor is passed as a dense diagonal matrix.  x (B, prod cols),
 * y (B, prod rows).  d <= 3, rows_j, cols_j <= 16. */
int sfb_kronecker_apply(int64_t B, int64_t d, const int64_t* rows_1d, const int64_t* cols_1d,
                        const double* factors, const double* x, double* y, sfb_stream_t stream);

/* Same, from/to HOST buffers (the config-2 end-to-end call): basis_host
 * (d,R,n) is uploaded once, F_host (E,d,R,n) streams in and out_sum_host
 * (E,R) streams out over element chunks, pipelined on internal streams of the
 * current device; returns when out_sum_host is complete. */
int sfb_hadamard_rowsum_batched_host(int64_t E, int64_t m, int64_t n, int64_t d,
                                     const double* basis_host, const double* F_host,
                                     double* out_sum_host);

/* ---- the reference's dense route (oracle.py) and general Kronecker passes --
 * All device pointers; every entry of the dense matrices is formed (zeros
 * included) with the reference's product order, so results are bitwise equal.
 *
 * dense_kronecker: out (prod rows, prod cols) = reduce(kron, reversed(factors))
 *   (oracle.py:39-51); factor j (rows_1d[j] x cols_1d[j], row-major) packed
 *   consecutively in `packed` (a diagonal factor passed as its dense diag).
 * dense_direction_factor: out (m n^(d-1), n^d) zeroed, then the basis (m,n)
 *   in slot `direction` times the ascending weight product (oracle.py:54-92).
 * dense_rank_one: out (R, C) = row_values[i] col_values[j] (oracle.py:111-124).
 * scatter_direction / gather_direction: direction `direction` of a compressed
 *   factor (entries values) to / from its dense (row_space, column_space)
 *   matrix through the pattern's (entries, d) rows/columns (oracle.py:127-160);
 *   scatter zeroes `out` first.
 * kronecker_pass: one direction of kronecker_apply (operators.py:274-318) for
 *   any extents: y[b][h][r][a] = sum_c A[r][c] x[b][h][c][a] (a < lo, h < hi),
 *   or y = A[r] x[...r...] when diag (A of length rows == cols). */
int sfb_dense_kronecker(int64_t d, const int64_t* rows_1d, const int64_t* cols_1d,
                        const double* packed, double* out, sfb_stream_t stream);
int sfb_dense_direction_factor(int64_t m, int64_t n, int64_t d, int64_t direction,
                               const double* basis, const double* weights, double* out,
                               sfb_stream_t stream);
int sfb_dense_rank_one(const double* row_values, int64_t R, const double* col_values, int64_t C,
                       double* out, sfb_stream_t stream);
int sfb_scatter_direction(const int64_t* rows, const int64_t* columns, int64_t d,
                          int64_t direction, int64_t entries, const double* values,
                          int64_t row_space, int64_t column_space, double* out,
                          sfb_stream_t stream);
int sfb_gather_direction(const int64_t* rows, const int64_t* columns, int64_t d,
                         int64_t direction, int64_t entries, const double* dense,
                         int64_t column_space, double* values, sfb_stream_t stream);
int sfb_kronecker_pass(int64_t B, int64_t lo, int64_t rows, int64_t cols, int64_t hi, int diag,
                       const double* A, const double* x, double* y, sfb_stream_t stream);

/* ---- 3-D compressible Euler, Chandrashekar flux, Cartesian (configs 3-4) ---
 * R[e,v,r] = scale * sum_j sum_l D[r_j,l] F#_j(U[e,:,r], U[e,:,r(j->l)])_v
 * with F#_j the Chandrashekar entropy-conservative two-point flux (DESIGN.md
 * "Flux"), logarithmic means by the shared series/log formula.  The volume
 * term of burgers.py:117-131 generalised to a 5-variable state; scale = 2
 * gives the 2 sum_j D o F# of BASELINE.json config 3.  n in 2..8.
 * D: HOST (n,n).  U, R: device, (E,5,n^3), 16-byte aligned. */
int sfb_euler_volume_cartesian(int64_t E, int64_t n, const double* D, double gamma, double scale,
                               const double* U, double* R, sfb_stream_t stream);

/* Same with an 8-byte device workspace (8-byte aligned) the call zeroes on
 * `stream`: the persistent kernels of n >= 5 then claim elements from it
 * (dynamic load balance) instead of a static split; bitwise the same
 * results.  NULL = the static split.  Concurrent calls need distinct
 * workspaces. */
int sfb_euler_volume_cartesian_ws(int64_t E, int64_t n, const double* D, double gamma,
                                  double scale, const double* U, double* R, void* workspace,
                                  sfb_stream_t stream);

/* Same, from/to HOST buffers: pipelined H2D / kernel / D2H over element
 * chunks on internal streams of the current device; returns after R_host is
 * complete (also on error: nothing is left in flight on the caller's buffers).
 * Pinned buffers let both copy directions overlap the kernel. */
int sfb_euler_volume_cartesian_host(int64_t E, int64_t n, const double* D_host, double gamma,
                                    double scale, const double* U_host, double* R_host);

/* ---- curvilinear modal Euler (config 5) ---------------------------------
 * u  = (V x V x V) Uhat            (kronecker_apply, operators.py:274-318)
 * r  = scale * sum_i sum_l D[r_i,l] Ft_i(u_r, u_{r(i->l)}),
 *      Ft_i = sum_m 1/2 (Ja[i][m](r) + Ja[i][m](r(i->l))) F#_m
 * Rhat = (Pi x Pi x Pi) r
 * sumsq[e] = sum over v, modes of Rhat[e,v,:]^2 (deterministic order), NULL ok.
 * V, Pi, D: HOST (n,n); Uhat, Rhat (E,5,n^3), Ja (E,3,3,n^3), sumsq (E):
 * device, 16-byte aligned.  n in 2..8.
 * workspace: 8 bytes of device memory (8-byte aligned) the call zeroes on
 * `stream` and uses as the element-claim counter of its persistent CTAs
 * (dynamic load balance); NULL = static element split (same results, bitwise).
 * Concurrent calls need distinct workspaces. */
int sfb_euler_volume_curvilinear_modal(int64_t E, int64_t n, const double* V, const double* Pi,
                                       const double* D, double gamma, double scale,
                                       const double* Uhat, const double* Ja, double* Rhat,
                                       double* sumsq, void* workspace, sfb_stream_t stream);

/* Same, from/to HOST buffers (the config-5 end-to-end call): Uhat_host,
 * Ja_host in, Rhat_host and (if not NULL) sumsq_host out, pipelined over
 * element chunks on internal streams (each with its own claim counter). */
int sfb_euler_volume_curvilinear_modal_host(int64_t E, int64_t n, const double* V,
                                            const double* Pi, const double* D, double gamma,
                                            double scale, const double* Uhat_host,
                                            const double* Ja_host, double* Rhat_host,
                                            double* sumsq_host);

/* Deterministic fixed-order block sums: partial[b] = sum of x[b*block ..
 * b*block+block-1] (pairwise tree, independent of launch geometry).
 * count must be a multiple of block; block a power of two <= 4096. */
int sfb_block_sums(const double* x, int64_t count, int64_t block, double* partial,
                   sfb_stream_t stream);

/* ---- seeded, element-addressable synthetic inputs (bench / tests) -------
 * Counter-based hash (splitmix64) so that any element can be regenerated
 * bit-for-bit on the host (tests/golden, oracle) and on the device.
 * U (E, 5, n^3) conserved states from primitives rho ~ U[rlo,rhi],
 * v_m ~ U[vlo,vhi], p ~ U[plo,phi], gamma; element ids start at e0. */
int sfb_generate_euler_states(int64_t E, int64_t e0, int64_t n, uint64_t seed, double gamma,
                              const double* bounds6, double* U, sfb_stream_t stream);
/* Modal coefficients Uhat (E, 5, n^3) of config 5 (see synth.modal_states):
 * (amps5[v] 2^-(k0+k1+k2)) (2u - 1), plus means5[v] c0 at mode 0. */
int sfb_generate_modal_states(int64_t E, int64_t e0, int64_t n, uint64_t seed,
                              const double* means5, const double* amps5, double c0,
                              double* Uhat, sfb_stream_t stream);
/* Metric cofactors Ja (E, 3, 3, n^3) of the warped K^3 lattice (config 5;
 * synth.metric_cofactors): x = X + amp prod_k sin(2 pi (X_k + phi_mk)),
 * Ja = adj(dx/dxi).  nodes: host GLL nodes (n).  Device sin/cos: equal to the
 * host generator to ~1e-15, not bitwise. */
int sfb_generate_metric(int64_t E, int64_t e0, int64_t n, uint64_t seed, const double* nodes,
                        int64_t K, double amp, double* Ja, sfb_stream_t stream);
/* F (E, d, R, n) entries U[lo,hi] on the pattern (config 2). */
int sfb_generate_uniform(int64_t count, int64_t i0, uint64_t seed, double lo, double hi,
                         double* out, sfb_stream_t stream);

#if defined(__GNUC__)
#pragma GCC visibility pop
#endif
#ifdef __cplusplus
}
#endif

#endif /* SUMFAC_B200_H */
