"""Generate the golden fixtures in tests/golden/ from the REFERENCE itself.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It copies /root/reference/pkg to a scratch directory (numba's cache=True would
otherwise write into the read-only reference tree), imports `sumfac` 0.1.0
from there, and records reference outputs for the hot path on seeded inputs
from paper_2306_11665_b200.synth (pure functions of a seed, so the GPU box can
regenerate the same inputs without the reference):

  operators.npz        GL / GLL nodes+weights, D, V, dV, Pi, interpolation, omega
  patterns.npz         build_sparsity_pattern rows/columns for several (m, n, d)
  config1.npz          2-D n=5 (A x I) o C: 125 stored nonzeros + 25 row sums,
                       and the dense O(n^4) evaluation
  config2.npz          3-D generic Hadamard, n=4: sample elements, per-element
                       hadamard_evaluate + hadamard_row_sum + direction sum
  euler_cartesian.npz  Chandrashekar volume term through the reference's
                       assemble_operand_factors / hadamard_evaluate /
                       hadamard_row_sum (index-trick operand), n = 2..8
  burgers.npz          volume_residual / time_derivative for seeded states
  kron.npz             kronecker_apply on seeded factor sets
  euler_modal.npz      config 5: V^3 -> contravariant Chandrashekar volume term
                       -> Pi^3 through kronecker_apply + the index-trick route
  dense.npz            the dense route (dense_kronecker, dense_direction_factor,
                       dense_rank_one_operand, scatter, gather) and
                       kronecker_apply beyond d = 3 / extents 16
  python tests/golden/make_golden.py dense   regenerates one fixture only
Only tests read these files; nothing on the GPU box reads /root/reference.
"""

import os
import shutil
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import euler_oracle  # noqa: E402
from paper_2306_11665_b200 import synth  # noqa: E402

REF_PKG = "/root/reference/pkg"


def import_reference():
    scratch = tempfile.mkdtemp(prefix="refpkg_")
    shutil.copytree(REF_PKG, os.path.join(scratch, "pkg"))
    os.environ.setdefault("NUMBA_CACHE_DIR", os.path.join(scratch, "numba_cache"))
    sys.dont_write_bytecode = True
    sys.path.insert(0, os.path.join(scratch, "pkg", "src"))
    import sumfac  # noqa: F401

    return sumfac


def make_operators(sf):
    out = {}
    for n in range(1, 11):
        gl = sf.gauss_legendre(n)
        out[f"gl{n}_nodes"] = gl.nodes
        out[f"gl{n}_weights"] = gl.weights
        out[f"gl{n}_D"] = sf.lagrange_diff_matrix(gl)
        out[f"gl{n}_V"] = sf.legendre_vandermonde(gl)
        out[f"gl{n}_dV"] = sf.legendre_vandermonde_derivative(gl)
        out[f"gl{n}_Pi"] = sf.projection_operator(gl)
        if n >= 2:
            gll = sf.gauss_lobatto_legendre(n)
            out[f"gll{n}_nodes"] = gll.nodes
            out[f"gll{n}_weights"] = gll.weights
            out[f"gll{n}_D"] = sf.lagrange_diff_matrix(gll)
            out[f"gll{n}_V"] = sf.legendre_vandermonde(gll)
            out[f"gll{n}_dV"] = sf.legendre_vandermonde_derivative(gll)
            out[f"gll{n}_Pi"] = sf.projection_operator(gll)
            for d in (1, 2, 3):
                out[f"gll{n}_omega{d}"] = sf.tensor_product_weights(gll.weights, d)
        for m in range(1, n):
            out[f"interp{n}_{m}"] = sf.lagrange_interpolation_matrix(
                gl.nodes, sf.gauss_legendre(m).nodes
            )
    np.savez_compressed(os.path.join(HERE, "operators.npz"), **out)


PATTERN_CASES = [(1, 1, 3), (2, 2, 2), (3, 3, 3), (4, 4, 3), (5, 5, 2), (2, 4, 3), (3, 2, 4),
                 (6, 4, 2), (8, 8, 3), (1, 5, 3), (4, 3, 1)]


def make_patterns(sf):
    out = {}
    for m, n, d in PATTERN_CASES:
        p = sf.build_sparsity_pattern(m, n, d)
        out[f"rows_{m}_{n}_{d}"] = np.asarray(p.rows)
        out[f"cols_{m}_{n}_{d}"] = np.asarray(p.columns)
    np.savez_compressed(os.path.join(HERE, "patterns.npz"), **out)


def config1_inputs():
    A = synth.uniform_array(25, 11, -1.0, 1.0).reshape(5, 5)
    C = synth.uniform_array(625, 12, -1.0, 1.0).reshape(25, 25)
    return A, C


def make_config1(sf):
    A, C = config1_inputs()
    n, d = 5, 2
    pattern = sf.build_sparsity_pattern(n, n, d)
    basis = sf.assemble_basis_factors(pattern, A, np.ones(n))  # slot j carries A
    operand = sf.SparseFactorSet(
        n, n, np.stack([sf.gather(C, pattern, j) for j in range(d)])
    )
    product = sf.hadamard_evaluate(basis, operand)
    sums = sf.hadamard_row_sum(product, pattern)
    # the paper's A (x) B with B = I_5: A in direction 1 (slow), I in direction 0
    stored = product.factor(1)
    dense = sf.dense_hadamard(sf.dense_kronecker([np.ones(n), A]), C)
    np.savez_compressed(
        os.path.join(HERE, "config1.npz"), A=A, C=C, stored=stored, row_sums=sums[1],
        dense=dense, dense_row_sums=dense @ np.ones(n * n),
        scatter=sf.scatter(stored, pattern, 1),
    )


CONFIG2_SAMPLE = 48


def make_config2(sf):
    n, d = 4, 3
    D = sf.lagrange_diff_matrix(sf.gauss_lobatto_legendre(n))
    pattern = sf.build_sparsity_pattern(n, n, d)
    basis = sf.assemble_basis_factors(pattern, D, np.ones(n))
    per = d * n ** (d + 1)
    F = synth.uniform_array(CONFIG2_SAMPLE * per, 2, -1.0, 1.0).reshape(CONFIG2_SAMPLE, d, n**d, n)
    out_dir = np.empty((CONFIG2_SAMPLE, d, n**d))
    out_sum = np.empty((CONFIG2_SAMPLE, n**d))
    for e in range(CONFIG2_SAMPLE):
        product = sf.hadamard_evaluate(basis, sf.SparseFactorSet(n, n, F[e].copy()))
        sums = sf.hadamard_row_sum(product, pattern)
        out_dir[e] = sums
        out_sum[e] = sums.sum(axis=0)
    np.savez_compressed(
        os.path.join(HERE, "config2.npz"), basis=basis.data, F=F, out_dir=out_dir,
        out_sum=out_sum, seed=2,
    )


def reference_euler_volume(sf, U, D, gamma=1.4, scale=2.0):
    """The volume term through the reference's own machinery (index trick).

    TwoPointOperand(arange(n^3), func=g): g receives (entries, d) arrays of
    row / column node indices, column j being direction j, and returns the
    restated flux component v in direction j at those pairs.
    """
    n = D.shape[0]
    d = 3
    pattern = sf.build_sparsity_pattern(n, n, d)
    basis = sf.assemble_basis_factors(pattern, D, np.ones(n))
    E = U.shape[0]
    R = np.empty_like(U)
    for e in range(E):
        rho, v, p, beta, vv = euler_oracle.primitives(U[e], gamma)
        for var in range(5):

            def g(ri, ci, var=var):
                ri = ri.astype(np.int64)
                ci = ci.astype(np.int64)
                out = np.empty(ri.shape)
                for j in range(d):
                    a = (rho[ri[:, j]], [vm[ri[:, j]] for vm in v], p[ri[:, j]],
                         beta[ri[:, j]], vv[ri[:, j]])
                    b = (rho[ci[:, j]], [vm[ci[:, j]] for vm in v], p[ci[:, j]],
                         beta[ci[:, j]], vv[ci[:, j]])
                    normal = [1.0 if m == j else 0.0 for m in range(3)]
                    out[:, j] = euler_oracle.chandrashekar(a, b, normal, gamma)[var]
                return out

            operand = sf.TwoPointOperand(np.arange(n**d, dtype=float), func=g)
            product = sf.hadamard_evaluate(basis, sf.assemble_operand_factors(pattern, operand))
            sums = sf.hadamard_row_sum(product, pattern)
            R[e, var] = scale * sums.sum(axis=0)
    return R


EULER_SAMPLE = {2: 6, 3: 5, 4: 4, 5: 3, 6: 2, 7: 2, 8: 2}


def make_euler(sf):
    out = {}
    for n, E in EULER_SAMPLE.items():
        D = sf.lagrange_diff_matrix(sf.gauss_lobatto_legendre(n))
        U = synth.euler_states(E, n, seed=3 + n)
        out[f"U{n}"] = U
        out[f"D{n}"] = D
        out[f"R{n}"] = reference_euler_volume(sf, U, D)
    np.savez_compressed(os.path.join(HERE, "euler_cartesian.npz"), **out)


BURGERS_CASES = [(1, 3), (1, 6), (2, 4), (2, 5), (3, 3), (3, 4), (3, 6), (2, 9)]


def make_burgers(sf):
    out = {}
    for d, n in BURGERS_CASES:
        u = synth.uniform_array(n**d, 100 + 10 * d + n, -1.0, 1.0)
        st = sf.BurgersState(d, n, u)
        out[f"u_{d}_{n}"] = u
        out[f"vol_ec_{d}_{n}"] = sf.volume_residual(st)
        out[f"vol_avg_{d}_{n}"] = sf.volume_residual(st, sf.average_flux)
        out[f"dudt_{d}_{n}"] = sf.time_derivative(st)
        out[f"dudt_avg_{d}_{n}"] = sf.time_derivative(st, sf.average_flux)
        out[f"dsdt_{d}_{n}"] = np.array(sf.entropy_time_derivative(st))
        out[f"dsdt_avg_{d}_{n}"] = np.array(sf.entropy_time_derivative(st, sf.average_flux))
        out[f"entropy_{d}_{n}"] = np.array(sf.total_entropy(st))
    np.savez_compressed(os.path.join(HERE, "burgers.npz"), **out)


def reference_rk4(sf, d, n, u, dt, steps, flux, every):
    """demos/burgers_entropy.py:25-51 verbatim in structure: classic RK4 on the
    reference's time_derivative, entropy sampled before every `every` steps."""

    def rhs(v):
        return sf.time_derivative(sf.BurgersState(d, n, v), flux)

    trace = []
    for step in range(steps + 1):
        if step % every == 0:
            trace.append(sf.total_entropy(sf.BurgersState(d, n, u)))
        if step == steps:
            break
        k1 = rhs(u)
        k2 = rhs(u + 0.5 * dt * k1)
        k3 = rhs(u + 0.5 * dt * k2)
        k4 = rhs(u + dt * k3)
        u = u + dt / 6.0 * (k1 + 2 * k2 + 2 * k3 + k4)
    return u, np.array(trace)


RK4_CASES = [(2, 5, 2e-3, 40, 10), (1, 6, 1e-3, 30, 10), (3, 4, 2e-3, 12, 4)]


def make_burgers_rk4(sf):
    out = {}
    for d, n, dt, steps, every in RK4_CASES:
        u0 = synth.uniform_array(n**d, 300 + 10 * d + n, -1.0, 1.0)
        out[f"u0_{d}_{n}"] = u0
        for name, flux in (("ec", sf.ec_two_point_flux), ("avg", sf.average_flux)):
            u, trace = reference_rk4(sf, d, n, u0.copy(), dt, steps, flux, every)
            out[f"u_{name}_{d}_{n}"] = u
            out[f"entropy_{name}_{d}_{n}"] = trace
    np.savez_compressed(os.path.join(HERE, "burgers_rk4.npz"), **out)


def make_kron(sf):
    out = {}
    case = 0
    for d in (1, 2, 3):
        for n in (2, 3, 4, 5, 6):
            factors = []
            kinds = []
            for j in range(d):
                if (case + j) % 4 == 3:
                    f = synth.uniform_array(n, 500 + case * 8 + j, -1.0, 1.0)
                    kinds.append(1)
                else:
                    f = synth.uniform_array(n * n, 500 + case * 8 + j, -1.0, 1.0).reshape(n, n)
                    kinds.append(2)
                factors.append(f)
                out[f"c{case}_f{j}"] = f
            v = synth.uniform_array(n**d, 900 + case, -1.0, 1.0)
            out[f"c{case}_v"] = v
            out[f"c{case}_y"] = sf.kronecker_apply(factors, v)
            out[f"c{case}_meta"] = np.array([d, n] + kinds)
            case += 1
    out["cases"] = np.array(case)
    np.savez_compressed(os.path.join(HERE, "kron.npz"), **out)


MODAL_SAMPLE = {6: 3, 4: 3, 3: 2}


def reference_curvilinear_modal(sf, Uhat, Ja, n, gamma=1.4, scale=2.0):
    """Config 5 through the reference's own machinery: kronecker_apply for the
    modal <-> nodal transforms (operators.py:274-318) and the index-trick
    Hadamard route for the contravariant flux (kernel.py:195-266)."""
    rule = sf.gauss_lobatto_legendre(n)
    D = sf.lagrange_diff_matrix(rule)
    V = sf.legendre_vandermonde(rule)
    Pi = sf.projection_operator(rule, V)
    d = 3
    pattern = sf.build_sparsity_pattern(n, n, d)
    basis = sf.assemble_basis_factors(pattern, D, np.ones(n))
    E = Uhat.shape[0]
    Rhat = np.empty_like(Uhat)
    for e in range(E):
        u = np.stack([sf.kronecker_apply([V, V, V], Uhat[e, v]) for v in range(5)])
        rho, vel, p, beta, vv = euler_oracle.primitives(u, gamma)
        r = np.empty_like(u)
        for var in range(5):

            def g(ri, ci, var=var):
                ri = ri.astype(np.int64)
                ci = ci.astype(np.int64)
                out = np.empty(ri.shape)
                for j in range(d):
                    a = (rho[ri[:, j]], [vm[ri[:, j]] for vm in vel], p[ri[:, j]],
                         beta[ri[:, j]], vv[ri[:, j]])
                    b = (rho[ci[:, j]], [vm[ci[:, j]] for vm in vel], p[ci[:, j]],
                         beta[ci[:, j]], vv[ci[:, j]])
                    normal = [0.5 * (Ja[e, j, m][ri[:, j]] + Ja[e, j, m][ci[:, j]])
                              for m in range(3)]
                    out[:, j] = euler_oracle.chandrashekar(a, b, normal, gamma)[var]
                return out

            operand = sf.TwoPointOperand(np.arange(n**d, dtype=float), func=g)
            product = sf.hadamard_evaluate(basis, sf.assemble_operand_factors(pattern, operand))
            r[var] = scale * sf.hadamard_row_sum(product, pattern).sum(axis=0)
        Rhat[e] = np.stack([sf.kronecker_apply([Pi, Pi, Pi], r[v]) for v in range(5)])
    return Rhat


def make_modal(sf):
    out = {}
    for n, E in MODAL_SAMPLE.items():
        Uhat = synth.modal_states(E, n, seed=50 + n)
        Ja = synth.metric_cofactors(E, n, seed=60 + n, e0=12345)
        out[f"Uhat{n}"] = Uhat
        out[f"Ja{n}"] = Ja
        out[f"Rhat{n}"] = reference_curvilinear_modal(sf, Uhat, Ja, n)
    np.savez_compressed(os.path.join(HERE, "euler_modal.npz"), **out)


DENSE_DIR_CASES = [(1, 3, 3), (2, 3, 4), (2, 2, 3), (3, 4, 4), (3, 2, 5)]  # (d, m, n)
KRON_GENERAL_CASES = [((3, 3, 3, 3), (3, 3, 3, 3), (2, 2, 2, 2)),  # extents, rows, kinds
                      ((20, 17), (18, 21), (2, 2)),
                      ((2, 2, 2, 2, 2), (2, 2, 2, 2, 2), (2, 1, 2, 1, 2)),
                      ((5, 4, 3, 2), (2, 3, 4, 5), (2, 2, 2, 2))]


def make_dense(sf):
    out = {}
    for k, (d, m, n) in enumerate(DENSE_DIR_CASES):
        b = synth.uniform_array(m * n, 700 + k, -1.0, 1.0).reshape(m, n)
        w = synth.uniform_array(n, 720 + k, 0.5, 1.5)
        out[f"dir{k}_basis"], out[f"dir{k}_weights"] = b, w
        for j in range(d):
            out[f"dir{k}_out{j}"] = sf.dense_direction_factor(b, w, j, d)
        # a Kronecker product mixing dense and diagonal slots
        facs = [b if j % 2 == 0 else w for j in range(d)]
        for j, f in enumerate(facs):
            out[f"kr{k}_f{j}"] = f
        out[f"kr{k}_out"] = sf.dense_kronecker(facs)
        rv = synth.uniform_array(m * n ** (d - 1), 740 + k, -2.0, 2.0)
        cv = synth.uniform_array(n**d, 760 + k, -2.0, 2.0)
        out[f"r1{k}_rv"], out[f"r1{k}_cv"] = rv, cv
        out[f"r1{k}_out"] = sf.dense_rank_one_operand(rv, cv)
        pattern = sf.build_sparsity_pattern(m, n, d)
        fac = sf.assemble_operand_factors(pattern, sf.TwoPointOperand(cv, row_values=rv))
        for j in range(d):
            out[f"sc{k}_out{j}"] = sf.scatter(fac.factor(j), pattern, j)
    out["dir_cases"] = np.array(DENSE_DIR_CASES)
    for k, (cols, rows, kinds) in enumerate(KRON_GENERAL_CASES):
        facs = []
        for j, (r, c, kind) in enumerate(zip(rows, cols, kinds)):
            if kind == 1:
                facs.append(synth.uniform_array(c, 800 + 10 * k + j, -1.0, 1.0))
            else:
                facs.append(synth.uniform_array(r * c, 800 + 10 * k + j, -1.0, 1.0).reshape(r, c))
            out[f"kg{k}_f{j}"] = facs[-1]
        v = synth.uniform_array(int(np.prod(cols)), 880 + k, -1.0, 1.0)
        out[f"kg{k}_v"] = v
        out[f"kg{k}_y"] = sf.kronecker_apply(facs, v)
        out[f"kg{k}_d"] = np.array(len(cols))
    out["kg_cases"] = np.array(len(KRON_GENERAL_CASES))
    np.savez_compressed(os.path.join(HERE, "dense.npz"), **out)


TARGETS = {
    "operators": make_operators, "patterns": make_patterns, "config1": make_config1,
    "config2": make_config2, "euler": make_euler, "burgers": make_burgers,
    "burgers_rk4": make_burgers_rk4, "kron": make_kron, "modal": make_modal, "dense": make_dense,
}


def main(argv=None):
    names = (sys.argv[1:] if argv is None else argv) or list(TARGETS)
    sf = import_reference()
    for name in names:
        TARGETS[name](sf)
    print("golden fixtures written to", HERE, names)


if __name__ == "__main__":
    main()
