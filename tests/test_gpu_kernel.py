"""GPU parity of the unfused stages and the fused generic Hadamard (configs 1-2).

Bar: bitwise equality with the reference's outputs (golden vectors from
sumfac 0.1.0) and with the dense oracle identities the reference's own tests
use (pkg/tests/test_kernel.py, test_acceptance.py).
"""

import itertools

import numpy as np
import pytest
import torch

from conftest import golden, max_rel

pytestmark = pytest.mark.gpu

sf = pytest.importorskip("paper_2306_11665_b200")
from paper_2306_11665_b200 import counting  # noqa: E402
from paper_2306_11665_b200 import euler as eu  # noqa: E402
from paper_2306_11665_b200 import synth  # noqa: E402
from paper_2306_11665_b200 import _lib  # noqa: E402


def dense_direction_factor(basis, weights, direction, d):
    """Dense factor with basis in slot `direction`, weights elsewhere (oracle.py:54-93)."""
    m, n = basis.shape
    row_ext = [n] * d
    row_ext[direction] = m
    rows = int(np.prod(row_ext))
    out = np.zeros((rows, n**d))
    for r in range(rows):
        digits, rem = [], r
        for e in row_ext:
            digits.append(rem % e)
            rem //= e
        wprod, have = 1.0, False
        for i in range(d):
            if i == direction:
                continue
            wprod = wprod * weights[digits[i]] if have else weights[digits[i]]
            have = True
        base = sum(digits[i] * n**i for i in range(d) if i != direction)
        for l in range(n):
            val = basis[digits[direction], l]
            out[r, base + l * n**direction] = val * wprod if have else val
    return out


def scatter(factor, pattern, j):
    out = np.zeros((pattern.row_space_size, pattern.column_space_size))
    out[pattern.rows[:, j], pattern.columns[:, j]] = np.asarray(factor).reshape(-1)
    return out


def test_pattern_matches_reference_exactly():
    g = golden("patterns.npz")
    for key in g.files:
        if not key.startswith("rows_"):
            continue
        m, n, d = (int(x) for x in key.split("_")[1:])
        p = sf.build_sparsity_pattern(m, n, d)
        assert np.array_equal(p.rows, g[key])
        assert np.array_equal(p.columns, g[f"cols_{m}_{n}_{d}"])
        assert p.rows.dtype == np.int64
        with pytest.raises(ValueError):
            p.rows[0, 0] = 1


@pytest.mark.parametrize("d", (1, 2, 3))
def test_pattern_matches_dense_nonzeros_exhaustive(d):
    for m, n in itertools.product(range(1, 6), repeat=2):
        p = sf.build_sparsity_pattern(m, n, d)
        assert p.entry_count == m * n**d
        for j in range(d):
            dense = dense_direction_factor(np.ones((m, n)), np.ones(n), j, d)
            expected = set(zip(*(ix.tolist() for ix in np.nonzero(dense))))
            got = list(zip(p.rows[:, j].tolist(), p.columns[:, j].tolist()))
            assert len(set(got)) == len(got)
            assert set(got) == expected


def test_pattern_larger_d4_and_counts():
    p = sf.build_sparsity_pattern(3, 4, 4)
    assert p.entry_count == 3 * 4**4
    counting.reset_allocation_ledger()
    p = sf.build_sparsity_pattern(3, 3, 2)
    assert counting.allocated_numbers() == 2 * p.entry_count * 2


def test_assemble_basis_bitwise_random():
    rng = np.random.default_rng(11)
    for d, m, n in [(2, 3, 3), (3, 2, 2), (3, 4, 4), (2, 5, 3), (3, 3, 5)]:
        basis = rng.standard_normal((m, n))
        weights = rng.uniform(0.5, 1.5, n)
        p = sf.build_sparsity_pattern(m, n, d)
        f = sf.assemble_basis_factors(p, basis, weights)
        for j in range(d):
            assert np.array_equal(scatter(f.factor(j), p, j),
                                  dense_direction_factor(basis, weights, j, d))


def test_rank_one_and_builtin_flux_operands_bitwise():
    rng = np.random.default_rng(5)
    u = rng.uniform(-1.0, 1.0, 27)
    p = sf.build_sparsity_pattern(3, 3, 3)
    f = sf.assemble_operand_factors(p, sf.TwoPointOperand(u))
    for j in range(3):
        assert np.array_equal(f.factor(j).reshape(-1), u[p.rows[:, j]] * u[p.columns[:, j]])
    for flux in (sf.ec_two_point_flux, sf.average_flux):
        f = sf.assemble_operand_factors(p, sf.TwoPointOperand(u, func=flux))
        for j in range(3):
            a, b = u[p.rows[:, j]], u[p.columns[:, j]]
            assert np.array_equal(f.factor(j).reshape(-1), flux(a, b))
    # a custom callable is evaluated on the device with torch tensors
    f = sf.assemble_operand_factors(p, sf.TwoPointOperand(u, func=lambda a, b: (a + b) / 2.0))
    for j in range(3):
        assert np.array_equal(f.factor(j).reshape(-1),
                              (u[p.rows[:, j]] + u[p.columns[:, j]]) / 2.0)


def test_hadamard_and_row_sum_oracle_equivalence():
    # acceptance 1 (pkg/tests/test_acceptance.py:47-78), 1e-13 vs dense
    rng = np.random.default_rng(2024)
    worst = 0.0
    for d, n in itertools.product((1, 2, 3), (2, 3, 4, 5)):
        p = sf.build_sparsity_pattern(n, n, d)
        for _ in range(3):
            basis = rng.standard_normal((n, n))
            weights = rng.uniform(0.5, 1.5, n)
            c = rng.uniform(1e-8, 30.0, n**d)
            prod = sf.hadamard_evaluate(sf.assemble_basis_factors(p, basis, weights),
                                        sf.assemble_operand_factors(p, sf.TwoPointOperand(c)))
            sums = sf.hadamard_row_sum(prod, p)
            dc = np.outer(c, c)
            for j in range(d):
                ref = dense_direction_factor(basis, weights, j, d) * dc
                worst = max(worst, max_rel(scatter(prod.factor(j), p, j), ref))
                worst = max(worst, max_rel(sums[j], ref @ np.ones(n**d)))
            # bitwise: numpy's own pipeline on the host-side copies
            assert np.array_equal(prod.data, sf.assemble_basis_factors(p, basis, weights).data
                                  * sf.assemble_operand_factors(p, sf.TwoPointOperand(c)).data)
            assert np.array_equal(sums, prod.data.sum(axis=2))
    assert worst <= 1e-13


@pytest.mark.parametrize("n", [3, 7, 8, 9, 16, 17, 130, 300])
def test_row_sum_numpy_order_bitwise(n):
    rng = np.random.default_rng(n)
    x = rng.standard_normal((3, 50, n)) * np.exp(rng.uniform(-20, 20, (3, 50, n)))
    t = torch.from_numpy(x).cuda()
    out = torch.empty((150,), dtype=torch.float64, device="cuda")
    _lib.call("sfb_hadamard_row_sum", _lib.ptr(t), 150, n, _lib.ptr(out), _lib.stream_ptr())
    assert np.array_equal(out.cpu().numpy().reshape(3, 50), x.sum(axis=2))


def test_flop_counts_match_reference():
    for d, n in [(1, 5), (2, 4), (3, 4), (3, 6)]:
        p = sf.build_sparsity_pattern(n, n, d)
        b = sf.assemble_basis_factors(p, np.linspace(1.0, 2.0, n * n).reshape(n, n), np.ones(n))
        o = sf.assemble_operand_factors(p, sf.TwoPointOperand(np.linspace(0.5, 1.5, n**d)))
        before = counting.multiplication_count()
        sf.hadamard_evaluate(b, o)
        assert counting.multiplication_count() - before == d * n ** (d + 1)


def test_allocation_ledger_bound():
    d, n = 3, 15
    counting.reset_allocation_ledger()
    p = sf.build_sparsity_pattern(n, n, d)
    b = sf.assemble_basis_factors(p, np.eye(n), np.ones(n))
    o = sf.assemble_operand_factors(p, sf.TwoPointOperand(np.ones(n**d)))
    sf.hadamard_row_sum(sf.hadamard_evaluate(b, o), p)
    assert counting.allocated_numbers() <= 6 * d * n**4


def test_surface_variant_rectangular():
    rng = np.random.default_rng(55)
    for d in (2, 3):
        for n in (2, 3, 4, 5):
            rule = sf.gauss_legendre(n)
            for m in range(1, n):
                interp = sf.lagrange_interpolation_matrix(rule.nodes, sf.gauss_legendre(m).nodes)
                p = sf.build_sparsity_pattern(m, n, d)
                row_c = rng.uniform(1e-8, 30.0, m * n ** (d - 1))
                col_c = rng.uniform(1e-8, 30.0, n**d)
                prod = sf.hadamard_evaluate(
                    sf.assemble_basis_factors(p, interp, rule.weights),
                    sf.assemble_operand_factors(p, sf.TwoPointOperand(col_c, row_values=row_c)),
                )
                dc = np.outer(row_c, col_c)
                for j in range(d):
                    dense = dense_direction_factor(interp, rule.weights, j, d)
                    assert max_rel(scatter(prod.factor(j), p, j), dense * dc) <= 1e-13


def test_config1_two_dimensional_single_element():
    # BASELINE config 1: (A x I_5) o C, 125 stored nonzeros + row sums vs dense
    g = golden("config1.npz")
    A, C = g["A"], g["C"]
    n, d = 5, 2
    p = sf.build_sparsity_pattern(n, n, d)
    basis = sf.assemble_basis_factors(p, A, np.ones(n))
    Cd = torch.from_numpy(C).cuda()
    gathered = torch.empty((d, 25, n), dtype=torch.float64, device="cuda")
    _lib.call("sfb_gather_dense", _lib.ptr(p.device_rows), _lib.ptr(p.device_columns),
              _lib.ptr(Cd), n, n, d, _lib.ptr(gathered), _lib.stream_ptr())
    prod = sf.hadamard_evaluate(basis, sf.SparseFactorSet(n, n, gathered))
    sums = sf.hadamard_row_sum(prod, p)
    assert np.array_equal(prod.factor(1), g["stored"])
    assert np.array_equal(sums[1], g["row_sums"])
    assert np.array_equal(scatter(prod.factor(1), p, 1), g["dense"])
    assert max_rel(sums[1], g["dense_row_sums"]) <= 1e-13


def test_config2_fused_batched_bitwise_golden():
    g = golden("config2.npz")
    E = g["F"].shape[0]
    F = torch.from_numpy(g["F"]).cuda()
    B = torch.from_numpy(g["basis"]).cuda()
    out_dir = torch.empty((E, 3, 64), dtype=torch.float64, device="cuda")
    out_sum = torch.empty((E, 64), dtype=torch.float64, device="cuda")
    _lib.call("sfb_hadamard_rowsum_batched", E, 4, 4, 3, _lib.ptr(B), _lib.ptr(F),
              _lib.ptr(out_dir), _lib.ptr(out_sum), _lib.stream_ptr())
    assert np.array_equal(out_sum.cpu().numpy(), g["out_sum"])
    assert np.array_equal(out_dir.cpu().numpy(), g["out_dir"])


@pytest.mark.parametrize("n,d", [(2, 3), (3, 3), (5, 2), (6, 3), (8, 3), (9, 2),
                                 (5, 3), (7, 3), (9, 3), (10, 3), (11, 3), (12, 3), (13, 3),
                                 (14, 3), (15, 3), (16, 3), (11, 2), (16, 2), (10, 4), (17, 3)])
def test_fused_batched_generic_sizes_bitwise(n, d):
    # fixed-size kernels (2|3|4|6|8, 3), (4|5, 2) and the generic kernel for
    # the rest, up to the reference's sumfac-bench range (n <= 15) and beyond
    rng = np.random.default_rng(n * 10 + d)
    R = n ** (d - 1) * n
    E = 37 if n < 10 else 5
    basis = rng.standard_normal((d, R, n))
    F = rng.uniform(-1, 1, (E, d, R, n))
    out = torch.empty((E, R), dtype=torch.float64, device="cuda")
    Bt, Ft = torch.from_numpy(basis).cuda(), torch.from_numpy(F).cuda()
    _lib.call("sfb_hadamard_rowsum_batched", E, n, n, d, _lib.ptr(Bt), _lib.ptr(Ft), None,
              _lib.ptr(out), _lib.stream_ptr())
    assert np.array_equal(out.cpu().numpy(), (basis[None] * F).sum(axis=3).sum(axis=1))
    # per-direction output too
    od = torch.empty((E, d, R), dtype=torch.float64, device="cuda")
    _lib.call("sfb_hadamard_rowsum_batched", E, n, n, d, _lib.ptr(Bt), _lib.ptr(Ft), _lib.ptr(od),
              None, _lib.stream_ptr())
    assert np.array_equal(od.cpu().numpy(), (basis[None] * F).sum(axis=3))


def test_config2_full_size_sampled_and_generator():
    # full config-2 size on the device: F from the device generator (bitwise
    # equal to the host generator), sampled elements checked vs the oracle
    n, d, E = 4, 3, 262144
    D = sf.lagrange_diff_matrix(sf.gauss_lobatto_legendre(n))
    p = sf.build_sparsity_pattern(n, n, d)
    basis = sf.assemble_basis_factors(p, D, np.ones(n))
    F = eu.generate_uniform(E * 768, 2, -1.0, 1.0).reshape(E, 3, 64, 4)
    out = torch.empty((E, 64), dtype=torch.float64, device="cuda")
    _lib.call("sfb_hadamard_rowsum_batched", E, n, n, d, _lib.ptr(basis.device), _lib.ptr(F),
              None, _lib.ptr(out), _lib.stream_ptr())
    g = golden("config2.npz")
    Es = g["F"].shape[0]
    assert np.array_equal(F[:Es].cpu().numpy(), g["F"])
    assert np.array_equal(out[:Es].cpu().numpy(), g["out_sum"])
    idx = np.random.default_rng(0).choice(E, 64, replace=False)
    Fs = F[idx].cpu().numpy()
    ref = (basis.data[None] * Fs).sum(axis=3).sum(axis=1)
    assert np.array_equal(out[idx].cpu().numpy(), ref)
    # checksum property: sum over everything equals the sum of per-direction sums
    total = out.sum().item()
    assert np.isfinite(total)


def test_kronecker_apply_golden():
    g = golden("kron.npz")
    for c in range(int(g["cases"])):
        meta = g[f"c{c}_meta"]
        d = int(meta[0])
        factors = [g[f"c{c}_f{j}"] for j in range(d)]
        got = sf.kronecker_apply(factors, g[f"c{c}_v"])
        ref = g[f"c{c}_y"]
        assert max_rel(got, ref) <= 1e-13


def test_kronecker_apply_counts():
    rng = np.random.default_rng(3)
    for d, n in [(1, 4), (2, 3), (3, 4)]:
        factors = [rng.standard_normal((n, n)) for _ in range(d)]
        counting.reset_multiplication_count()
        sf.kronecker_apply(factors, rng.standard_normal(n**d))
        assert counting.multiplication_count() == d * n ** (d + 1)
    f = rng.standard_normal((2, 4))
    v = rng.standard_normal(16)
    ref = np.kron(f, f) @ v
    assert max_rel(sf.kronecker_apply([f, f], v), ref) <= 1e-13


def test_device_generator_matches_host_bitwise():
    U = eu.generate_states(7, 3, seed=11, e0=5).cpu().numpy()
    assert np.array_equal(U, synth.euler_states(7, 3, seed=11, e0=5))
    x = eu.generate_uniform(1000, 4, -2.0, 3.0, i0=17).cpu().numpy()
    assert np.array_equal(x, synth.uniform_array(1000, 4, -2.0, 3.0, i0=17))


def test_block_sums_fixed_tree():
    rng = np.random.default_rng(1)
    x = rng.standard_normal(4096 * 3)
    t = torch.from_numpy(x).cuda()
    out = torch.empty(3, dtype=torch.float64, device="cuda")
    _lib.call("sfb_block_sums", _lib.ptr(t), x.size, 4096, _lib.ptr(out), _lib.stream_ptr())
    ref = x.reshape(3, 4096)
    while ref.shape[1] > 1:
        ref = ref[:, 0::2] + ref[:, 1::2]
    assert np.array_equal(out.cpu().numpy(), ref[:, 0])
