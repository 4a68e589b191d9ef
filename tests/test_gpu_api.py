"""Drop-in API behaviour: the reference's exception types and invariants.

The product package must fail like sumfac 0.1.0 does (kernel.py:84-92,
185-188, 200-217, 239-243, 258-263; burgers.py:56-71, 104-108): ValueError
for bad extents / shapes / non-finite values / foreign objects, IndexError for
a bad direction, read-only pattern arrays, and the same simple identities
(identity basis, ones operand, vanishing row sums of D).
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

sf = pytest.importorskip("paper_2306_11665_b200")


@pytest.mark.parametrize("m,n,d", [(0, 4, 3), (4, 0, 3), (4, 4, 0), (-1, 2, 2), (3, 2**33, 3)])
def test_pattern_bad_extents_raise_value_error(m, n, d):
    with pytest.raises(ValueError):
        sf.build_sparsity_pattern(m, n, d)


def test_pattern_arrays_read_only_and_direction_checked():
    p = sf.build_sparsity_pattern(3, 2, 2)
    with pytest.raises(ValueError):
        p.columns[1, 0] = 7
    f = sf.assemble_basis_factors(p, np.ones((3, 2)), np.ones(2))
    with pytest.raises(IndexError):
        f.factor(2)


def test_basis_assembly_shape_checks():
    p = sf.build_sparsity_pattern(4, 4, 3)
    with pytest.raises(ValueError):
        sf.assemble_basis_factors(p, np.eye(3), np.ones(4))
    with pytest.raises(ValueError):
        sf.assemble_basis_factors(p, np.eye(4), np.ones(5))
    with pytest.raises(ValueError):
        sf.assemble_basis_factors(None, np.eye(4), np.ones(4))


def test_operand_checks():
    p = sf.build_sparsity_pattern(2, 2, 3)
    with pytest.raises(ValueError):
        sf.TwoPointOperand(np.array([0.5, np.inf]))
    with pytest.raises(ValueError):
        sf.TwoPointOperand(np.zeros((3, 3)))
    with pytest.raises(ValueError):
        sf.assemble_operand_factors(p, sf.TwoPointOperand(np.ones(7)))
    with pytest.raises(ValueError):
        sf.assemble_operand_factors(p, np.ones(8))
    op = sf.TwoPointOperand(np.array([1.5, 4.0]))
    assert op.is_rank_one
    assert op.evaluate(1, 0) == op.evaluate(0, 1) == 6.0


def test_hadamard_and_row_sum_reject_foreign_factor_sets():
    pa, pb = sf.build_sparsity_pattern(2, 2, 3), sf.build_sparsity_pattern(3, 3, 3)
    basis = sf.assemble_basis_factors(pa, np.eye(2), np.ones(2))
    with pytest.raises(ValueError):
        sf.hadamard_evaluate(basis, sf.assemble_operand_factors(pb, sf.TwoPointOperand(np.ones(27))))
    prod = sf.hadamard_evaluate(basis, sf.assemble_operand_factors(pa, sf.TwoPointOperand(np.ones(8))))
    with pytest.raises(ValueError):
        sf.hadamard_row_sum(prod, pb)


def test_identities():
    for d, n in [(1, 4), (2, 2), (3, 3)]:
        p = sf.build_sparsity_pattern(n, n, d)
        ident = sf.assemble_basis_factors(p, np.eye(n), np.ones(n))
        ones = sf.assemble_operand_factors(p, sf.TwoPointOperand(np.ones(n**d)))
        assert np.array_equal(ones.data, np.ones_like(ones.data))
        prod = sf.hadamard_evaluate(ident, ones)
        assert np.array_equal(prod.data, ident.data)
        assert np.array_equal(sf.hadamard_row_sum(prod, p), np.ones((d, n**d)))
        # rows of a differentiation matrix sum to zero: so do the row sums of D o 1
        D = sf.lagrange_diff_matrix(sf.gauss_lobatto_legendre(n))
        dprod = sf.hadamard_evaluate(sf.assemble_basis_factors(p, D, np.ones(n)), ones)
        assert np.abs(sf.hadamard_row_sum(dprod, p)).max() <= 1e-13


def test_burgers_state_validation_and_flux_values():
    assert sf.ec_two_point_flux(1.0, 2.0) == pytest.approx(7.0 / 6.0, rel=0, abs=1e-16)
    with pytest.raises(ValueError):
        sf.BurgersState(0, 3, np.ones(1))
    with pytest.raises(ValueError):
        sf.BurgersState(2, 3, np.ones(8))
    with pytest.raises(ValueError):
        sf.BurgersState(1, 3, np.array([0.0, np.nan, 1.0]))
    st = sf.BurgersState(2, 3, np.ones(9), rule=sf.gauss_legendre(3))
    with pytest.raises(ValueError):  # flux differencing needs Lobatto nodes
        sf.volume_residual(st)
    # a constant state is steady; the zero state has zero entropy rate
    const = sf.BurgersState(3, 3, np.full(27, 0.7))
    assert np.abs(sf.time_derivative(const)).max() <= 1e-14
    assert sf.entropy_time_derivative(sf.BurgersState(2, 4, np.zeros(16))) == 0.0


def test_c_program_through_the_host_abi(tmp_path):
    """A plain C11 program (tests/c_abi/host_call.c) calls the host-buffer entry
    sfb_euler_volume_cartesian_host; its checksum equals the Python device path's
    on the same inputs and operator."""
    import os
    import subprocess

    import torch

    from conftest import ROOT
    from paper_2306_11665_b200 import _lib
    from paper_2306_11665_b200 import euler as eu

    exe = tmp_path / "host_call"
    libdir = os.path.dirname(_lib.LIB_PATH)
    subprocess.run(["gcc", "-std=c11", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "c_abi", "host_call.c"), "-o", str(exe), "-L",
                    libdir, "-lsumfac_b200", f"-Wl,-rpath,{libdir}"], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split()
    assert out[0] == "ok"
    checksum = float(out[2])
    E, n, nodes = 3, 4, 64
    D = np.array([-3.0, 4.04508497187474, -1.54508497187474, 0.5,
                  -0.809016994374947, 0.0, 1.11803398874989, -0.309016994374947,
                  0.309016994374947, -1.11803398874989, 0.0, 0.809016994374947,
                  -0.5, 1.54508497187474, -4.04508497187474, 3.0]).reshape(4, 4)
    U = np.zeros((E, 5, nodes))
    for e in range(E):
        for r in range(nodes):
            rho = 1.0 + 0.01 * ((r * 7 + e) % 11)
            U[e, 0, r], U[e, 1, r] = rho, rho * 0.05
            U[e, 4, r] = 1.0 / 0.4 + 0.5 * rho * 0.05 * 0.05
    R = eu.volume_cartesian(torch.from_numpy(U).cuda(), n, D=D).cpu().numpy()
    ref = float((R * R).sum())
    assert abs(checksum - ref) <= 1e-12 * ref
