"""Drop-in completeness on the device: the reference's dense route, general
kronecker_apply, numpy semantics of user callables, live factor-set data, the
batched host-buffer entries and the sumfac-bench harness.

Golden vectors: tests/golden/dense.npz, produced by the reference itself
(make_golden.py make_dense): dense_kronecker / dense_direction_factor /
dense_rank_one_operand / scatter (oracle.py:39-160) and kronecker_apply beyond
d = 3 or extents 16 (operators.py:274-318).
"""

import io

import numpy as np
import pytest
import torch

from conftest import golden, max_rel

pytestmark = pytest.mark.gpu

sf = pytest.importorskip("paper_2306_11665_b200")


def test_dense_route_bitwise_against_reference():
    g = golden("dense.npz")
    for k, (d, m, n) in enumerate(g["dir_cases"]):
        b, w = g[f"dir{k}_basis"], g[f"dir{k}_weights"]
        for j in range(d):
            got = sf.dense_direction_factor(b, w, j, d)
            ref = g[f"dir{k}_out{j}"]
            assert np.array_equal(got, ref) and np.array_equal(np.signbit(got), np.signbit(ref))
        facs = [g[f"kr{k}_f{j}"] for j in range(d)]
        got = sf.dense_kronecker(facs)
        ref = g[f"kr{k}_out"]
        assert np.array_equal(got, ref) and np.array_equal(np.signbit(got), np.signbit(ref))
        rv, cv = g[f"r1{k}_rv"], g[f"r1{k}_cv"]
        assert np.array_equal(sf.dense_rank_one_operand(rv, cv), g[f"r1{k}_out"])
        pattern = sf.build_sparsity_pattern(m, n, d)
        fac = sf.assemble_operand_factors(pattern, sf.TwoPointOperand(cv, row_values=rv))
        for j in range(d):
            dense = sf.scatter(fac.factor(j), pattern, j)
            assert np.array_equal(dense, g[f"sc{k}_out{j}"])
            assert np.array_equal(sf.gather(dense, pattern, j), fac.factor(j))


def test_dense_counts_and_validation():
    sf.reset_multiplication_count()
    a = np.ones((6, 6))
    sf.dense_hadamard(a, a)
    sf.dense_rank_one_operand(np.ones(6), np.ones(6))
    assert sf.multiplication_count() == 72
    out = np.empty((6, 6))
    assert sf.dense_hadamard(a, 2 * a, out=out) is out and np.all(out == 2.0)
    with pytest.raises(ValueError):
        sf.dense_hadamard(np.ones((2, 3)), np.ones((3, 2)))
    with pytest.raises(ValueError):
        sf.dense_kronecker([np.ones((100, 100))] * 2, capacity=10_000)
    with pytest.raises(ValueError):
        sf.dense_kronecker([])
    with pytest.raises(ValueError):
        sf.dense_kronecker([np.ones((2, 2, 2))])
    with pytest.raises(IndexError):
        sf.dense_direction_factor(np.eye(3), np.ones(3), 2, 2)
    p = sf.build_sparsity_pattern(2, 2, 2)
    with pytest.raises(IndexError):
        sf.scatter(np.ones((4, 2)), p, 2)
    with pytest.raises(ValueError):
        sf.gather(np.ones((4, 5)), p, 0)
    assert sf.DEFAULT_CAPACITY == 100_000_000


def test_kronecker_apply_any_d_and_extents():
    g = golden("dense.npz")
    for k in range(int(g["kg_cases"])):
        d = int(g[f"kg{k}_d"])
        facs = [g[f"kg{k}_f{j}"] for j in range(d)]
        got = sf.kronecker_apply(facs, g[f"kg{k}_v"])
        assert max_rel(got, g[f"kg{k}_y"]) <= 1e-13


def test_custom_two_point_func_gets_numpy():
    # the reference calls func with numpy arrays (kernel.py:226-229); np.size,
    # np.where and friends must work, and the call happens once per assembly
    calls = []

    def f(a, b):
        assert isinstance(a, np.ndarray) and isinstance(b, np.ndarray)
        calls.append(np.size(a))
        return np.where(a > b, a * b, a + b)

    n, d = 4, 3
    p = sf.build_sparsity_pattern(n, n, d)
    u = np.linspace(0.5, 1.5, n**d)
    fac = sf.assemble_operand_factors(p, sf.TwoPointOperand(u, func=f))
    assert calls == [p.entry_count * d]
    a, b = u[p.rows], u[p.columns]
    ref = np.ascontiguousarray(np.where(a > b, a * b, a + b).T).reshape(d, -1, n)
    assert np.array_equal(fac.data, ref)
    # and it flows through the device stages
    basis = sf.assemble_basis_factors(p, np.eye(n), np.ones(n))
    prod = sf.hadamard_evaluate(basis, fac)
    assert np.array_equal(prod.data, basis.data * ref)


def test_factor_set_mutation_is_seen_by_later_stages():
    n, d = 3, 2
    p = sf.build_sparsity_pattern(n, n, d)
    basis = sf.assemble_basis_factors(p, np.ones((n, n)), np.ones(n))
    ops = sf.assemble_operand_factors(p, sf.TwoPointOperand(np.arange(1.0, 10.0)))
    first = sf.hadamard_evaluate(basis, ops).data.copy()
    ops.data[0] *= 2.0  # in place, through the numpy array the reference exposes
    second = sf.hadamard_evaluate(basis, ops).data
    assert np.array_equal(second[0], 2.0 * first[0]) and np.array_equal(second[1], first[1])
    ops.factor(1)[:] = 0.0  # through a factor view
    assert np.all(sf.hadamard_evaluate(basis, ops).data[1] == 0.0)
    ops.data = np.ones_like(ops.data)  # reassignment
    assert np.array_equal(sf.hadamard_evaluate(basis, ops).data, basis.data)
    rows = sf.hadamard_row_sum(sf.hadamard_evaluate(basis, ops), p)
    assert np.array_equal(rows, basis.data.sum(axis=2))


def test_batched_hadamard_host_entry_bitwise():
    n, d, E = 4, 3, 1000
    D = sf.lagrange_diff_matrix(sf.gauss_lobatto_legendre(n))
    basis = sf.assemble_basis_factors(sf.build_sparsity_pattern(n, n, d), D, np.ones(n))
    F = np.random.default_rng(3).uniform(-1, 1, (E, d, 64, n))
    got = sf.kernel.hadamard_rowsum_batched_host(basis, F)
    ref = (basis.data[None] * F).sum(axis=3).sum(axis=1)
    assert np.array_equal(got, ref)
    dev = sf.kernel.hadamard_rowsum_batched(basis, torch.from_numpy(F).cuda())
    assert np.array_equal(dev.cpu().numpy(), ref)


def test_modal_host_entry_equals_device_path():
    from paper_2306_11665_b200 import euler as eu

    n, E = 6, 37
    Uh = eu.generate_modal_states(E, n, seed=5)
    Ja = eu.generate_metric(E, n, seed=6)
    ss = torch.empty(E, dtype=torch.float64, device="cuda")
    Rd = eu.volume_curvilinear_modal(Uh, Ja, n, sumsq=ss)
    Uh_h, Ja_h = Uh.cpu(), Ja.cpu()
    ss_h = torch.empty(E, dtype=torch.float64)
    Rh = eu.volume_curvilinear_modal_host(Uh_h, Ja_h, n, sumsq=ss_h)
    assert torch.equal(Rh, Rd.cpu()) and torch.equal(ss_h, ss.cpu())


def test_bench_harness_csv_and_gate(tmp_path, monkeypatch):
    from paper_2306_11665_b200 import bench

    cfg = bench.BenchConfig(d=3, n_min=3, n_max=3, repetitions=2)
    recs = bench.run_benchmark(cfg)
    assert len(recs) == 4
    for r in recs:
        assert r.elapsed_s > 0
        assert r.mul_count == (3 * 3**4 if r.method == "sumfac" else 3 * 3**6)
    recs += bench.run_benchmark(bench.BenchConfig(d=3, n_min=4, n_max=6, repetitions=1,
                                                  methods=("batched",)))
    path = tmp_path / "r.csv"
    bench.emit_csv(recs, path)
    assert bench.read_csv(path) == sorted(recs, key=lambda r: (r.d, r.n, r.method, r.rep))
    assert path.read_text().splitlines()[0] == "d,n,method,rep,elapsed_s,mul_count,timestamp"
    assert bench.main(["--dim", "2", "--n-min", "3", "--n-max", "3", "--reps", "1",
                       "--methods", "sumfac,batched", "--out", str(path)]) == 0
    assert bench.main(["--methods", "sparse"]) == 1
    monkeypatch.setattr(bench, "GATE_RTOL", -1.0)
    with pytest.raises(bench.CorrectnessGateError, match="row-sum"):
        bench.run_benchmark(bench.BenchConfig(d=3, n_min=7, n_max=7, repetitions=1,
                                              methods=("sumfac",)))
    assert bench.main(["--dim", "2", "--n-min", "3", "--n-max", "3", "--reps", "1"]) == 2


def test_bench_entropy_demo():
    from paper_2306_11665_b200 import bench

    out = io.StringIO()
    assert bench.run_entropy_demo(seed=3, states_per_case=2, stream=out)
    assert "entropy d=3 n=6" in out.getvalue() and "FAIL" not in out.getvalue()
