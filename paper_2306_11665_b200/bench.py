"""sumfac-bench on the B200: the reference's scaling benchmark with device methods.

Drop-in for ``sumfac.bench`` (sumfac/bench.py:71-468): the same
configuration object, records, CSV schema ``d,n,method,rep,elapsed_s,
mul_count,timestamp``, correctness gate, slope fit, entropy demo and CLI exit
codes (1 bad configuration, 2 gate failure, 3 I/O error).  What differs is
where the timed work runs:

  sumfac   the sum-factorized pipeline of one element (basis assembly,
           operand assembly, Hadamard evaluation) through this package's
           device kernels, synchronised at the end of the region;
  dense    the O(n^{2d}) route with device-resident dense factors and
           buffers: the rank-one operand matrix and d entrywise products
           (csrc/dense.cu, sfb_hadamard_evaluate), synchronised;
  batched  (B200 addition, not in the default set) the fused batched kernel
           (hadamard + row sum + direction sum, sfb_hadamard_rowsum_batched)
           over ~2^24 stored entries; elapsed_s is the time per element.

Single-element regions on a GPU are launch-latency-bound, so their fitted
slopes are not the CPU's O(n^{d+1}) / O(n^{2d}) exponents; the batched
method is the one whose time follows the work.  Every point is gated before
it is timed: scatter of the product against the dense route up to
DENSE_GATE_MAX_N, the rank-one row-sum identity (K_j o c c^T) 1 = c (K_j c)
above it (bench.py:134-164).
"""

import argparse
import csv
import sys
import time
import warnings
from dataclasses import dataclass
from datetime import datetime, timezone

import numpy as np
import torch

from . import _lib, counting
from .burgers import BurgersState, average_flux, entropy_time_derivative, time_derivative, \
    total_entropy
from .dense import (DEFAULT_CAPACITY, dense_direction_factor, dense_hadamard,
                    dense_rank_one_operand, scatter)
from .kernel import (TwoPointOperand, assemble_basis_factors, assemble_operand_factors,
                     build_sparsity_pattern, hadamard_evaluate, hadamard_row_sum,
                     hadamard_rowsum_batched)
from .operators import gauss_legendre, kronecker_apply, lagrange_diff_matrix, \
    tensor_product_weights

METHODS = ("dense", "sumfac")
ALL_METHODS = METHODS + ("batched",)
CSV_FIELDS = ("d", "n", "method", "rep", "elapsed_s", "mul_count", "timestamp")
DENSE_GATE_MAX_N = 6
GATE_RTOL = 1e-13
BATCH_ENTRIES = 1 << 24


class CorrectnessGateError(Exception):
    """A benchmark point failed its pre-check against the dense route; nothing was timed."""


@dataclass
class BenchConfig:
    """Sweep settings (bench.py:71-102); validate() raises ValueError."""

    d: int = 3
    n_min: int = 3
    n_max: int = 15
    repetitions: int = 5
    seed: int = 0
    methods: tuple = METHODS
    low: float = 1e-8
    high: float = 30.0
    include_pattern: bool = False

    def validate(self):
        checks = (
            (self.d >= 1, f"d must be >= 1, got {self.d}"),
            (1 <= self.n_min <= self.n_max,
             f"need 1 <= n_min <= n_max, got [{self.n_min}, {self.n_max}]"),
            (self.repetitions >= 1, f"repetitions must be >= 1, got {self.repetitions}"),
            (len(self.methods) > 0, "at least one method is required"),
        )
        for ok, msg in checks:
            if not ok:
                raise ValueError(msg)
        unknown = [m for m in self.methods if m not in ALL_METHODS]
        if unknown:
            raise ValueError(f"unknown method {unknown[0]!r}, expected one of {ALL_METHODS}")
        if not (np.isfinite(self.low) and np.isfinite(self.high)):
            raise ValueError("operand bounds must be finite")
        if self.low > self.high:
            raise ValueError(f"need low <= high, got [{self.low}, {self.high}]")


@dataclass
class BenchRecord:
    """One timed repetition of one (d, n, method) point."""

    d: int
    n: int
    method: str
    rep: int
    elapsed_s: float
    mul_count: int
    timestamp: str


def _operand_vector(config, n):
    """The point's rank-one generator c, seeded by (seed, d, n) as in the reference."""
    return np.random.default_rng((config.seed, config.d, n)).uniform(
        config.low, config.high, n**config.d)


def _rel(got, ref):
    peak = float(np.max(np.abs(ref)))
    diff = float(np.max(np.abs(np.asarray(got) - ref)))
    return diff if peak == 0.0 else diff / peak


class _Point:
    """Everything one sweep size needs: operators, pattern, generator, device buffers."""

    def __init__(self, config, n):
        self.config, self.n, self.d = config, n, config.d
        self.c = _operand_vector(config, n)
        self.diff = lagrange_diff_matrix(gauss_legendre(n))
        self.weights = np.ones(n)
        self.pattern = build_sparsity_pattern(n, n, self.d)

    # ---- gate ---------------------------------------------------------------
    def gate(self):
        d, n, pattern = self.d, self.n, self.pattern
        product = hadamard_evaluate(
            assemble_basis_factors(pattern, self.diff, self.weights),
            assemble_operand_factors(pattern, TwoPointOperand(self.c)))
        tol = GATE_RTOL  # module global, read per call (tests patch it)
        if n <= DENSE_GATE_MAX_N:
            cc = dense_rank_one_operand(self.c, self.c)
            for j in range(d):
                ref = dense_hadamard(dense_direction_factor(self.diff, self.weights, j, d), cc)
                err = _rel(scatter(product.factor(j), pattern, j), ref)
                if err > tol:
                    raise CorrectnessGateError(
                        f"sum-factorized product deviates from the dense route at n={n}, "
                        f"direction {j}: relative error {err:.3e}")
            return
        sums = hadamard_row_sum(product, pattern)
        for j in range(d):
            slots = [self.weights] * d
            slots[j] = self.diff
            err = _rel(sums[j], self.c * kronecker_apply(slots, self.c))
            if err > tol:
                raise CorrectnessGateError(
                    f"row-sum self-consistency check failed at n={n}, direction {j}: "
                    f"relative error {err:.3e}")

    # ---- timed regions (each returns the evaluation-stage multiplications) --
    def sumfac(self, operand):
        pattern = self.pattern
        if self.config.include_pattern:
            pattern = build_sparsity_pattern(self.n, self.n, self.d)
        basis = assemble_basis_factors(pattern, self.diff, self.weights)
        factors = assemble_operand_factors(pattern, operand)
        before = counting.multiplication_count()
        hadamard_evaluate(basis, factors)
        used = counting.multiplication_count() - before
        torch.cuda.synchronize()
        return used

    def dense_setup(self, capacity):
        size = self.n**self.d
        if size * size > capacity:
            warnings.warn(f"skipping dense at n={self.n}: {size * size} entries exceed the "
                          f"capacity cap of {capacity}", stacklevel=3)
            return False
        self.dense_factors = [
            torch.from_numpy(dense_direction_factor(self.diff, self.weights, j, self.d,
                                                    capacity)).cuda()
            for j in range(self.d)]
        # operand and product buffers live outside the timed region, like the
        # reference's scratch arrays (bench.py:246-250)
        self.cc = torch.empty((size, size), dtype=torch.float64, device="cuda")
        self.prod = torch.empty_like(self.cc)
        self.dc = torch.from_numpy(self.c).cuda()
        return True

    def dense(self):
        size = self.n**self.d
        _lib.call("sfb_dense_rank_one", _lib.ptr(self.dc), size, _lib.ptr(self.dc), size,
                  _lib.ptr(self.cc), _lib.stream_ptr())
        counting.add_multiplications(size * size)
        before = counting.multiplication_count()
        for f in self.dense_factors:
            _lib.call("sfb_hadamard_evaluate", _lib.ptr(f), _lib.ptr(self.cc), f.numel(),
                      _lib.ptr(self.prod), _lib.stream_ptr())
            counting.add_multiplications(f.numel())
        used = counting.multiplication_count() - before
        torch.cuda.synchronize()
        return used

    def batched_setup(self):
        d, n = self.d, self.n
        per = d * n ** (d + 1)
        self.E = max(1, BATCH_ENTRIES // per)
        basis = assemble_basis_factors(self.pattern, self.diff, self.weights)
        self.B = basis.device
        rng = np.random.default_rng((self.config.seed, d, n, 1))
        F = rng.uniform(self.config.low, self.config.high, (min(self.E, 64),) + self.B.shape)
        self.F = torch.from_numpy(F).cuda().repeat((self.E + 63) // 64, 1, 1, 1)[:self.E]
        self.F = self.F.contiguous()
        self.out = torch.empty((self.E, self.B.shape[1]), dtype=torch.float64, device="cuda")

    def batched(self):
        hadamard_rowsum_batched(self.B, self.F, out=self.out)
        torch.cuda.synchronize()
        return self.d * self.n ** (self.d + 1)


def _stamp():
    return datetime.now(timezone.utc).isoformat(timespec="microseconds")


def _repeat(reps, region, per=1):
    out = []
    for _ in range(reps):
        t0 = time.perf_counter()
        region()
        out.append((time.perf_counter() - t0) / per)
    return out


def run_benchmark(config, capacity=DEFAULT_CAPACITY):
    """Gate and time every (n, method); one BenchRecord per repetition.

    Dense points over the capacity cap are skipped with a warning.  One
    warm-up per point is discarded and reads the multiplication count.
    """
    config.validate()
    _lib.require_cuda()
    records = []
    for n in range(config.n_min, config.n_max + 1):
        pt = _Point(config, n)
        pt.gate()
        for method in config.methods:
            if method == "sumfac":
                operand = TwoPointOperand(pt.c)
                muls = pt.sumfac(operand)
                times = _repeat(config.repetitions, lambda: pt.sumfac(operand))
            elif method == "dense":
                if not pt.dense_setup(capacity):
                    continue
                muls = pt.dense()
                times = _repeat(config.repetitions, pt.dense)
            else:
                pt.batched_setup()
                muls = pt.batched()
                times = _repeat(config.repetitions, pt.batched, per=pt.E)
            records.extend(BenchRecord(config.d, n, method, rep, t, muls, _stamp())
                           for rep, t in enumerate(times))
    return records


def median_timings(records, method):
    """{n: median elapsed seconds} for one method."""
    by_n = {}
    for r in records:
        if r.method == method:
            by_n.setdefault(r.n, []).append(r.elapsed_s)
    return {n: float(np.median(v)) for n, v in sorted(by_n.items())}


def fit_slope(records, method):
    """Least-squares slope of log(median time) on log(n); needs >= 3 sizes."""
    med = median_timings(records, method)
    if len(med) < 3:
        raise ValueError(f"slope fit needs at least 3 distinct sizes for {method!r}, "
                         f"got {len(med)}")
    ns = np.array(sorted(med), dtype=float)
    return float(np.polyfit(np.log(ns), np.log([med[int(n)] for n in ns]), 1)[0])


def emit_csv(records, path):
    """Records as CSV sorted by (d, n, method, rep); floats at repr precision."""
    rows = sorted(records, key=lambda r: (r.d, r.n, r.method, r.rep))
    with open(path, "w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(CSV_FIELDS)
        w.writerows([r.d, r.n, r.method, r.rep, repr(r.elapsed_s), r.mul_count, r.timestamp]
                    for r in rows)


def read_csv(path):
    """Parse emit_csv output back into BenchRecord objects (exact floats)."""
    with open(path, newline="") as fh:
        rd = csv.DictReader(fh)
        if tuple(rd.fieldnames or ()) != CSV_FIELDS:
            raise ValueError(f"unexpected CSV header {rd.fieldnames}, expected {list(CSV_FIELDS)}")
        return [BenchRecord(int(x["d"]), int(x["n"]), x["method"], int(x["rep"]),
                            float(x["elapsed_s"]), int(x["mul_count"]), x["timestamp"])
                for x in rd]


def _mass_rate(state):
    omega = tensor_product_weights(state.rule.weights, state.d)
    return float(np.dot(omega, time_derivative(state)))


def run_entropy_demo(seed=0, states_per_case=20, stream=None):
    """Entropy-conservation spot check over d = 1..3, n = 3..6 (bench.py:348-382):
    the EC flux keeps |dS/dt| <= 1e-12 (1 + |S|) and the mass rate <= 1e-12 on
    every random state; the average flux breaks it (> 1e-6) on >= 95 % of them."""
    out = sys.stdout if stream is None else stream
    rng = np.random.default_rng(seed)
    passed = True
    for d in (1, 2, 3):
        for n in (3, 4, 5, 6):
            ec = mass = 0.0
            broken = 0
            for _ in range(states_per_case):
                st = BurgersState(d, n, rng.uniform(-1.0, 1.0, n**d))
                ec = max(ec, abs(entropy_time_derivative(st)) / (1.0 + abs(total_entropy(st))))
                mass = max(mass, abs(_mass_rate(st)))
                broken += abs(entropy_time_derivative(st, average_flux)) > 1e-6
            frac = broken / states_per_case
            ok = ec <= 1e-12 and mass <= 1e-12 and frac >= 0.95
            passed = passed and ok
            print(f"entropy d={d} n={n}: |dS/dt|/(1+|S|) <= {ec:.2e}, mass rate <= {mass:.2e}, "
                  f"control broken on {frac:.0%} [{'ok' if ok else 'FAIL'}]", file=out)
    return passed


class _Parser(argparse.ArgumentParser):
    # bad flags exit 1 (argparse's own 2 is reserved for gate failures)
    def error(self, message):
        self.print_usage(sys.stderr)
        print(f"{self.prog}: error: {message}", file=sys.stderr)
        raise SystemExit(1)


def _build_parser():
    p = _Parser(prog="sumfac-bench",
                description="Sum-factorized vs dense Hadamard products on the B200.")
    p.add_argument("--dim", type=int, default=3, help="tensor dimension d")
    p.add_argument("--n-min", type=int, default=3, help="smallest 1D size")
    p.add_argument("--n-max", type=int, default=15, help="largest 1D size")
    p.add_argument("--reps", type=int, default=5, help="timed repetitions per point")
    p.add_argument("--seed", type=int, default=0, help="operand RNG seed")
    p.add_argument("--methods", default="dense,sumfac",
                   help="comma-separated subset of: dense, sumfac, batched")
    p.add_argument("--out", default=None, help="write raw records to this CSV")
    p.add_argument("--include-pattern", action="store_true",
                   help="move sparsity-pattern construction inside the timed region")
    p.add_argument("--low", type=float, default=1e-8, help="operand lower bound")
    p.add_argument("--high", type=float, default=30.0, help="operand upper bound")
    p.add_argument("--demo-entropy", action="store_true",
                   help="run the entropy-conservation demo instead of the sweep")
    return p


def _summary(config, records, out):
    for method in config.methods:
        med = median_timings(records, method)
        if not med:
            print(f"{method}: no timed points", file=out)
            continue
        print(f"{method}:", file=out)
        for n, t in med.items():
            print(f"  n={n:3d}  median {t:.6e} s", file=out)
        try:
            print(f"  fitted log-log slope: {fit_slope(records, method):.3f}", file=out)
        except ValueError:
            print("  slope: not enough sizes to fit", file=out)


def main(argv=None):
    a = _build_parser().parse_args(argv)
    if a.demo_entropy:
        return 0 if run_entropy_demo(seed=a.seed) else 2
    config = BenchConfig(d=a.dim, n_min=a.n_min, n_max=a.n_max, repetitions=a.reps, seed=a.seed,
                         methods=tuple(m.strip() for m in a.methods.split(",") if m.strip()),
                         low=a.low, high=a.high, include_pattern=a.include_pattern)
    try:
        config.validate()
    except ValueError as exc:
        print(f"invalid configuration: {exc}", file=sys.stderr)
        return 1
    try:
        records = run_benchmark(config)
    except CorrectnessGateError as exc:
        print(f"correctness gate failed: {exc}", file=sys.stderr)
        return 2
    _summary(config, records, sys.stdout)
    if a.out is not None:
        try:
            emit_csv(records, a.out)
        except OSError as exc:
            print(f"could not write {a.out}: {exc}", file=sys.stderr)
            return 3
        print(f"wrote {len(records)} records to {a.out}")
    return 0


if __name__ == "__main__":
    raise SystemExit(main())
