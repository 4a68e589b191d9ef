"""Seeded inputs and reference operators for the CPU arms (TEST INFRASTRUCTURE ONLY).

bench.py's reference arm (--impl reference) and its cpu_baseline legs build
their inputs here without importing the product package, so that no process
timing the CPU reference ever maps libsumfac_b200.so:

  * the seeded generators are the pure-numpy module
    paper_2306_11665_b200/synth.py loaded BY FILE PATH (the workload
    definition shared with the device generators; importing it as part of the
    package would run the package __init__ and load the CUDA library);
  * the 1-D operators (D, V, Pi, nodes) are the reference's own outputs,
    recorded by tests/golden/make_golden.py from sumfac 0.1.0
    (tests/golden/operators.npz: gauss_lobatto_legendre / lagrange_diff_matrix /
    legendre_vandermonde / projection_operator, operators.py:96-232).
"""

import importlib.util
import os

import numpy as np

_ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
_synth = None
_ops = None


def synth():
    global _synth
    if _synth is None:
        spec = importlib.util.spec_from_file_location(
            "_sfb_workload_synth", os.path.join(_ROOT, "paper_2306_11665_b200", "synth.py"))
        mod = importlib.util.module_from_spec(spec)
        spec.loader.exec_module(mod)
        _synth = mod
    return _synth


def gll_operators(n):
    """(nodes, D, V, Pi) of the n-point GLL rule as the reference computed them."""
    global _ops
    if _ops is None:
        _ops = dict(np.load(os.path.join(_ROOT, "tests", "golden", "operators.npz")))
    return tuple(np.ascontiguousarray(_ops[f"gll{n}_{k}"]) for k in ("nodes", "D", "V", "Pi"))


def config2_basis(n=4, d=3):
    """B_j[R,l] = D[r_j, l] (assemble_basis_factors with weights ones, _kernels.py:43-76)."""
    D = gll_operators(n)[1]
    r = np.arange(n**d)
    return np.ascontiguousarray(np.stack([D[(r // n**j) % n] for j in range(d)]))


def loaded_native_libraries():
    """Shared objects of this repository mapped into the current process."""
    root = os.path.realpath(_ROOT)
    out = set()
    try:
        with open("/proc/self/maps") as f:
            for line in f:
                path = line.split()[-1] if len(line.split()) >= 6 else ""
                if path.endswith(".so") and os.path.realpath(path).startswith(root):
                    out.add(os.path.relpath(os.path.realpath(path), root))
    except OSError:
        pass
    return sorted(out)
