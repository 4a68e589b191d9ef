"""Small invocation of every kernel, for compute-sanitizer runs (one tool per call)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2306_11665_b200 as sf  # noqa: E402
from paper_2306_11665_b200 import _lib, shard  # noqa: E402
from paper_2306_11665_b200 import euler as eu  # noqa: E402

for n in (2, 3, 4, 5, 6, 7, 8):
    U = eu.generate_states(9, n, seed=1)
    eu.volume_cartesian(U, n)
for n in (3, 4, 6):
    Uh = eu.generate_modal_states(5, n, seed=2)
    Ja = eu.generate_metric(5, n, seed=3)
    ss = torch.empty(5, dtype=torch.float64, device="cuda")
    eu.volume_curvilinear_modal(Uh, Ja, n, sumsq=ss)
p = sf.build_sparsity_pattern(3, 4, 3)
b = sf.assemble_basis_factors(p, np.ones((3, 4)), np.ones(4))
o = sf.assemble_operand_factors(p, sf.TwoPointOperand(np.ones(64), row_values=np.ones(48)))
sf.hadamard_row_sum(sf.hadamard_evaluate(b, o), p)
D = sf.lagrange_diff_matrix(sf.gauss_lobatto_legendre(4))
p4 = sf.build_sparsity_pattern(4, 4, 3)
basis = sf.assemble_basis_factors(p4, D, np.ones(4))
F = eu.generate_uniform(7 * 768, 2, -1.0, 1.0).reshape(7, 3, 64, 4)
out = torch.empty((7, 64), dtype=torch.float64, device="cuda")
_lib.call("sfb_hadamard_rowsum_batched", 7, 4, 4, 3, _lib.ptr(basis.device), _lib.ptr(F), None,
          _lib.ptr(out), _lib.stream_ptr())
sf.volume_residual(sf.BurgersState(3, 4, np.linspace(-1, 1, 64)))
sf.kronecker_apply([np.eye(3), np.ones((2, 3)), np.ones(3)], np.ones(27))
shard.global_norm(torch.rand(4096 * 2, dtype=torch.float64, device="cuda"), block=4096)
eu.volume_cartesian_host(eu.generate_states(5, 4, seed=4).cpu().numpy(), 4)
# round-2 entry points: dynamic claims, dense route, general Kronecker passes, host entries
for n in (5, 6, 7, 8):
    eu.volume_cartesian(eu.generate_states(11, n, seed=5), n, dynamic=True)
sf.dense_kronecker([np.ones((2, 3)), np.arange(3.0), np.eye(2)])
sf.dense_direction_factor(np.ones((2, 3)), np.ones(3), 1, 3)
sf.dense_rank_one_operand(np.ones(5), np.ones(7))
sf.scatter(o, p, 2)
sf.gather(sf.scatter(o, p, 1), p, 1)
sf.kronecker_apply([np.ones((3, 5)), np.ones(5), np.ones((2, 5)), np.ones((4, 5))], np.ones(625))
sf.kernel.hadamard_rowsum_batched_host(basis, F.cpu().numpy())
Uh = eu.generate_modal_states(7, 6, seed=2).cpu()
Ja = eu.generate_metric(7, 6, seed=3).cpu()
eu.volume_curvilinear_modal_host(Uh, Ja, 6, sumsq=torch.empty(7, dtype=torch.float64))
torch.cuda.synchronize()
print("sanitize run ok")
