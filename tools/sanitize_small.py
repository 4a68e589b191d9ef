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
torch.cuda.synchronize()
print("sanitize run ok")
