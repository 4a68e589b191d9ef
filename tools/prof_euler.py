"""Small driver for ncu captures of the Euler volume kernel (n, E from argv)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2306_11665_b200 import euler as eu  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4
E = int(sys.argv[2]) if len(sys.argv) > 2 else 262144
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
U = eu.generate_states(E, n, seed=3)
R = torch.empty_like(U)
for _ in range(reps):
    eu.volume_cartesian(U, n, out=R)
torch.cuda.synchronize()
print("ok", n, E, float(R.abs().max()))
