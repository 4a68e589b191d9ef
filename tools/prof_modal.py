"""Driver for ncu captures of the config-5 kernel (n, E from argv)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2306_11665_b200 import euler as eu  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 6
E = int(sys.argv[2]) if len(sys.argv) > 2 else 65536
Uh = eu.generate_modal_states(E, n, seed=5)
Ja = eu.generate_metric(E, n, seed=6)
R = torch.empty_like(Uh)
ss = torch.empty(E, dtype=torch.float64, device="cuda")
for _ in range(3):
    eu.volume_curvilinear_modal(Uh, Ja, n, out=R, sumsq=ss)
torch.cuda.synchronize()
print("ok", float(ss.sum()))
