"""A/B of the config-4 points n = 5..8: ms per launch with dynamic claims vs the static split."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2306_11665_b200 import euler as eu  # noqa: E402

for n in range(int(sys.argv[1]) if len(sys.argv) > 1 else 5, 9):
    E = round(2**24 / n**3)
    U = eu.generate_states(E, n, seed=4)
    R = torch.empty_like(U)
    out = {}
    for dyn in (False, True, False, True):
        for _ in range(3):
            eu.volume_cartesian(U, n, out=R, dynamic=dyn)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(20):
            eu.volume_cartesian(U, n, out=R, dynamic=dyn)
        b.record()
        torch.cuda.synchronize()
        out.setdefault(dyn, []).append(a.elapsed_time(b) / 20)
        if dyn:
            R2 = R.clone()
        else:
            R1 = R.clone()
    print(f"n={n} static {min(out[False]):.4f} ms  dynamic {min(out[True]):.4f} ms  "
          f"bitwise {torch.equal(R1, R2)}")
