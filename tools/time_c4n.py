"""Config-4 point(s) n (argv): ms per launch, best of 3 x 20."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2306_11665_b200 import euler as eu  # noqa: E402

for n in map(int, sys.argv[1:] or ["5"]):
    E = round(2**24 / n**3)
    U = eu.generate_states(E, n, seed=4)
    R = torch.empty_like(U)
    for _ in range(3):
        eu.volume_cartesian(U, n, out=R)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(3):
        a.record()
        for _ in range(20):
            eu.volume_cartesian(U, n, out=R)
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b) / 20)
    print(f"n={n} {best:.4f} ms")
