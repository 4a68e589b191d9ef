"""f3 Burgers RK4 (as bench.py's extras line): ms for 1M elements x 20 steps, d=2, n=5."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2306_11665_b200 import burgers as bg  # noqa: E402
from paper_2306_11665_b200 import euler as eu  # noqa: E402

E, d, n, steps = 1 << 20, 2, 5, 20
u0 = eu.generate_uniform(E * n**d, 11, -1.0, 1.0).reshape(E, n**d)
bg.integrate_rk4(u0[:1024], d, n, 1e-3, 2, every=1)
torch.cuda.synchronize()
best = 1e9
for _ in range(3):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    bg.integrate_rk4(u0, d, n, 1e-3, steps, every=steps)
    b.record()
    torch.cuda.synchronize()
    best = min(best, a.elapsed_time(b))
print(f"rk4 {best:.2f} ms")
