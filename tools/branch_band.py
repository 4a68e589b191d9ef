"""Log-mean branch band (as tests/test_gpu_euler.py) for n = 2..8: max_rel and the
worst per-element error relative to the flux scale."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from oracle import c_oracle  # noqa: E402
from paper_2306_11665_b200 import euler as eu  # noqa: E402

for n in range(2, 9):
    E = 512
    U = eu.generate_states(E, n, seed=21)
    base = U[:, :, :1].clone()
    amp = torch.logspace(-1, -7, E, dtype=torch.float64, device="cuda")[:, None, None]
    U = base + amp * (U - base)
    R = eu.volume_cartesian(U, n).cpu().numpy()
    D = eu.gll_operators(n)[1]
    ref = c_oracle.euler_volume_cartesian(U.cpu().numpy(), D, threads=8)
    mr = float(np.abs(R - ref).max() / np.abs(ref).max())
    scale = np.abs(U.cpu().numpy()).max(axis=(1, 2)) ** 2
    per = np.abs(R - ref).max(axis=(1, 2)) / scale
    worst = int(per.argmax())
    print(f"n={n} max_rel {mr:.2e} worst element {worst} (amp {amp[worst].item():.1e}) "
          f"err/scale {per[worst]:.2e}")
