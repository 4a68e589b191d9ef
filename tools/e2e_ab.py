"""A/B of the host-buffer entry (config 3, pinned buffers): ms per call under the
current SFB_HOST_* environment, and the same-buffer copy ceiling."""
import sys
import time

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2306_11665_b200 import euler as eu  # noqa: E402

n, E = 4, 262144
U = eu.generate_states(E, n, seed=3)
Uh = eu.pinned_empty(tuple(U.shape))
Uh.copy_(U.cpu())
Rh = eu.pinned_empty(tuple(U.shape))
for _ in range(2):
    eu.volume_cartesian_host(Uh, n, out=Rh)
ts = []
for _ in range(10):
    t = time.perf_counter()
    eu.volume_cartesian_host(Uh, n, out=Rh)
    ts.append(time.perf_counter() - t)
ts.sort()
print(f"e2e ms mean {1e3 * sum(ts) / len(ts):.3f} min {1e3 * ts[0]:.3f} "
      f"ceiling {bench.pcie_ceiling_ms(Uh, Rh, U):.3f}")
