"""Experiment: per-CTA start/end times of the config-3 kernel (variant built with
SFB_WARP_EXP_TIMES=1, loaded through SFB_LIB): how long is the tail?"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2306_11665_b200 import euler as eu  # noqa: E402

n, E = 4, 262144
G = 148 * 12
U = eu.generate_states(E, n, seed=3)
R = torch.empty_like(U)
for rep in range(5):
    eu.volume_cartesian(U, n, out=R)
    torch.cuda.synchronize()
    raw = R.view(-1)[: 3 * G].cpu().numpy().view(np.int64)
    end, start = raw[:G].astype(np.float64), raw[G:2 * G].astype(np.float64)
    t0 = start.min()
    s, e = (start - t0) / 1e3, (end - t0) / 1e3
    d = e - s
    print(f"rep {rep}: start max {s.max():.1f} us; end min/median/max {e.min():.1f}/{np.median(e):.1f}/{e.max():.1f} us; "
          f"duration min/median/max {d.min():.1f}/{np.median(d):.1f}/{d.max():.1f}; "
          f"mean active fraction {d.sum() / (G * e.max()):.3f}")
    sm = raw[2 * G:3 * G]
    print('   CTAs per SM min/max', np.bincount(sm, minlength=148).min(), np.bincount(sm, minlength=148).max())
    per_sm_end = np.array([e[sm == k].max() for k in range(148)])
    print(f"   per-SM last end min/median/max {per_sm_end.min():.1f}/{np.median(per_sm_end):.1f}/{per_sm_end.max():.1f}")
