import sys; sys.path.insert(0,'.')
import numpy as np, torch
from paper_2306_11665_b200 import euler as eu
from oracle import euler_oracle as eo
for n in (2,3,5):
  for E in (1,2,3,4,7):
    U = eu.generate_states(E, n, seed=4)
    R = eu.volume_cartesian(U, n).cpu().numpy()
    _, D, _, _ = eu.gll_operators(n)
    ref = eo.euler_volume_cartesian(U.cpu().numpy(), D)
    err = np.abs(R-ref).max(axis=2)/np.abs(ref).max()
    print(n, E, err.max(), np.argwhere(err>1e-12)[:6].tolist())
