"""Seeded, element-addressable synthetic inputs (host restatement of gen.cu).

Every value is a pure function of (seed, global index) through a splitmix64
counter hash, so

  * the host arrays built here are bit-identical to the device generator's
    (sfb_generate_uniform / sfb_generate_euler_states) - tests pin this;
  * any element can be regenerated on its own (the CPU oracle checks sampled
    elements of a full-size GPU run);
  * an element shard [e0, e0 + E) is the same whatever the number of ranks.

Distributions are BASELINE.json's: config 2 F ~ U[-1, 1]; configs 3-4
rho ~ U[0.8, 1.2], v_m ~ U[-0.3, 0.3], p ~ U[0.8, 1.2], gamma = 1.4.
"""

import numpy as np

_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)
EULER_BOUNDS = (0.8, 1.2, -0.3, 0.3, 0.8, 1.2)
GAMMA = 1.4


def splitmix64(z):
    """splitmix64 finaliser on uint64 arrays (wrapping arithmetic)."""
    z = np.asarray(z, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = z + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


def _key(seed):
    return splitmix64(np.array([seed], dtype=np.uint64))[0]


def u01(key, idx):
    with np.errstate(over="ignore"):
        h = splitmix64(np.uint64(key) + np.asarray(idx, dtype=np.uint64))
    return (h >> np.uint64(11)).astype(np.float64) * 2.0**-53


def uniform_array(count, seed, lo, hi, i0=0):
    """out[t] = lo + (hi - lo) * u(seed, i0 + t)."""
    idx = np.arange(i0, i0 + count, dtype=np.uint64)
    return lo + (hi - lo) * u01(_key(seed), idx)


def euler_states(E, n, seed, gamma=GAMMA, bounds=EULER_BOUNDS, e0=0):
    """Conserved states U (E, 5, n^3) for elements e0 .. e0+E-1."""
    nodes = n**3
    key = _key(seed)
    e = np.arange(e0, e0 + E, dtype=np.uint64)[:, None]
    r = np.arange(nodes, dtype=np.uint64)[None, :]
    g = e * np.uint64(5 * nodes) + r
    rlo, rhi, vlo, vhi, plo, phi = bounds
    rho = rlo + (rhi - rlo) * u01(key, g)
    v0 = vlo + (vhi - vlo) * u01(key, g + np.uint64(nodes))
    v1 = vlo + (vhi - vlo) * u01(key, g + np.uint64(2 * nodes))
    v2 = vlo + (vhi - vlo) * u01(key, g + np.uint64(3 * nodes))
    p = plo + (phi - plo) * u01(key, g + np.uint64(4 * nodes))
    vv = v0 * v0 + v1 * v1 + v2 * v2
    et = p / (gamma - 1.0) + 0.5 * rho * vv
    return np.stack([rho, rho * v0, rho * v1, rho * v2, et], axis=1)
