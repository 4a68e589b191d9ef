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

# config 5: modal states and the warped-mesh metric
MODAL_MEANS = (1.0, 0.0, 0.0, 0.0, 2.5)  # rho = 1, v = 0, p ~ 1 (gamma = 1.4)
MODAL_AMPS = (0.02, 0.02, 0.02, 0.02, 0.02)
MODAL_C0 = 2.0 * np.sqrt(2.0)  # 1 / phi_0 of the orthonormal Legendre basis in 3-D
MESH_K = 128  # elements per direction of the periodic lattice (128^3 = 2^21)
WARP_AMP = 0.05


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


def mode_decay(n):
    """2^-(k0+k1+k2) for the n^3 modes (x-fastest)."""
    k = np.arange(n**3)
    deg = k % n + (k // n) % n + k // (n * n)
    return np.ldexp(1.0, -deg)


def modal_states(E, n, seed, e0=0):
    """Modal conserved coefficients Uhat (E, 5, n^3) in the orthonormal Legendre basis.

    Uhat[e,v,k] = (A_v 2^-|k|) (2u - 1) (+ mean_v C0 at k = 0), u the counter
    hash of ((e*5 + v) n^3 + k).  |perturbation| <= 10 A_v at every node, so
    rho in [0.8, 1.2], |v| < 0.25, p > 0.85 (positive states by construction).
    """
    modes = n**3
    key = _key(seed)
    e = np.arange(e0, e0 + E, dtype=np.uint64)[:, None, None]
    v = np.arange(5, dtype=np.uint64)[None, :, None]
    k = np.arange(modes, dtype=np.uint64)[None, None, :]
    idx = (e * np.uint64(5) + v) * np.uint64(modes) + k
    w = 2.0 * u01(key, idx) - 1.0
    amp = np.asarray(MODAL_AMPS)[None, :, None] * mode_decay(n)[None, None, :]
    out = amp * w
    out[:, :, 0] = np.asarray(MODAL_MEANS)[None, :] * MODAL_C0 + out[:, :, 0]
    return out


def warp_phases(seed):
    """phi[m][k] in [0, 1): phase of component m's sine factor along direction k."""
    key = _key(seed)
    return u01(key, np.arange(9, dtype=np.uint64)).reshape(3, 3)


def metric_cofactors(E, n, seed, e0=0, K=MESH_K, amp=WARP_AMP, nodes=None):
    """Ja (E, 3, 3, n^3): Ja[e,i,m,r] = J dxi^i/dx_m on the warped lattice.

    Element e sits at lattice cell (e mod K^3) of [0,1]^3 (x fastest), h = 1/K;
    node r maps to X = (cell + (xi+1)/2) h and then to
        x_m = X_m + amp prod_k sin(2 pi (X_k + phi[m][k])),
    so dx/dxi = (h/2)(I + amp 2 pi G'(X)) and Ja = adj(dx/dxi) analytically.
    """
    if nodes is None:
        from .operators import gauss_lobatto_legendre

        nodes = gauss_lobatto_legendre(n).nodes
    phi = warp_phases(seed)
    h = 1.0 / K
    cell = (np.arange(e0, e0 + E) % (K**3))[:, None]
    cx, cy, cz = cell % K, (cell // K) % K, cell // (K * K)
    r = np.arange(n**3)[None, :]
    X = [(cx + (nodes[r % n] + 1.0) * 0.5) * h,
         (cy + (nodes[(r // n) % n] + 1.0) * 0.5) * h,
         (cz + (nodes[r // (n * n)] + 1.0) * 0.5) * h]
    two_pi = 2.0 * np.pi
    G = np.empty((3, 3) + X[0].shape)
    for m in range(3):
        sn = [np.sin(two_pi * (X[k] + phi[m][k])) for k in range(3)]
        cs = [np.cos(two_pi * (X[k] + phi[m][k])) for k in range(3)]
        for i in range(3):
            prod = cs[i] * sn[(i + 1) % 3] * sn[(i + 2) % 3]
            G[m, i] = 0.5 * h * ((1.0 if m == i else 0.0) + amp * two_pi * prod)
    Ja = np.empty((E, 3, 3, n**3))
    for i in range(3):
        for m in range(3):
            # adj(G)[i][m] = cofactor C[m][i]
            a, b = [x for x in range(3) if x != m]
            c, d = [x for x in range(3) if x != i]
            minor = G[a, c] * G[b, d] - G[a, d] * G[b, c]
            Ja[:, i, m] = minor if (i + m) % 2 == 0 else -minor
    return Ja
