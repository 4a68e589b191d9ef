"""GPU parity of the periodic Burgers time derivative and RK4 integration.

SURVEY 8(f) rows f1 (interface term, burgers.py:134-162) and f3 (classic RK4
around the residual with entropy monitoring, demos/burgers_entropy.py:25-51).
Golden vectors come from the reference itself (tests/golden/make_golden.py:
make_burgers / make_burgers_rk4); time derivatives and RK4 trajectories are
bitwise, the entropy monitors (numpy's BLAS dot vs a fixed-order device sum)
match to 1e-14 relative.
"""

import numpy as np
import pytest
import torch

from conftest import golden

pytestmark = pytest.mark.gpu

sf = pytest.importorskip("paper_2306_11665_b200")
from paper_2306_11665_b200 import burgers as bg  # noqa: E402
from paper_2306_11665_b200 import synth  # noqa: E402

CASES = [(1, 3), (1, 6), (2, 4), (2, 5), (3, 3), (3, 4), (3, 6), (2, 9)]
RK4_CASES = [(2, 5, 2e-3, 40, 10), (1, 6, 1e-3, 30, 10), (3, 4, 2e-3, 12, 4)]


@pytest.mark.parametrize("d,n", CASES)
def test_time_derivative_bitwise(d, n):
    g = golden("burgers.npz")
    st = sf.BurgersState(d, n, g[f"u_{d}_{n}"])
    assert np.array_equal(sf.time_derivative(st), g[f"dudt_{d}_{n}"])
    assert np.array_equal(sf.time_derivative(st, sf.average_flux), g[f"dudt_avg_{d}_{n}"])


def test_time_derivative_batched_matches_single():
    d, n, E = 2, 5, 2001
    u = torch.from_numpy(synth.uniform_array(E * n**d, 77, -1.0, 1.0).reshape(E, n**d)).cuda()
    out = bg.time_derivative_batched(u, d, n).cpu().numpy()
    for e in (0, 1, 999, E - 1):
        ref = sf.time_derivative(sf.BurgersState(d, n, u[e].cpu().numpy()))
        assert np.array_equal(out[e], ref)


@pytest.mark.parametrize("d,n,dt,steps,every", RK4_CASES)
@pytest.mark.parametrize("name", ["ec", "avg"])
def test_rk4_trajectory_bitwise(d, n, dt, steps, every, name):
    g = golden("burgers_rk4.npz")
    flux = sf.ec_two_point_flux if name == "ec" else sf.average_flux
    u0 = torch.from_numpy(g[f"u0_{d}_{n}"]).cuda().reshape(1, -1).repeat(3, 1)
    u, ent, mass = bg.integrate_rk4(u0, d, n, dt, steps, flux, every=every)
    for e in range(3):
        assert np.array_equal(u[e].cpu().numpy(), g[f"u_{name}_{d}_{n}"])
    ref = g[f"entropy_{name}_{d}_{n}"]
    got = ent[0].cpu().numpy()
    assert got.shape == ref.shape
    assert np.max(np.abs(got - ref) / np.abs(ref)) <= 1e-14
    # mass sum omega u is conserved by the periodic scheme (to rounding)
    m = mass[0].cpu().numpy()
    assert np.max(np.abs(m - m[0])) <= 1e-13 * (1 + np.abs(u0[0].cpu().numpy()).max())


def test_rk4_entropy_conservation_contrast():
    # the demo's point: EC flux keeps S to time-discretisation error, the
    # average flux drifts at first order
    d, n, dt, steps = 2, 5, 2e-3, 200
    u0 = torch.from_numpy(synth.uniform_array(n**d, 12, -1.0, 1.0)).cuda().reshape(1, -1)
    _, ent_ec, _ = bg.integrate_rk4(u0, d, n, dt, steps, sf.ec_two_point_flux, every=50)
    _, ent_avg, _ = bg.integrate_rk4(u0, d, n, dt, steps, sf.average_flux, every=50)
    s0 = ent_ec[0, 0].item()
    drift_ec = (ent_ec[0] - s0).abs().max().item() / s0
    drift_avg = (ent_avg[0] - s0).abs().max().item() / s0
    assert drift_ec < 1e-8 and drift_avg > 100 * drift_ec


def test_rk4_large_batch_elements_independent():
    d, n, E, steps = 2, 5, 100_003, 5
    u0 = torch.from_numpy(synth.uniform_array(E * n**d, 5, -1.0, 1.0).reshape(E, n**d)).cuda()
    u, _, _ = bg.integrate_rk4(u0, d, n, 1e-3, steps)
    for e in (0, 77_777, E - 1):
        ue, _, _ = bg.integrate_rk4(u0[e:e + 1], d, n, 1e-3, steps)
        assert torch.equal(u[e], ue[0])


def test_rk4_arguments():
    u0 = torch.zeros((2, 25), dtype=torch.float64, device="cuda")
    with pytest.raises(ValueError):
        bg.integrate_rk4(u0, 2, 5, 1e-3, 3, flux=lambda a, b: a * b)
    with pytest.raises(ValueError):
        bg.integrate_rk4(u0, 2, 5, 1e-3, -1)
    u, ent, mass = bg.integrate_rk4(u0, 2, 5, 1e-3, 0, every=1)
    assert torch.equal(u, u0) and ent.shape == (2, 1)


def test_acceptance_entropy_and_mass_conservation():
    # the reference's acceptance 6 (pkg/tests/test_acceptance.py:183-216) on the
    # device path: EC flux |dS/dt| <= 1e-12 (1 + |S|) and mass conservation on
    # 108 random states over d in {1,2,3}, n in {3..6}; the average flux breaks
    # entropy conservation on >= 95% of them
    rng = np.random.default_rng(66)
    states = broken = 0
    worst_ec = worst_mass = 0.0
    for d in (1, 2, 3):
        for n in (3, 4, 5, 6):
            omega = sf.tensor_product_weights(sf.gauss_lobatto_legendre(n).weights, d)
            u = rng.uniform(-1.0, 1.0, (9, n**d))
            ut = torch.from_numpy(u).cuda()
            ec = bg.time_derivative_batched(ut, d, n).cpu().numpy()
            avg = bg.time_derivative_batched(ut, d, n, sf.average_flux).cpu().numpy()
            for k in range(9):
                s = 0.5 * np.dot(omega, u[k] * u[k])
                worst_ec = max(worst_ec, abs(np.dot(omega * u[k], ec[k])) / (1.0 + abs(s)))
                worst_mass = max(worst_mass, abs(float(np.dot(omega, ec[k]))))
                broken += abs(np.dot(omega * u[k], avg[k])) > 1e-6
                states += 1
    assert states == 108
    assert worst_ec <= 1e-12 and worst_mass <= 1e-12
    assert broken >= 0.95 * states
