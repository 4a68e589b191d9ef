"""GPU parity of the fused Euler flux-differencing kernel (configs 3-4).

Bar (BASELINE.json north star): norm-wise relative error
max|got - ref| / max|ref| <= 1e-12 in FP64 against the reference pipeline
(golden vectors from sumfac 0.1.0 through the index-trick operand) and
against the CPU oracle at larger sizes; size-independent properties at the
full config sizes.
"""

import numpy as np
import pytest
import torch

from conftest import golden, max_rel

pytestmark = pytest.mark.gpu

sf = pytest.importorskip("paper_2306_11665_b200")
from paper_2306_11665_b200 import euler as eu  # noqa: E402
from paper_2306_11665_b200 import synth  # noqa: E402
from oracle import c_oracle  # noqa: E402
from oracle import euler_oracle as eo  # noqa: E402

TOL = 1e-12  # FP64 parity bar of BASELINE.json


@pytest.mark.parametrize("n", range(2, 9))
def test_euler_cartesian_matches_reference_golden(n):
    g = golden("euler_cartesian.npz")
    U = torch.from_numpy(g[f"U{n}"]).cuda()
    R = eu.volume_cartesian(U, n, D=g[f"D{n}"]).cpu().numpy()
    assert max_rel(R, g[f"R{n}"]) <= TOL


@pytest.mark.parametrize("n", range(2, 9))
def test_euler_cartesian_matches_oracle_many_elements(n):
    E = {2: 4099, 3: 1501, 4: 1031, 5: 403, 6: 211, 7: 97, 8: 61}[n]  # ragged tails
    U = eu.generate_states(E, n, seed=40 + n)
    R = eu.volume_cartesian(U, n).cpu().numpy()
    _, D, _, _ = eu.gll_operators(n)
    ref = c_oracle.euler_volume_cartesian(U.cpu().numpy(), D, threads=8)
    assert max_rel(R, ref) <= TOL
    # per-element check too (no element hides behind another's scale)
    worst = max(max_rel(R[e], ref[e]) for e in range(0, E, max(1, E // 50)))
    assert worst <= 1e-11


def test_single_and_empty_batches():
    n = 4
    U = eu.generate_states(1, n, seed=1)
    R = eu.volume_cartesian(U, n).cpu().numpy()
    _, D, _, _ = eu.gll_operators(n)
    assert max_rel(R, eo.euler_volume_cartesian(U.cpu().numpy(), D)) <= TOL
    U0 = torch.empty((0, 5, 64), dtype=torch.float64, device="cuda")
    assert eu.volume_cartesian(U0, n).shape == (0, 5, 64)


def test_bad_arguments_raise():
    n = 4
    U = eu.generate_states(3, n, seed=1)
    with pytest.raises(ValueError):
        eu.volume_cartesian(U[:, :4].contiguous(), n)
    with pytest.raises(ValueError):
        eu.volume_cartesian(U.float(), n)
    with pytest.raises(NotImplementedError):
        eu.volume_cartesian(torch.empty((2, 5, 729), dtype=torch.float64, device="cuda"), 9,
                            D=np.eye(9))
    # host entry: outputs that the library would write through must be checked
    Uh = U.cpu().numpy()
    for bad in (np.empty((3, 5, 64), dtype=np.float32), np.empty((2, 5, 64)),
                np.empty((3, 64, 5)).transpose(0, 2, 1), torch.empty((3, 5, 64), dtype=torch.float64)):
        with pytest.raises(ValueError):
            eu.volume_cartesian_host(Uh, n, out=bad)
    ro = np.empty((3, 5, 64))
    ro.flags.writeable = False
    with pytest.raises(ValueError):
        eu.volume_cartesian_host(Uh, n, out=ro)
    Ut = U.cpu()
    for bad in (torch.empty((3, 64, 5), dtype=torch.float64).transpose(1, 2), torch.empty_like(U),
                np.empty((3, 5, 64))):
        with pytest.raises(ValueError):
            eu.volume_cartesian_host(Ut, n, out=bad)


def test_constant_state_is_steady_full_size():
    n, E = 4, 262144
    U = eu.generate_states(E, n, seed=3)
    U[:] = U[:, :, :1]  # element-wise constant states
    R = eu.volume_cartesian(U, n)
    assert R.abs().max().item() <= 1e-12 * U.abs().max().item()


def test_full_config3_sampled_and_properties():
    n, E = 4, 262144
    U = eu.generate_states(E, n, seed=3)
    R = eu.volume_cartesian(U, n)
    # generator is the host one, element-addressably
    idx = np.sort(np.random.default_rng(7).choice(E, 96, replace=False))
    Us = np.concatenate([synth.euler_states(1, n, seed=3, e0=int(e)) for e in idx])
    assert np.array_equal(U[idx].cpu().numpy(), Us)
    _, D, _, _ = eu.gll_operators(n)
    ref = eo.euler_volume_cartesian(Us, D)
    assert max_rel(R[idx].cpu().numpy(), ref) <= TOL
    # linearity in scale (exact: power-of-two scaling)
    R4 = eu.volume_cartesian(U, n, scale=4.0)
    assert torch.equal(R4, 2.0 * R)
    # SBP telescoping: omega . R equals the boundary flux difference
    rule, _, _, _ = eu.gll_operators(n)
    omega = torch.from_numpy(sf.tensor_product_weights(rule.weights, 3)).cuda()
    tot = (R * omega).sum(dim=2)
    rho = U[:, 0]
    v = U[:, 1:4] / rho[:, None]
    p = 0.4 * (U[:, 4] - 0.5 * rho * (v * v).sum(1))
    r = torch.arange(n**3, device="cuda")
    w = torch.from_numpy(rule.weights).cuda()
    expect = torch.zeros_like(tot)
    for j in range(3):
        rj = (r // n**j) % n
        sgn = (rj == n - 1).double() - (rj == 0).double()
        wf = omega / w[rj] * sgn
        fl = [rho * v[:, j], U[:, 1] * v[:, j] + p * (j == 0), U[:, 2] * v[:, j] + p * (j == 1),
              U[:, 3] * v[:, j] + p * (j == 2), (U[:, 4] + p) * v[:, j]]
        for var in range(5):
            expect[:, var] += (wf * fl[var]).sum(1)
    assert (tot - expect).abs().max().item() <= 1e-12 * (1 + expect.abs().max().item())


def test_host_buffer_entry_matches_device_entry():
    n, E = 4, 20000
    U = eu.generate_states(E, n, seed=12)
    Rd = eu.volume_cartesian(U, n)
    Uh = eu.pinned_empty((E, 5, 64))
    Uh.copy_(U.cpu())
    Rh = eu.volume_cartesian_host(Uh, n)
    assert torch.equal(Rh, Rd.cpu())
    Rn = eu.volume_cartesian_host(U.cpu().numpy(), n)  # pageable numpy path
    assert np.array_equal(Rn, Rd.cpu().numpy())
    out = np.full((E, 5, 64), np.nan)  # caller-supplied numpy output
    assert eu.volume_cartesian_host(U.cpu().numpy(), n, out=out) is out
    assert np.array_equal(out, Rd.cpu().numpy())


@pytest.mark.parametrize("n,E", [(4, 100003), (3, 77777), (6, 30001)])
def test_host_entry_many_chunks(n, E, monkeypatch):
    # a ragged last chunk, and with a small chunk size many chunks cycling
    # through every stream of the pipeline
    U = eu.generate_states(E, n, seed=13)
    Rd = eu.volume_cartesian(U, n).cpu()
    Uh = eu.pinned_empty((E, 5, n**3))
    Uh.copy_(U.cpu())
    for env in ({}, {"SFB_HOST_CHUNK_MB": "2"}, {"SFB_HOST_CHUNK_MB": "5"}):
        for k, v in env.items():
            monkeypatch.setenv(k, v)
        assert torch.equal(eu.volume_cartesian_host(Uh, n), Rd), env
        for k in env:
            monkeypatch.delenv(k)


@pytest.mark.parametrize("d,n", [(1, 6), (2, 4), (3, 3), (3, 4), (3, 6), (2, 9)])
def test_burgers_volume_residual_golden(d, n):
    g = golden("burgers.npz")
    u = g[f"u_{d}_{n}"]
    st = sf.BurgersState(d, n, u)
    assert np.array_equal(sf.volume_residual(st), g[f"vol_ec_{d}_{n}"])
    assert np.array_equal(sf.volume_residual(st, sf.average_flux), g[f"vol_avg_{d}_{n}"])
    assert max_rel(sf.time_derivative(st), g[f"dudt_{d}_{n}"]) <= 1e-13
    s = float(g[f"entropy_{d}_{n}"])
    assert abs(sf.entropy_time_derivative(st)) <= 1e-12 * (1 + abs(s))


def test_burgers_flop_count_and_batched():
    d, n = 2, 4
    st = sf.BurgersState(d, n, np.linspace(-1.0, 1.0, n**d))
    sf.volume_residual(st)
    before = sf.multiplication_count()
    sf.volume_residual(st)
    assert sf.multiplication_count() - before == d * n ** (d + 1)
    u = torch.from_numpy(np.stack([synth.uniform_array(27, s, -1, 1) for s in range(9)])).cuda()
    out = sf.volume_residual_batched(u, 3, 3).cpu().numpy()
    for e in range(9):
        ref = sf.volume_residual(sf.BurgersState(3, 3, u[e].cpu().numpy()))
        assert np.array_equal(out[e], ref)


@pytest.mark.parametrize("n", [3, 5, 7])
def test_many_blocks_per_cta_odd_sizes(n):
    # odd 5 n^3: element blocks start at odd double offsets, so the bulk copy is
    # shifted by one double; enough elements that every CTA loops over both
    # input slots, and a ragged tail that takes the plain-load path
    E = {3: 40001, 5: 12001, 7: 4001}[n]
    U = eu.generate_states(E, n, seed=90 + n)
    R = eu.volume_cartesian(U, n)
    _, D, _, _ = eu.gll_operators(n)
    idx = np.concatenate([np.arange(3), np.random.default_rng(n).choice(E, 40, replace=False),
                          np.arange(E - 3, E)])
    ref = eo.euler_volume_cartesian(U[idx].cpu().numpy(), D)
    assert max_rel(R[idx].cpu().numpy(), ref) <= TOL


@pytest.mark.parametrize("n", range(2, 9))
def test_log_mean_branch_band_matches_oracle(n):
    # element-wise perturbations of a constant state with amplitudes 1e-1..1e-7:
    # neighbour ratios sweep u = (d/s)^2 through both log-mean branches and
    # across the ~1e-5 threshold (every n: each has its own kernel)
    E = 512
    U = eu.generate_states(E, n, seed=21)
    base = U[:, :, :1].clone()
    amp = torch.logspace(-1, -7, E, dtype=torch.float64, device="cuda")[:, None, None]
    U = base + amp * (U - base)
    R = eu.volume_cartesian(U, n).cpu().numpy()
    _, D, _, _ = eu.gll_operators(n)
    ref = c_oracle.euler_volume_cartesian(U.cpu().numpy(), D, threads=8)
    assert max_rel(R, ref) <= TOL
    # per element against the D-weighted flux scale (the residual itself shrinks
    # with amp; rounding enters through 3(n-1) D-weighted fluxes per row, so the
    # bound carries ||D||_inf: 2e-14 x 9.1 at n = 4, x 51 at n = 8)
    scale = np.abs(U.cpu().numpy()).max(axis=(1, 2)) ** 2 * np.abs(D).sum(axis=1).max()
    assert (np.abs(R - ref).max(axis=(1, 2)) <= 2e-14 * scale).all()


@pytest.mark.parametrize("n", range(2, 9))
def test_non_physical_state_is_contained(n):
    # a negative density (non-physical) makes that element's logarithms NaN;
    # the kernels are branch-free, so the NaN stays in that element and the
    # others are untouched (no trap, no cross-element contamination)
    E = 37
    U = eu.generate_states(E, n, seed=8)
    ref = eu.volume_cartesian(U, n).cpu()
    bad = 17
    U[bad, 0, 3] = -U[bad, 0, 3]
    R = eu.volume_cartesian(U, n).cpu()
    assert torch.isnan(R[bad]).any()
    keep = [e for e in range(E) if e != bad]
    assert torch.equal(R[keep], ref[keep])


def test_misaligned_pointer_rejected():
    from paper_2306_11665_b200 import _lib

    n, E = 4, 8
    U = eu.generate_states(E + 1, n, seed=2).reshape(-1)
    R = torch.empty_like(U)
    _, D, _, _ = eu.gll_operators(n)
    Dh = np.ascontiguousarray(D)
    with pytest.raises(ValueError):  # 8-byte offset: not 16-byte aligned
        _lib.call("sfb_euler_volume_cartesian", E, n, Dh.ctypes.data, 1.4, 2.0,
                  _lib.ptr(U) + 8, _lib.ptr(R), _lib.stream_ptr())


def test_beyond_int32_double_offsets():
    # 7,000,000 elements at n = 4: U and R hold 2.24e9 doubles each, past
    # 2^31 - element offsets must be 64-bit in every index computation
    n, E = 4, 7_000_000
    U = eu.generate_states(E, n, seed=77)
    R = eu.volume_cartesian(U, n)
    idx = np.array([0, 6_710_887, 6_710_888, E - 2, E - 1])  # around 2^31 / 320
    _, D, _, _ = eu.gll_operators(n)
    Us = np.concatenate([synth.euler_states(1, n, seed=77, e0=int(e)) for e in idx])
    assert np.array_equal(U[idx].cpu().numpy(), Us)
    assert max_rel(R[idx].cpu().numpy(), eo.euler_volume_cartesian(Us, D)) <= TOL
    del U, R
    torch.cuda.empty_cache()


@pytest.mark.parametrize("n", range(2, 9))
def test_runs_are_bitwise_reproducible(n):
    # fixed summation orders everywhere (no atomics): repeated launches agree bitwise
    U = eu.generate_states(20_000 if n < 6 else 4_000, n, seed=5)
    a = eu.volume_cartesian(U, n)
    b = eu.volume_cartesian(U, n)
    assert torch.equal(a, b)


@pytest.mark.parametrize("n", range(2, 9))
def test_general_operator_gamma_and_scale(n):
    # D, gamma and scale are parameters of the ABI: a dense random operator
    # (no GLL structure, nonzero diagonal), gamma = 5/3 and scale = -0.75
    rng = np.random.default_rng(100 + n)
    D = rng.standard_normal((n, n))
    E, gamma, scale = 57, 5.0 / 3.0, -0.75
    U = eu.generate_states(E, n, seed=60 + n, gamma=gamma)
    R = eu.volume_cartesian(U, n, D=D, gamma=gamma, scale=scale).cpu().numpy()
    ref = eo.euler_volume_cartesian(U.cpu().numpy(), D, gamma=gamma, scale=scale)
    assert max_rel(R, ref) <= TOL


def test_launch_is_ordered_on_the_callers_stream():
    # inputs produced on a side stream, the kernel launched on that stream, the
    # result read after that stream only: no implicit default-stream ordering
    n, E = 4, 20000
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        U = eu.generate_states(E, n, seed=8)
        R = torch.empty_like(U)
        for _ in range(3):
            eu.volume_cartesian(U, n, out=R, stream=s)
        R2 = R * 1.0
    s.synchronize()
    ref = eu.volume_cartesian(U, n)
    assert torch.equal(R2, ref)
