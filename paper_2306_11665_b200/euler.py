"""3-D compressible Euler flux-differencing volume terms (batched device tier).

The reference's flux-differencing entry point, ``volume_residual``
(sumfac/burgers.py:117-131), is scalar and single-element; BASELINE configs 3-5
extend the same Hadamard-product volume term to the 5-variable Euler state
with the Chandrashekar entropy-conservative flux, batched over elements:

  volume_cartesian(U, n)          R = scale sum_j (D_j o F#_j) 1      (configs 3, 4)
  volume_cartesian_host(U, n)     same, numpy in / numpy out, pipelined H2D/D2H
  volume_curvilinear_modal(...)   Rhat = Pi^3 [scale sum_i (D_i o Ft_i) 1] (V^3 Uhat)
                                  with contravariant fluxes            (config 5)

States are (E, 5, n^3) float64 ([rho, rho v, E] per element, node axis
fastest).  All arithmetic runs in sm_100a kernels (csrc/euler_warp.cu for
n = 2, 3, 4, csrc/euler.cu for n = 5..8, csrc/modal.cu); there is no CPU path.
"""

import numpy as np
import torch

from . import _lib, synth
from .operators import (
    gauss_lobatto_legendre,
    lagrange_diff_matrix,
    legendre_vandermonde,
    projection_operator,
)

GAMMA = 1.4
_ops_cache = {}


def gll_operators(n):
    """(rule, D, V, Pi) for the n-point GLL rule, built once on the host."""
    if n not in _ops_cache:
        rule = gauss_lobatto_legendre(n)
        D = lagrange_diff_matrix(rule)
        V = legendre_vandermonde(rule)
        Pi = projection_operator(rule, V)
        _ops_cache[n] = (rule, D, V, Pi)
    return _ops_cache[n]


def _host_matrix(D, n):
    D = np.ascontiguousarray(D, dtype=np.float64)
    if D.shape != (n, n):
        raise ValueError(f"operator shape {D.shape} does not match ({n}, {n})")
    return D


def _check_states(U, n, name="U"):
    if not isinstance(U, torch.Tensor) or not U.is_cuda or U.dtype != torch.float64:
        raise ValueError(f"{name} must be a CUDA float64 tensor")
    if U.dim() != 3 or U.shape[1] != 5 or U.shape[2] != n**3:
        raise ValueError(f"{name} must have shape (E, 5, {n**3}), got {tuple(U.shape)}")
    if not U.is_contiguous():
        raise ValueError(f"{name} must be contiguous")


def volume_cartesian(U, n, D=None, gamma=GAMMA, scale=2.0, out=None, stream=None, dynamic=True):
    """R[e,:,r] = scale sum_j sum_l D[r_j,l] F#_j(U[e,:,r], U[e,:,r(j->l)]).

    ``dynamic``: for n >= 5 the persistent kernels claim elements from a
    per-call counter (an 8-byte workspace tensor) instead of a static split;
    the results are bitwise the same.
    """
    _lib.require_cuda()
    D = _host_matrix(gll_operators(n)[1] if D is None else D, n)
    _check_states(U, n)
    if out is None:
        out = torch.empty_like(U)
    else:
        _check_states(out, n, "out")
    ws = torch.empty(1, dtype=torch.int64, device=U.device) if dynamic and n >= 5 else None
    if ws is not None and stream is not None:
        ws.record_stream(stream)  # freed on return: keep it out of reuse until the launch ran
    _lib.call(
        "sfb_euler_volume_cartesian_ws", U.shape[0], n, D.ctypes.data, float(gamma),
        float(scale), _lib.ptr(U), _lib.ptr(out), _lib.ptr(ws), _lib.stream_ptr(stream),
    )
    return out


def volume_cartesian_host(U, n, D=None, gamma=GAMMA, scale=2.0, out=None):
    """Host-buffer entry: numpy (E, 5, n^3) in, numpy out; chunked H2D/kernel/D2H.

    Use pinned buffers (``pinned_empty``) for overlapped transfers.
    """
    _lib.require_cuda()
    D = _host_matrix(gll_operators(n)[1] if D is None else D, n)
    if isinstance(U, torch.Tensor):
        if U.is_cuda or U.dtype != torch.float64 or not U.is_contiguous():
            raise ValueError("U must be a contiguous float64 host tensor (use volume_cartesian "
                             "for device tensors)")
        if tuple(U.shape[1:]) != (5, n**3):
            raise ValueError(f"U must have shape (E, 5, {n**3})")
        U_ptr, E = U.data_ptr(), U.shape[0]
        if out is None:
            out = torch.empty_like(U)
        elif (not isinstance(out, torch.Tensor) or out.is_cuda or out.shape != U.shape
              or out.dtype != torch.float64 or not out.is_contiguous()):
            raise ValueError("out must be a contiguous float64 host tensor shaped like U")
        R_ptr = out.data_ptr()
    else:
        U = np.ascontiguousarray(U, dtype=np.float64)
        E = U.shape[0]
        if U.shape != (E, 5, n**3):
            raise ValueError(f"U must have shape (E, 5, {n**3})")
        if out is None:
            out = np.empty_like(U)
        elif (not isinstance(out, np.ndarray) or out.dtype != np.float64 or out.shape != U.shape
              or not out.flags.c_contiguous or not out.flags.writeable):
            raise ValueError("out must be a writeable C-contiguous float64 ndarray shaped like U")
        U_ptr, R_ptr = U.ctypes.data, out.ctypes.data
    _lib.call(
        "sfb_euler_volume_cartesian_host", E, n, D.ctypes.data, float(gamma), float(scale),
        U_ptr, R_ptr,
    )
    return out


def pinned_empty(shape):
    """Page-locked host float64 tensor (for overlapped host<->device copies)."""
    return torch.empty(shape, dtype=torch.float64, pin_memory=True)


def generate_states(E, n, seed, e0=0, gamma=GAMMA, bounds=synth.EULER_BOUNDS, device=None):
    """Device-side seeded states, bitwise equal to synth.euler_states(E, n, seed, e0=e0)."""
    _lib.require_cuda()
    U = torch.empty((E, 5, n**3), dtype=torch.float64, device=device or "cuda")
    b = np.ascontiguousarray(bounds, dtype=np.float64)
    _lib.call(
        "sfb_generate_euler_states", E, e0, n, seed, float(gamma), b.ctypes.data, _lib.ptr(U),
        _lib.stream_ptr(),
    )
    return U


def generate_uniform(count, seed, lo, hi, i0=0, device=None):
    """Device-side seeded uniforms, bitwise equal to synth.uniform_array."""
    _lib.require_cuda()
    out = torch.empty(count, dtype=torch.float64, device=device or "cuda")
    _lib.call("sfb_generate_uniform", count, i0, seed, float(lo), float(hi), _lib.ptr(out),
              _lib.stream_ptr())
    return out


def volume_curvilinear_modal(Uhat, Ja, n, gamma=GAMMA, scale=2.0, out=None, sumsq=None,
                             stream=None, dynamic=True):
    """Config 5: Rhat = (Pi x Pi x Pi) r, r = scale sum_i (D_i o Ft_i) 1, u = (V x V x V) Uhat.

    Uhat (E, 5, n^3) modal coefficients (orthonormal Legendre), Ja (E, 3, 3, n^3)
    metric cofactors Ja[e,i,m,r] = J dxi^i/dx_m.  If ``sumsq`` (E,) is given it
    receives sum_v sum_k Rhat[e,v,k]^2 per element.  ``dynamic``: the kernel's
    CTAs claim elements from a per-call counter (an 8-byte workspace tensor)
    instead of a static split; the results are bitwise the same.
    """
    _lib.require_cuda()
    _, D, V, Pi = gll_operators(n)
    _check_states(Uhat, n, "Uhat")
    E = Uhat.shape[0]
    if (not isinstance(Ja, torch.Tensor) or not Ja.is_cuda or Ja.shape != (E, 3, 3, n**3)
            or Ja.dtype != torch.float64 or not Ja.is_contiguous()):
        raise ValueError(f"Ja must be a contiguous CUDA float64 tensor of shape (E, 3, 3, {n**3})")
    if out is None:
        out = torch.empty_like(Uhat)
    else:
        _check_states(out, n, "out")
    if sumsq is not None and (not isinstance(sumsq, torch.Tensor) or not sumsq.is_cuda
                              or sumsq.dtype != torch.float64 or sumsq.shape != (E,)
                              or not sumsq.is_contiguous()):
        raise ValueError(f"sumsq must be a contiguous CUDA float64 tensor of shape ({E},)")
    ws = torch.empty(1, dtype=torch.int64, device=Uhat.device) if dynamic else None
    if ws is not None and stream is not None:
        ws.record_stream(stream)  # freed on return: keep it out of reuse until the launch ran
    _lib.call(
        "sfb_euler_volume_curvilinear_modal", E, n, V.ctypes.data, Pi.ctypes.data, D.ctypes.data,
        float(gamma), float(scale), _lib.ptr(Uhat), _lib.ptr(Ja), _lib.ptr(out),
        _lib.ptr(sumsq), _lib.ptr(ws), _lib.stream_ptr(stream),
    )
    return out


def volume_curvilinear_modal_host(Uhat, Ja, n, gamma=GAMMA, scale=2.0, out=None, sumsq=None):
    """Config 5 from/to host buffers (CPU float64 tensors, pinned for overlapped
    copies): Uhat (E, 5, n^3) and Ja (E, 3, 3, n^3) in, Rhat (and the per-element
    sum of squares if ``sumsq`` (E,) is given) out, through the C-ABI host entry
    (chunked H2D / kernel / D2H pipeline)."""
    _lib.require_cuda()
    _, D, V, Pi = gll_operators(n)
    for name, t, shp in (("Uhat", Uhat, (5, n**3)), ("Ja", Ja, (3, 3, n**3))):
        if (not isinstance(t, torch.Tensor) or t.is_cuda or t.dtype != torch.float64
                or not t.is_contiguous() or tuple(t.shape[1:]) != shp):
            raise ValueError(f"{name} must be a contiguous float64 host tensor of shape (E, "
                             f"{', '.join(map(str, shp))})")
    E = Uhat.shape[0]
    if Ja.shape[0] != E:
        raise ValueError("Uhat and Ja element counts differ")
    if out is None:
        out = torch.empty_like(Uhat)
    for name, t, shp in (("out", out, tuple(Uhat.shape)), ("sumsq", sumsq, (E,))):
        if t is not None and (t.is_cuda or t.dtype != torch.float64 or not t.is_contiguous()
                              or tuple(t.shape) != shp):
            raise ValueError(f"{name} must be a contiguous float64 host tensor of shape {shp}")
    _lib.call("sfb_euler_volume_curvilinear_modal_host", E, n, V.ctypes.data, Pi.ctypes.data,
              D.ctypes.data, float(gamma), float(scale), Uhat.data_ptr(), Ja.data_ptr(),
              out.data_ptr(), None if sumsq is None else sumsq.data_ptr())
    return out


def generate_modal_states(E, n, seed, e0=0, device=None):
    """Device-side config-5 modal coefficients, bitwise equal to synth.modal_states."""
    _lib.require_cuda()
    U = torch.empty((E, 5, n**3), dtype=torch.float64, device=device or "cuda")
    means = np.ascontiguousarray(synth.MODAL_MEANS, dtype=np.float64)
    amps = np.ascontiguousarray(synth.MODAL_AMPS, dtype=np.float64)
    _lib.call("sfb_generate_modal_states", E, e0, n, seed, means.ctypes.data, amps.ctypes.data,
              float(synth.MODAL_C0), _lib.ptr(U), _lib.stream_ptr())
    return U


def generate_metric(E, n, seed, e0=0, K=synth.MESH_K, amp=synth.WARP_AMP, device=None):
    """Device-side warped-lattice metric cofactors (synth.metric_cofactors to ~1e-15)."""
    _lib.require_cuda()
    Ja = torch.empty((E, 3, 3, n**3), dtype=torch.float64, device=device or "cuda")
    nodes = np.ascontiguousarray(gll_operators(n)[0].nodes, dtype=np.float64)
    _lib.call("sfb_generate_metric", E, e0, n, seed, nodes.ctypes.data, K, float(amp),
              _lib.ptr(Ja), _lib.stream_ptr())
    return Ja
