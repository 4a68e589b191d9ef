"""ctypes binding of the C ABI in ``include/sumfac_b200.h``.

The shared library is built in-tree (``build.py``); importing this module
never falls back to a CPU path.  If ``libsumfac_b200.so`` is missing the
import raises, and every entry point raises if CUDA is unavailable, so a GPU
run without the native code fails loudly instead of silently computing
elsewhere.
"""

import ctypes
import os

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SFB_LIB") or os.path.join(_HERE, "libsumfac_b200.so")

SFB_OK = 0
SFB_EINVAL = 1
SFB_ECUDA = 2
SFB_ENOTSUP = 3

FLUX_PRODUCT = 0
FLUX_BURGERS_EC = 1
FLUX_BURGERS_AVG = 2

_i64 = ctypes.c_int64
_u64 = ctypes.c_uint64
_int = ctypes.c_int
_dbl = ctypes.c_double
_p = ctypes.c_void_p

# name -> argtypes (restype is int unless listed in _RESTYPES)
SIGNATURES = {
    "sfb_last_error": [],
    "sfb_version": [],
    "sfb_launch_count": [],
    "sfb_fill_pattern": [_i64, _i64, _i64, _p, _p, _p],
    "sfb_assemble_basis": [_p, _p, _p, _p, _i64, _i64, _i64, _p, _p],
    "sfb_assemble_two_point": [_p, _p, _p, _p, _i64, _i64, _i64, _int, _p, _p],
    "sfb_gather_dense": [_p, _p, _p, _i64, _i64, _i64, _p, _p],
    "sfb_hadamard_evaluate": [_p, _p, _i64, _p, _p],
    "sfb_hadamard_row_sum": [_p, _i64, _i64, _p, _p],
    "sfb_hadamard_rowsum_batched": [_i64, _i64, _i64, _i64, _p, _p, _p, _p, _p],
    "sfb_hadamard_rowsum_batched_host": [_i64, _i64, _i64, _i64, _p, _p, _p],
    "sfb_burgers_volume": [_i64, _i64, _i64, _p, _p, _int, _p, _p, _p],
    "sfb_burgers_time_derivative": [_i64, _i64, _i64, _p, _p, _dbl, _dbl, _int, _p, _p, _p],
    "sfb_burgers_rk4": [_i64, _i64, _i64, _p, _p, _dbl, _dbl, _int, _dbl, _i64, _i64, _p, _p, _p,
                        _p],
    "sfb_kronecker_apply": [_i64, _i64, _p, _p, _p, _p, _p, _p],
    "sfb_dense_kronecker": [_i64, _p, _p, _p, _p, _p],
    "sfb_dense_direction_factor": [_i64, _i64, _i64, _i64, _p, _p, _p, _p],
    "sfb_dense_rank_one": [_p, _i64, _p, _i64, _p, _p],
    "sfb_scatter_direction": [_p, _p, _i64, _i64, _i64, _p, _i64, _i64, _p, _p],
    "sfb_gather_direction": [_p, _p, _i64, _i64, _i64, _p, _i64, _p, _p],
    "sfb_kronecker_pass": [_i64, _i64, _i64, _i64, _i64, _int, _p, _p, _p, _p],
    "sfb_euler_volume_cartesian": [_i64, _i64, _p, _dbl, _dbl, _p, _p, _p],
    "sfb_euler_volume_cartesian_ws": [_i64, _i64, _p, _dbl, _dbl, _p, _p, _p, _p],
    "sfb_euler_volume_cartesian_host": [_i64, _i64, _p, _dbl, _dbl, _p, _p],
    "sfb_euler_volume_curvilinear_modal": [
        _i64, _i64, _p, _p, _p, _dbl, _dbl, _p, _p, _p, _p, _p, _p,
    ],
    "sfb_euler_volume_curvilinear_modal_host": [
        _i64, _i64, _p, _p, _p, _dbl, _dbl, _p, _p, _p, _p,
    ],
    "sfb_block_sums": [_p, _i64, _i64, _p, _p],
    "sfb_generate_euler_states": [_i64, _i64, _i64, _u64, _dbl, _p, _p, _p],
    "sfb_generate_uniform": [_i64, _i64, _u64, _dbl, _dbl, _p, _p],
    "sfb_generate_modal_states": [_i64, _i64, _i64, _u64, _p, _p, _dbl, _p, _p],
    "sfb_generate_metric": [_i64, _i64, _i64, _u64, _p, _i64, _dbl, _p, _p],
}
_RESTYPES = {
    "sfb_last_error": ctypes.c_char_p,
    "sfb_launch_count": ctypes.c_int64,
}


class NativeError(RuntimeError):
    """A CUDA-side failure reported through the C ABI."""


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'` "
            "(there is no CPU fallback for this package)"
        )
    lib = ctypes.CDLL(LIB_PATH)
    for name, argtypes in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.argtypes = argtypes
        fn.restype = _RESTYPES.get(name, ctypes.c_int)
    return lib


LIB = _load()


def last_error():
    msg = LIB.sfb_last_error()
    return msg.decode() if msg else ""


def launch_count():
    return int(LIB.sfb_launch_count())


def require_cuda():
    if not torch.cuda.is_available():
        raise RuntimeError(
            "paper_2306_11665_b200 computes on a B200 only: CUDA is not available "
            "(no CPU fallback exists by design)"
        )


def call(name, *args):
    """Invoke an ``sfb_*`` entry point and map its status to an exception."""
    rc = getattr(LIB, name)(*args)
    if rc == SFB_OK:
        return
    msg = last_error()
    if rc == SFB_EINVAL:
        raise ValueError(f"{name}: {msg}")
    if rc == SFB_ENOTSUP:
        raise NotImplementedError(f"{name}: {msg}")
    raise NativeError(f"{name}: {msg}")


def ptr(t):
    """Device (or host) address of a contiguous tensor / ndarray, or None."""
    if t is None:
        return None
    if isinstance(t, torch.Tensor):
        if not t.is_contiguous():
            raise ValueError("tensor must be contiguous")
        if t.is_cuda and t.device.index != torch.cuda.current_device():
            # the library launches on the current device (C ABI convention)
            raise ValueError(f"tensor on {t.device} but the current device is "
                             f"cuda:{torch.cuda.current_device()} (use torch.cuda.device)")
        return t.data_ptr()
    # numpy array (host pointer)
    if not t.flags["C_CONTIGUOUS"]:
        raise ValueError("array must be C-contiguous")
    return t.ctypes.data


def stream_ptr(stream=None):
    s = torch.cuda.current_stream() if stream is None else stream
    return s.cuda_stream
