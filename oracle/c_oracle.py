"""ctypes wrapper of the C oracle (TEST INFRASTRUCTURE ONLY; see oracle/__init__.py)."""

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle_c.so")
_lib = None


def build():
    subprocess.run(["make", "-s", "-C", _HERE, "liboracle_c.so"], check=True)
    return _LIB_PATH


def _load():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH) or os.access(os.path.join(_HERE, "Makefile"), os.W_OK):
            try:
                build()  # make is a no-op when the library is current
            except Exception:
                if not os.path.exists(_LIB_PATH):
                    raise
        lib = ctypes.CDLL(_LIB_PATH)
        p, i64, i, d = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_double
        lib.oracle_euler_volume_cartesian.argtypes = [i64, i, p, d, d, p, p, i]
        lib.oracle_hadamard_rowsum_batched.argtypes = [i64, i64, i, i, p, p, p, i]
        lib.oracle_euler_volume_curvilinear_modal.argtypes = [i64, i, p, p, p, d, d, p, p, p, p,
                                                              i]
        lib.oracle_euler_volume_dense.argtypes = [i64, i, p, d, d, p, p, i]
        _lib = lib
    return _lib


def euler_volume_cartesian(U, D, gamma=1.4, scale=2.0, threads=1):
    U = np.ascontiguousarray(U, dtype=np.float64)
    D = np.ascontiguousarray(D, dtype=np.float64)
    R = np.empty_like(U)
    rc = _load().oracle_euler_volume_cartesian(
        U.shape[0], D.shape[0], D.ctypes.data, gamma, scale, U.ctypes.data, R.ctypes.data, threads
    )
    if rc:
        raise ValueError("oracle_euler_volume_cartesian: bad arguments")
    return R


def hadamard_rowsum_batched(basis, F, threads=1):
    basis = np.ascontiguousarray(basis, dtype=np.float64)
    F = np.ascontiguousarray(F, dtype=np.float64)
    d, R, n = basis.shape
    E = F.shape[0]
    out = np.empty((E, R))
    rc = _load().oracle_hadamard_rowsum_batched(
        E, R, n, d, basis.ctypes.data, F.ctypes.data, out.ctypes.data, threads
    )
    if rc:
        raise ValueError("oracle_hadamard_rowsum_batched: bad arguments")
    return out


def euler_volume_curvilinear_modal(Uhat, Ja, V, Pi, D, gamma=1.4, scale=2.0, threads=1):
    """Config 5 (euler_oracle.euler_volume_curvilinear_modal in C): (Rhat, sumsq)."""
    Uhat = np.ascontiguousarray(Uhat, dtype=np.float64)
    Ja = np.ascontiguousarray(Ja, dtype=np.float64)
    V, Pi, D = (np.ascontiguousarray(a, dtype=np.float64) for a in (V, Pi, D))
    E, n = Uhat.shape[0], D.shape[0]
    if Uhat.shape != (E, 5, n**3) or Ja.shape != (E, 3, 3, n**3):
        raise ValueError("Uhat (E, 5, n^3) and Ja (E, 3, 3, n^3) expected")
    Rhat = np.empty_like(Uhat)
    ss = np.empty(E)
    rc = _load().oracle_euler_volume_curvilinear_modal(
        E, n, V.ctypes.data, Pi.ctypes.data, D.ctypes.data, gamma, scale, Uhat.ctypes.data,
        Ja.ctypes.data, Rhat.ctypes.data, ss.ctypes.data, threads)
    if rc:
        raise ValueError("oracle_euler_volume_curvilinear_modal: bad arguments")
    return Rhat, ss


def euler_volume_dense(U, D, gamma=1.4, scale=2.0, threads=1):
    """The dense O(n^{2d}) route of the config-3 volume term (oracle.py:54-112 applied
    to the Chandrashekar operand): every entry of the n^d x n^d factor and flux
    matrices is formed, zeros included."""
    U = np.ascontiguousarray(U, dtype=np.float64)
    D = np.ascontiguousarray(D, dtype=np.float64)
    R = np.empty_like(U)
    rc = _load().oracle_euler_volume_dense(U.shape[0], D.shape[0], D.ctypes.data, gamma, scale,
                                           U.ctypes.data, R.ctypes.data, threads)
    if rc:
        raise ValueError("oracle_euler_volume_dense: bad arguments")
    return R
