"""The reference's dense O(n^{2d}) route on the device (sumfac/oracle.py names).

The paper's baseline forms the full n^d x n^d Kronecker factors and operand
matrices; the reference package exports that route for cross-checks and for
its benchmark (oracle.py:39-160).  Here every matrix is formed by an sm_100a
kernel (csrc/dense.cu) with the reference's product order, so the numpy
arrays returned are bitwise equal to the reference's; validation, the
capacity cap and the multiplication counter are host-side, as in the
reference.  Structural validation of a pattern (duplicate positions) uses the
pattern's host index arrays.
"""

import numpy as np
import torch

from . import _lib, counting

DEFAULT_CAPACITY = 100_000_000


def _cap(rows, cols, capacity, what):
    if rows * cols > capacity:
        raise ValueError(
            f"{what} would hold {rows * cols} entries, over the capacity cap of {capacity}"
        )


def _dev(a, dtype=torch.float64):
    _lib.require_cuda()
    return torch.from_numpy(np.ascontiguousarray(a)).to("cuda", dtype)


def _dense_of(factor):
    f = np.asarray(factor, dtype=float)
    if f.ndim == 1:
        return np.diag(f)
    if f.ndim == 2:
        return f
    raise ValueError(f"factors must be 1D or 2D, got ndim={f.ndim}")


def dense_kronecker(factors, capacity=DEFAULT_CAPACITY):
    """Full Kronecker product, factors[j] along direction j (x fastest; a 1-D
    factor is a diagonal).  Entry (r, c) = prod_j factors[j][r_j, c_j]."""
    if len(factors) == 0:
        raise ValueError("dense_kronecker needs at least one factor")
    mats = [_dense_of(f) for f in factors]
    rows = np.array([m.shape[0] for m in mats], dtype=np.int64)
    cols = np.array([m.shape[1] for m in mats], dtype=np.int64)
    R, C = int(np.prod(rows)), int(np.prod(cols))
    _cap(R, C, capacity, "dense Kronecker product")
    if len(mats) > 16:
        raise ValueError("dense_kronecker supports at most 16 factors")
    packed = _dev(np.concatenate([m.ravel() for m in mats]))
    out = torch.empty((R, C), dtype=torch.float64, device="cuda")
    _lib.call("sfb_dense_kronecker", len(mats), rows.ctypes.data, cols.ctypes.data,
              _lib.ptr(packed), _lib.ptr(out), _lib.stream_ptr())
    return out.cpu().numpy()


def dense_direction_factor(basis, weights, direction, d, capacity=DEFAULT_CAPACITY):
    """The dense factor with the m x n basis in direction `direction` and
    diag(weights) in every other slot, bitwise as assemble_basis_factors."""
    basis = np.asarray(basis, dtype=float)
    weights = np.asarray(weights, dtype=float)
    m, n = basis.shape
    if weights.shape != (n,):
        raise ValueError(f"weights shape {weights.shape} does not match ({n},)")
    if direction < 0 or direction >= d:
        raise IndexError(f"direction {direction} out of range [0, {d})")
    R, C = m * n ** (d - 1), n**d
    _cap(R, C, capacity, "dense factor")
    out = torch.empty((R, C), dtype=torch.float64, device="cuda")
    b, w = _dev(basis), _dev(weights)
    _lib.call("sfb_dense_direction_factor", m, n, d, direction, _lib.ptr(b), _lib.ptr(w),
              _lib.ptr(out), _lib.stream_ptr())
    return out.cpu().numpy()


def _as_device_matrix(a):
    if isinstance(a, torch.Tensor):
        return a.to("cuda", torch.float64).contiguous()
    return _dev(np.asarray(a, dtype=float))


def dense_hadamard(a, c, out=None):
    """Entrywise product of two dense matrices; every multiplication counted."""
    a_np, c_np = np.asarray(a, dtype=float), np.asarray(c, dtype=float)
    if a_np.ndim != 2 or a_np.shape != c_np.shape:
        raise ValueError(f"shape mismatch: {a_np.shape} vs {c_np.shape}")
    if out is not None and out.shape != a_np.shape:
        raise ValueError(f"out shape {out.shape} does not match {a_np.shape}")
    da, dc = _as_device_matrix(a_np), _as_device_matrix(c_np)
    prod = torch.empty_like(da)
    _lib.call("sfb_hadamard_evaluate", _lib.ptr(da), _lib.ptr(dc), da.numel(), _lib.ptr(prod),
              _lib.stream_ptr())
    counting.add_multiplications(a_np.size)
    if out is None:
        return prod.cpu().numpy()
    out[...] = prod.cpu().numpy()
    return out


def dense_rank_one_operand(row_values, col_values, out=None):
    """Full operand matrix C[i, j] = row_values[i] * col_values[j]."""
    rv = np.asarray(row_values, dtype=float)
    cv = np.asarray(col_values, dtype=float)
    if rv.ndim != 1 or cv.ndim != 1:
        raise ValueError("operand generators must be 1D arrays")
    shape = (rv.shape[0], cv.shape[0])
    if out is not None and out.shape != shape:
        raise ValueError(f"out shape {out.shape} does not match {shape}")
    res = torch.empty(shape, dtype=torch.float64, device="cuda")
    drv, dcv = _dev(rv), _dev(cv)
    _lib.call("sfb_dense_rank_one", _lib.ptr(drv), shape[0], _lib.ptr(dcv), shape[1],
              _lib.ptr(res), _lib.stream_ptr())
    counting.add_multiplications(shape[0] * shape[1])
    if out is None:
        return res.cpu().numpy()
    out[...] = res.cpu().numpy()
    return out


def _direction_ok(pattern, direction):
    if direction < 0 or direction >= pattern.d:
        raise IndexError(f"direction {direction} out of range [0, {pattern.d})")


def scatter(sparse, pattern, direction):
    """Dense matrix of one direction's compressed factor (a SparseFactorSet or a
    (m n^(d-1), n) array) placed at the pattern positions."""
    _direction_ok(pattern, direction)
    vals = sparse.factor(direction) if hasattr(sparse, "factor") else sparse
    vals = np.asarray(vals, dtype=float)
    want = (pattern.row_space_size, pattern.columns_size_1d)
    if vals.shape != want:
        raise ValueError(f"factor shape {vals.shape} does not match {want}")
    keys = pattern.rows[:, direction] * pattern.column_space_size + pattern.columns[:, direction]
    if np.unique(keys).size != keys.size:
        raise RuntimeError("pattern lists a (row, column) position twice; the pattern is corrupt")
    out = torch.empty((pattern.row_space_size, pattern.column_space_size), dtype=torch.float64,
                      device="cuda")
    dv = _dev(vals)
    _lib.call("sfb_scatter_direction", _lib.ptr(pattern.device_rows),
              _lib.ptr(pattern.device_columns), pattern.d, direction, pattern.entry_count,
              _lib.ptr(dv), pattern.row_space_size, pattern.column_space_size, _lib.ptr(out),
              _lib.stream_ptr())
    return out.cpu().numpy()


def gather(dense, pattern, direction):
    """One direction's compressed factor read from a dense matrix (inverse of scatter)."""
    _direction_ok(pattern, direction)
    dense = np.asarray(dense, dtype=float)
    want = (pattern.row_space_size, pattern.column_space_size)
    if dense.shape != want:
        raise ValueError(f"dense shape {dense.shape} does not match {want}")
    dd = _dev(dense)
    vals = torch.empty(pattern.entry_count, dtype=torch.float64, device="cuda")
    _lib.call("sfb_gather_direction", _lib.ptr(pattern.device_rows),
              _lib.ptr(pattern.device_columns), pattern.d, direction, pattern.entry_count,
              _lib.ptr(dd), pattern.column_space_size, _lib.ptr(vals), _lib.stream_ptr())
    return vals.cpu().numpy().reshape(pattern.row_space_size, pattern.columns_size_1d)
