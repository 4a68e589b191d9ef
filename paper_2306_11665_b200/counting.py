"""Analytic multiplication counter and allocation ledger.

Host-side mirror of the reference's accounting (sumfac/counting.py:18-55).
The drop-in must tally exactly what the reference tallies, because the
reference's tests assert exact counts (Theorem 1's d*n^(d+1), the pattern's
2*entries*d, the memory bound 6*d*n^(d+1)).  The GPU kernels do not count;
each Python entry point adds the analytic number of multiplications its
algorithm performs, the same number the reference adds.  Not thread-safe,
like the reference.
"""

_state = {"mul": 0, "alloc": 0}


def reset_multiplication_count():
    """Zero the multiplication tally."""
    _state["mul"] = 0


def multiplication_count():
    """Scalar multiplications tallied since the last reset."""
    return _state["mul"]


def add_multiplications(count):
    if count < 0:
        raise ValueError(f"multiplication count must be nonnegative, got {count}")
    _state["mul"] += int(count)


def reset_allocation_ledger():
    """Zero the allocation ledger."""
    _state["alloc"] = 0


def allocated_numbers():
    """Scalars materialised by kernel containers since the last reset."""
    return _state["alloc"]


def register_allocation(count):
    if count < 0:
        raise ValueError(f"allocation size must be nonnegative, got {count}")
    _state["alloc"] += int(count)
