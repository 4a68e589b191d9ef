"""The host-side x-fastest layout contract (indexing.py; reference
sumfac/indexing.py:17-84): the index math every kernel hard-codes."""

import itertools

import numpy as np
import pytest

from paper_2306_11665_b200 import TensorLayout, flatten, unflatten
from paper_2306_11665_b200.kernel import SparsityPattern


@pytest.mark.parametrize("extents", [(5,), (4, 4), (4, 4, 4), (2, 3, 5), (3, 1, 2, 2), (6, 6, 6)])
def test_flatten_unflatten_bijection(extents):
    lay = TensorLayout(extents)
    assert lay.size == int(np.prod(extents))
    seen = set()
    for multi in itertools.product(*(range(e) for e in extents)):
        f = flatten(multi, lay)
        assert unflatten(f, lay) == tuple(multi)
        seen.add(f)
    assert seen == set(range(lay.size))


def test_direction_zero_is_fastest():
    lay = TensorLayout((4, 4, 4))
    assert lay.strides == (1, 4, 16)
    # the kernels' node index r = r0 + r1 n + r2 n^2 and r(j -> l)
    for r in range(64):
        digits = unflatten(r, lay)
        assert r == digits[0] + 4 * digits[1] + 16 * digits[2]
        for j, l in itertools.product(range(3), range(4)):
            moved = list(digits)
            moved[j] = l
            assert flatten(moved, lay) == r + (l - digits[j]) * 4**j


def test_rectangular_row_layout_matches_pattern():
    # SparsityPattern.row_layout puts extent m in slot j (kernel.py:58-66)
    p = SparsityPattern(3, 5, 3, np.zeros((1, 3), np.int64), np.zeros((1, 3), np.int64))
    assert p.row_layout(1).extents == (5, 3, 5)
    assert p.column_layout().extents == (5, 5, 5)
    with pytest.raises(IndexError):
        p.row_layout(3)


def test_errors():
    lay = TensorLayout((2, 3))
    with pytest.raises(IndexError):
        flatten((2, 0), lay)
    with pytest.raises(IndexError):
        flatten((0, -1), lay)
    with pytest.raises(ValueError):
        flatten((0, 0, 0), lay)
    with pytest.raises(IndexError):
        unflatten(6, lay)
    with pytest.raises(IndexError):
        unflatten(-1, lay)
    for bad in ((), (0, 3), (-2,)):
        with pytest.raises(ValueError):
            TensorLayout(bad)
    with pytest.raises(ValueError):
        TensorLayout((2**40, 2**40))


def test_equality_and_hash():
    assert TensorLayout((2, 3)) == TensorLayout([2, 3])
    assert TensorLayout((2, 3)) != TensorLayout((3, 2))
    assert len({TensorLayout((2, 3)), TensorLayout((2, 3))}) == 1
    assert "TensorLayout" in repr(TensorLayout((2,)))
