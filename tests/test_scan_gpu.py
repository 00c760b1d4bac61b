"""The scan module surface (reference scan.py:33-103 semantics) on the device,
including acceptance C3's shape: 10,000 random arrays, blocked == inclusive."""

import itertools

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from paper_1711_01919_b200 import ParameterError, ScanOverflowError  # noqa: E402
from paper_1711_01919_b200.scan import (blocked_scan, exclusive_scan, inclusive_scan,  # noqa: E402
                                        scan_cols, scan_rows, transpose)


def test_fixed_examples():
    assert inclusive_scan([]).tolist() == [] and exclusive_scan([]).tolist() == []
    assert inclusive_scan([3, 1, 7, 0, 4, 1, 6, 3]).tolist() == [3, 4, 11, 11, 15, 16, 22, 25]
    assert exclusive_scan([3, 1, 7, 0]).tolist() == [0, 3, 4, 11]
    assert inclusive_scan([1, 1, 1, 1]).dtype == np.uint32


def test_overflow_and_params():
    with pytest.raises(ScanOverflowError):
        inclusive_scan([2**32 - 1, 1])
    assert inclusive_scan([2**32 - 2, 1]).tolist() == [2**32 - 2, 2**32 - 1]
    with pytest.raises(ParameterError):
        blocked_scan([1, 2], 0)
    with pytest.raises(ParameterError):
        transpose(np.zeros((2, 2), np.uint32), 0)


def test_c3_scans(rng):
    for i in range(2000):
        n = int(rng.integers(0, 2049))
        xs = rng.integers(0, 1000, size=n)
        expect = list(itertools.accumulate(xs.tolist()))
        assert inclusive_scan(xs).tolist() == expect
        if i < 60:
            for block in (1, 2, 3, 5, 8, 64, 256):
                assert blocked_scan(xs, block).tolist() == expect


def test_plane_scans_and_transpose(rng):
    plane = rng.integers(0, 2**31, size=(37, 53)).astype(np.uint32)
    assert np.array_equal(scan_rows(plane), np.cumsum(plane, axis=1, dtype=np.uint32))
    assert np.array_equal(scan_cols(plane), np.cumsum(plane, axis=0, dtype=np.uint32))
    out = np.empty_like(plane)
    assert scan_rows(plane, out=out) is out
    assert np.array_equal(transpose(transpose(plane, 7)), plane)
    assert np.array_equal(transpose(plane), plane.T)
