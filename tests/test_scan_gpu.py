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


# --- K6 kernels against the reference's own outputs (tests/golden/scans.npz) --

import os  # noqa: E402

import torch  # noqa: E402

from paper_1711_01919_b200 import scan as S  # noqa: E402

_Z = np.load(os.path.join(os.path.dirname(__file__), "golden", "scans.npz"))
_CASES = sorted({k.split("__")[0] for k in _Z.files})


def _input(name):
    key = f"{name}__in" if f"{name}__in" in _Z.files else f"{str(_Z[f'{name}__in_of'])}__in"
    return _Z[key]


def _call(name, x):
    kind = name.split("_")[0]
    fn = {"incl": S.inclusive_scan, "excl": S.exclusive_scan, "rows": S.scan_rows,
          "cols": S.scan_cols, "tr": S.transpose}.get(kind)
    return S.blocked_scan(x, 7) if kind == "blk7" else fn(x)


@pytest.mark.parametrize("name", _CASES)
def test_device_scans_match_reference_golden(name):
    x = _input(name)
    if f"{name}__raises" in _Z.files:
        exc = {"ScanOverflowError": ScanOverflowError, "AxisError": np.exceptions.AxisError}
        with pytest.raises(exc[str(_Z[f"{name}__raises"])]):
            _call(name, x)
        return
    want = _Z[f"{name}__out"]
    got = _call(name, x)
    assert isinstance(got, np.ndarray) and got.dtype == want.dtype and np.array_equal(got, want)


def test_device_tensor_inputs_stay_on_device(rng):
    """CUDA tensors in -> CUDA tensors out; unaligned views take the scalar
    load / store paths of k6_scan_apply."""
    base = torch.from_numpy(rng.integers(0, 1000, 70001)).cuda()
    for off in (0, 1, 3):
        v = base[off:]
        got = S.inclusive_scan(v)
        assert got.is_cuda and got.dtype == torch.uint32
        assert np.array_equal(got.cpu().numpy(), np.cumsum(v.cpu().numpy()).astype(np.uint32))
        ex = S.exclusive_scan(v).cpu().numpy()
        assert ex[0] == 0 and np.array_equal(ex[1:], got.cpu().numpy()[:-1])
    plane = torch.from_numpy(rng.integers(0, 256, (300, 777), dtype=np.uint8)).cuda()
    host = plane.cpu().numpy()
    assert np.array_equal(S.scan_rows(plane).cpu().numpy(), np.cumsum(host, 1, dtype=np.uint32))
    assert np.array_equal(S.scan_cols(plane).cpu().numpy(), np.cumsum(host, 0, dtype=np.uint32))
    assert torch.equal(S.transpose(S.transpose(plane)), plane)
    out = torch.empty((300, 777), dtype=torch.uint32, device="cuda")
    assert S.scan_rows(plane, out=out) is out


def test_large_scan_properties():
    """Size-independent checks at 3*10^8 elements (> 146k tiles, the one-CTA
    totals scan loops): ones -> 1..n; a single 2^32-n element overflows at
    the very last prefix only."""
    n = 300_000_000
    ones = torch.ones(n, dtype=torch.int64, device="cuda")
    got = S.inclusive_scan(ones)
    ar = torch.arange(1, n + 1, dtype=torch.int64, device="cuda")
    assert torch.equal(got.to(torch.int64), ar)
    assert torch.equal(S.exclusive_scan(ones).to(torch.int64), ar - 1)
    del got, ar
    ones[n // 2] = 2**32 - n + 1  # the last inclusive prefix is exactly 2^32
    with pytest.raises(ScanOverflowError):
        S.inclusive_scan(ones)
    assert int(S.exclusive_scan(ones)[-1]) == 2**32 - 1  # exclusive stops one short


def test_transpose_large_rows_grid():
    """More than 65535 row bands (the grid-strided y loop) and odd extents."""
    a = torch.randint(0, 2**15, (65536 * 32 + 17, 3), dtype=torch.int16, device="cuda")
    t = S.transpose(a)
    assert torch.equal(t, a.t().contiguous())


def test_repeated_calls(rng):
    """Back-to-back calls on one stream (the overflow flag and tile totals are
    reset per call), sizes from one tile to many."""
    for n in (1, 2047, 2048, 2049, 100_000, 3_000_001, 7):
        x = torch.from_numpy(rng.integers(0, 1000, n)).cuda()
        want = np.cumsum(x.cpu().numpy()).astype(np.uint32)
        for _ in range(3):
            assert np.array_equal(S.inclusive_scan(x).cpu().numpy(), want), n
