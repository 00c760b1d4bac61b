"""The oracle's scan restatement (oracle/oracle.py np_*scan*) against the
reference scan module's own outputs (tests/golden/scans.npz, written by
tests/golden/make_golden.py from /root/reference scan.py:33-103)."""

import os

import numpy as np
import pytest

from oracle import oracle as O

Z = np.load(os.path.join(os.path.dirname(__file__), "golden", "scans.npz"))
CASES = sorted({k.split("__")[0] for k in Z.files})


def case_input(name):
    return Z[f"{name}__in"] if f"{name}__in" in Z.files else Z[f"{str(Z[f'{name}__in_of'])}__in"]


def oracle_call(name, x):
    kind = name.split("_")[0]
    if kind == "incl":
        return O.np_inclusive_scan(x)
    if kind == "excl":
        return O.np_exclusive_scan(x)
    if kind == "blk7":
        return O.np_blocked_scan(x, 7)
    if kind == "rows":
        return O.np_scan_axis(x, 1)
    if kind == "cols":
        return O.np_scan_axis(x, 0)
    return np.ascontiguousarray(np.asarray(x).T)


@pytest.mark.parametrize("name", CASES)
def test_oracle_scans_match_reference(name):
    x = case_input(name)
    if f"{name}__raises" in Z.files:
        exc = {"ScanOverflowError": O.ScanOverflow, "AxisError": np.exceptions.AxisError}
        with pytest.raises(exc[str(Z[f"{name}__raises"])]):
            oracle_call(name, x)
        return
    want = Z[f"{name}__out"]
    got = oracle_call(name, x)
    assert got.dtype == want.dtype and np.array_equal(got, want)
