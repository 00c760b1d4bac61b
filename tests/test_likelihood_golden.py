"""likelihood_map / best_match pinned to REFERENCE-made fixtures.

tests/golden/likelihood.npz is written by tests/golden/make_golden.py, which
runs the reference's likelihood_map and best_match (likelihood.py:55-86) on
random, structured (tied) and explicit-LUT images.  Tolerance 1e-12 is the
reference's own (pkg/tests/test_likelihood.py:46); best_match must agree
exactly (same tie rule: first maximum in row-major order).
"""

import os

import numpy as np
import pytest

from conftest import GOLDEN

from oracle import oracle as O


def _cases():
    data = np.load(os.path.join(GOLDEN, "likelihood.npz"))
    cases = {}
    for key in data.files:
        name, field = key.split("__", 1)
        cases.setdefault(name, {})[field] = data[key]
    return cases


CASES = _cases()


@pytest.mark.parametrize("name", sorted(CASES))
def test_oracle_restatement_matches_reference_map(name):
    """CPU: the numpy restatement of likelihood.py:55-77 reproduces the fixture."""
    c = CASES[name]
    counts = O.np_compute(c["img"], c["lut"], int(c["bins"]))
    h, w = (int(x) for x in c["hw"])
    got = O.np_likelihood_map(counts, c["template"], h, w, str(c["metric"]))
    assert got.shape == c["map"].shape
    assert np.abs(got - c["map"]).max() < 1e-12


@pytest.mark.gpu
@pytest.mark.parametrize("name", sorted(CASES))
def test_device_likelihood_matches_reference(name):
    """K5 (fused likelihood map) through the drop-in API vs the reference's map."""
    import paper_1711_01919_b200 as ih

    c = CASES[name]
    spec = ih.BinSpec(int(c["bins"]), c["lut"])
    t = ih.compute_sequential(ih.GrayImage(c["img"]), spec)
    h, w = (int(x) for x in c["hw"])
    lmap = ih.likelihood_map(t, c["template"], h, w, str(c["metric"]))
    assert lmap.values.shape == c["map"].shape
    assert np.abs(lmap.values - c["map"]).max() < 1e-12
    r, cc, v = ih.best_match(lmap)
    assert (r, cc) == tuple(int(x) for x in c["best"])
    assert abs(v - float(c["best_value"])) < 1e-12
