"""Documentation that runs: the reference-side ctypes stub of INTEGRATION.md §2, executed
verbatim (its relative imports pointed at this package's mirror types and its
library path at the in-tree .so) against the oracle."""

import os
import re

import numpy as np
import pytest

from conftest import ROOT
from oracle import oracle as O

pytestmark = pytest.mark.gpu


def test_integration_ctypes_stub_runs():
    text = open(os.path.join(ROOT, "INTEGRATION.md")).read()
    code = re.search(r"```python\n(# inthist/_b200\.py.*?)```", text, re.S).group(1)
    code = code.replace("from .core import", "from paper_1711_01919_b200.core import")
    code = code.replace("from .errors import", "from paper_1711_01919_b200.errors import")
    code = code.replace('ctypes.CDLL("libinthist_b200.so")',
                        'ctypes.CDLL(%r)' % os.path.join(ROOT, "paper_1711_01919_b200",
                                                        "libinthist_b200.so"))
    code = code.replace('ctypes.CDLL("libcudart.so")', 'ctypes.CDLL("libcudart.so.12")')
    ns = {}
    exec(compile(code, "INTEGRATION.md:_b200.py", "exec"), ns)
    import paper_1711_01919_b200 as ih

    rng = np.random.default_rng(5)
    for (h, w, b) in [(90, 333, 16), (1080, 1920, 32), (7, 5, 3)]:
        img = ih.GrayImage(rng.integers(0, 256, (h, w), dtype=np.uint8))
        spec = ih.BinSpec.uniform(b)
        got = ns["compute_sequential"](img, spec).counts
        assert np.array_equal(got, O.compute_crossweave(img.pixels, spec.table, b)), (h, w, b)


@pytest.mark.parametrize("doc", ["README.md", "INTEGRATION.md"])
def test_drop_in_snippets_run(doc):
    """The drop-in snippets of README.md and INTEGRATION.md §1 run as written."""
    text = open(os.path.join(ROOT, doc)).read()
    code = re.search(r"```python\n(import paper_1711_01919_b200 as inthist.*?)```", text, re.S).group(1)
    pixels = np.random.default_rng(1).integers(0, 256, (120, 200), dtype=np.uint8)
    ns = {"pixels_u8": pixels}
    exec(compile(code, doc, "exec"), ns)
    want = O.brute_region_counts(pixels, O.np_uniform_table(32), 32, 10, 20, 59, 99)
    assert np.array_equal(ns["h"].counts, want)
