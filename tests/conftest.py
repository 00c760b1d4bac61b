import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: long-running (large tensors)")


def has_cuda() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if has_cuda():
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container (run under gpurun)")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


@pytest.fixture
def rng():
    """Same seed as the reference's test fixture (tests/conftest.py:30-32)."""
    return np.random.default_rng(20260823)


@pytest.fixture(scope="session")
def golden_c1():
    with open(os.path.join(GOLDEN, "c1_instances.json")) as fh:
        return json.load(fh)


@pytest.fixture(scope="session")
def golden_configs():
    with open(os.path.join(GOLDEN, "configs.json")) as fh:
        return json.load(fh)


@pytest.fixture(scope="session")
def golden_small():
    data = np.load(os.path.join(GOLDEN, "small_cases.npz"))
    cases = {}
    for key in data.files:
        name, field = key.split("__", 1)
        cases.setdefault(name, {})[field] = data[key]
    return cases


def c1_images(count=200):
    """Regenerate the acceptance-C1 instance stream (reference
    tests/test_acceptance.py:48-75, seed 20260823): yields (w, h, bins, tile, pixels)."""
    seed = 20260823
    widths = [1, 2, 3, 5, 17, 33, 64, 97, 131, 257]
    heights = [1, 2, 7, 19, 33, 61, 96, 128, 193]
    bins_choices = [1, 2, 3, 16, 64]
    tiles = [1, 7, 64]
    rng = np.random.default_rng(seed)
    inst = [(1, 1, 1, 1), (1, 1, 64, 64), (257, 193, 16, 64), (257, 193, 64, 7)]
    while len(inst) < count:
        inst.append((int(rng.choice(widths)), int(rng.choice(heights)),
                     int(rng.choice(bins_choices)), int(rng.choice(tiles))))
    for w, h, b, t in inst:
        yield w, h, b, t, rng.integers(0, 256, size=(h, w), dtype=np.uint8)
