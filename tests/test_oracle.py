"""The oracle (oracle/, test infrastructure) pinned against the reference's own
outputs: golden fixtures made by tests/golden/make_golden.py with the
reference package, and SURVEY.md Appendix A.  CPU only."""

import zlib

import numpy as np
import pytest

from conftest import c1_images
from oracle import oracle as O


def test_c1_instances_match_reference(golden_c1):
    """All 200 acceptance-C1 instances: C sequential == C crossweave == reference crc."""
    for (w, h, b, tile, px), gold in zip(c1_images(200), golden_c1):
        assert (w, h, b, tile) == (gold["w"], gold["h"], gold["bins"], gold["tile"])
        assert f"{zlib.crc32(px.tobytes()):08x}" == gold["img_crc"]
        lut = O.np_uniform_table(b)
        seq = O.compute_sequential(px, lut, b)
        assert O.tensor_checksum(seq) == gold["crc"]
        for workers in (1, 3):
            assert O.compute_crossweave(px, lut, b, workers).tobytes() == seq.tobytes()


def test_numpy_restatement_matches_c(golden_c1):
    for (w, h, b, tile, px), gold in list(zip(c1_images(200), golden_c1))[:60]:
        t = O.np_compute(px, O.np_uniform_table(b), b)
        assert O.tensor_checksum(t) == gold["crc"]


@pytest.mark.parametrize("key", ["64x64x16", "512x512x32", "1920x1080x32"])
def test_config_checksums(golden_configs, key):
    w, h, b = (int(x) for x in key.split("x"))
    img = O.synth_image(w, h, 0)
    assert f"{zlib.crc32(img.tobytes()):08x}" == golden_configs[key]["img_crc"]
    t = O.compute_crossweave(img, O.np_uniform_table(b), b)
    assert O.tensor_checksum(t) == golden_configs[key]["crc"]


def test_hd_frames_first_four(golden_configs):
    lut = O.np_uniform_table(32)
    for k in range(4):
        t = O.compute_crossweave(O.synth_image(1920, 1080, k), lut, 32)
        assert O.tensor_checksum(t) == golden_configs["1920x1080x32_frames"][k]


def test_plane_crc_streams_whole_tensor_crc(golden_configs):
    """Per-plane streamed crc chained over planes == whole-tensor checksum."""
    img = O.synth_image(512, 512, 0)
    lut = O.np_uniform_table(32)
    crc = 0
    for b in range(32):
        crc = O.plane_crc32(img, lut, b, crc)
    assert f"{crc:08x}" == golden_configs["512x512x32"]["crc"]


@pytest.mark.slow
def test_8k_plane_crcs_appendix_a(golden_configs):
    """Two planes of the 8192x8192x256 tensor against SURVEY.md Appendix A
    (reference compute_streamed); O(W) memory."""
    img = O.synth_image(8192, 8192, 0)
    lut = O.np_uniform_table(256)
    planes = golden_configs["8192x8192x256"]["plane_crc"]
    for b in (0, 255):
        assert f"{O.plane_crc32(img, lut, b):08x}" == planes[b]


def test_small_cases_exact(golden_small):
    for name, case in golden_small.items():
        px, lut, bins = case["img"], case["lut"], int(case["bins"])
        gold = case["counts"]
        assert np.array_equal(O.compute_sequential(px, lut, bins), gold), name
        assert np.array_equal(O.compute_crossweave(px, lut, bins), gold), name
        assert np.array_equal(O.np_compute(px, lut, bins), gold), name
        if "regions" in case:
            got = O.region_histograms(gold, case["regions"])
            assert np.array_equal(got, case["region_counts"]), name
            for k, reg in enumerate(case["regions"]):
                assert np.array_equal(O.np_region_histogram(gold, *reg), case["region_counts"][k])
        for key in case:
            if key.startswith("win_"):
                h, w = (int(x) for x in key[4:].split("x"))
                assert np.array_equal(O.window_counts(gold, h, w), case[key]), (name, key)
                assert np.array_equal(O.np_window_counts(gold, h, w), case[key]), (name, key)


def test_known_answers():
    """Reference tests/test_strategies.py:39-61 known answers."""
    t = O.compute_sequential(np.array([[0, 255], [128, 0]], np.uint8), O.np_uniform_table(2), 2)
    assert t[0, 1, 1] == 2 and t[1, 1, 1] == 2
    rng = np.random.default_rng(1)
    t = O.compute_sequential(rng.integers(0, 256, (4, 6), dtype=np.uint8), O.np_uniform_table(1), 1)
    assert (t[0] == np.arange(1, 5)[:, None] * np.arange(1, 7)[None, :]).all()


def test_brute_force_tiny(rng):
    for _ in range(10):
        w, h = int(rng.integers(1, 8)), int(rng.integers(1, 8))
        px = rng.integers(0, 256, (h, w), dtype=np.uint8)
        b = int(rng.choice([1, 2, 3, 16]))
        lut = O.np_uniform_table(b)
        assert np.array_equal(O.compute_sequential(px, lut, b),
                              O.brute_integral_histogram(px, lut, b))
