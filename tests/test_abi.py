"""The C-ABI library: builds, loads without a GPU, exports every symbol the
header declares, and validates arguments in the reference's error order
before touching the device (so these run on CPU)."""

import ctypes
import os
import re

import numpy as np
import pytest

from conftest import ROOT
from paper_1711_01919_b200 import _native
from paper_1711_01919_b200.errors import CapacityError, ParameterError, ShapeError

HEADER = os.path.join(ROOT, "include", "inthist_b200.h")


def header_functions():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(ih_[a-z_0-9]+)\s*\(", text)))


def test_header_and_binding_agree():
    assert header_functions() == sorted(_native.EXPORTS)


def test_library_exports_every_header_symbol():
    L = _native.lib()
    for name in header_functions():
        assert hasattr(L, name), name
    assert L.ih_abi_version() >> 16 == 1


def test_library_is_sm100a():
    """The shared library carries sm_100a SASS (cuobjdump lists the cubin arch)."""
    import shutil
    import subprocess

    tool = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(tool):
        pytest.skip("cuobjdump not available")
    out = subprocess.run([tool, "--list-elf", _native.LIB_PATH], capture_output=True, text=True)
    assert "sm_100a" in out.stdout


def test_status_strings():
    L = _native.lib()
    for code in range(6):
        assert L.ih_status_string(code).decode().startswith("IH_")


def _call(**kw):
    L = _native.lib()
    lut = kw.pop("lut", np.zeros(256, np.uint8))
    args = dict(img=1, frames=1, H=4, W=4, pitch=4, fstride=16, bins=2, lo=0, hi=2, out=1,
                ws=0, ws_bytes=0, kernel=0, stream=0)
    args.update(kw)
    return L.ih_integral_histogram(
        args["img"], args["frames"], args["H"], args["W"], args["pitch"], args["fstride"],
        lut.ctypes.data, args["bins"], args["lo"], args["hi"], args["out"], args["ws"],
        args["ws_bytes"], args["kernel"], args["stream"])


def test_validation_order_without_device():
    assert _call(H=0) == _native.IH_ERR_SHAPE
    assert _call(bins=0) == _native.IH_ERR_SHAPE
    assert _call(bins=257) == _native.IH_ERR_SHAPE
    assert _call(lut=np.full(256, 2, np.uint8)) == _native.IH_ERR_SHAPE
    assert _call(lo=1, hi=1) == _native.IH_ERR_SHAPE
    # capacity: W*H > 2^32-1 (core.py:53-57) before parameter errors
    assert _call(H=1 << 16, W=(1 << 16) + 1, pitch=0) == _native.IH_ERR_CAPACITY
    assert _call(pitch=3) == _native.IH_ERR_PARAM
    assert _call(kernel=7) == _native.IH_ERR_PARAM
    # column-tiled single pass: the row carries need a workspace
    assert _call(W=20000, pitch=20000, kernel=_native.KERNEL_SINGLE_PASS) == _native.IH_ERR_PARAM


def test_status_maps_to_reference_exceptions():
    with pytest.raises(ShapeError):
        _native.check(_call(H=0))
    with pytest.raises(CapacityError):
        _native.check(_call(H=1 << 16, W=(1 << 16) + 1, pitch=0))
    with pytest.raises(ParameterError):
        _native.check(_call(pitch=3))


def test_window_and_region_validation():
    L = _native.lib()
    assert L.ih_window_counts(1, 2, 4, 4, 0, 1, 1, 0) == _native.IH_ERR_PARAM
    assert L.ih_window_counts(1, 2, 4, 4, 5, 1, 1, 0) == _native.IH_ERR_BOUNDS
    assert L.ih_region_histograms(1, 0, 4, 4, 1, 1, 1, 0) == _native.IH_ERR_SHAPE
    assert L.ih_region_histograms(1, 2, 4, 4, 16, 0, 1, 0) == _native.IH_OK  # Q = 0: no-op


def test_workspace_plan():
    L = _native.lib()
    # frames are split into row segments until ~4 waves of CTAs exist; the
    # carry table is (frames, nseg, nbp, Wp) u16
    for frames in (1, 8, 64):
        n = L.ih_workspace_bytes(frames, 1080, 1920, 32, 0)
        assert n > 0 and n % (frames * 32 * 1920 * 2) == 0
    # tiny problems with few rows need no carries
    assert L.ih_workspace_bytes(1, 20, 64, 4, 0) == 0
    # cross-weave needs none
    assert L.ih_workspace_bytes(1, 1080, 1920, 32, _native.KERNEL_CROSSWEAVE) == 0
    # column tiles (W > 2048): k2_rowleft's (T-1, H, nbp) u32 row carries; 20000
    # columns -> 10 tiles of 2048 (16 chunks) ... as even as possible
    n = L.ih_workspace_bytes(1, 16, 20000, 8, 0)
    assert n >= 9 * 16 * 8 * 4


def test_column_tile_plan():
    """W > 2048 splits rows into column tiles of <= 16 chunks, as even as possible."""
    from paper_1711_01919_b200 import device

    p = device.plan(1, 2160, 3840, 128)
    assert (p["kernel"], p["column_tiles"], p["tile_width"], p["chunks_per_lane"]) == \
        ("single_pass", 2, 1920, 1)
    p = device.plan(1, 8192, 8192, 32)
    assert (p["column_tiles"], p["tile_width"]) == (4, 2048)
    p = device.plan(64, 1080, 1920, 32)
    assert (p["column_tiles"], p["tile_width"]) == (1, 1920)
    p = device.plan(1, 3, 30001, 4)
    assert p["column_tiles"] * p["tile_width"] >= 30001 and p["tile_width"] <= 2048


def test_plan_hint_overrides_segments():
    """ih_plan_hint pins the row-segment count for one shape only; 0 removes it."""
    from paper_1711_01919_b200 import device

    base = device.plan(8, 1080, 1920, 32)["segments"]
    device.set_plan_hint(8, 1080, 1920, 32, 5)
    try:
        assert device.plan(8, 1080, 1920, 32)["segments"] == 5
        assert device.plan(8, 1080, 1920, 16)["segments"] == device.plan(8, 1080, 1920, 16)["segments"]
        assert device.plan(9, 1080, 1920, 32)["segments"] != 5 or base == 5
    finally:
        device.set_plan_hint(8, 1080, 1920, 32, 0)
    assert device.plan(8, 1080, 1920, 32)["segments"] == base
    cands = device.segment_candidates(8, 1080, 1920, 32)
    assert base in cands and all(1 <= n <= 34 for n in cands)


def test_plan_variants_on_cpu(monkeypatch):
    """Planner decisions that need no device: row packing for 1-/2-bin slabs,
    tail splits from hints, hint validation."""
    from paper_1711_01919_b200 import device
    from paper_1711_01919_b200.errors import ParameterError as PE

    p1 = device.plan(64, 1080, 1920, 1)
    p4 = device.plan(64, 1080, 1920, 4)
    assert p1["workspace_bytes"] * 4 == p4["workspace_bytes"]  # KB = 1: nbp = 1 (not 4)
    monkeypatch.setenv("IH_NO_ROWPACK", "1")
    assert device.plan(64, 1080, 1920, 1)["workspace_bytes"] == p4["workspace_bytes"]
    monkeypatch.delenv("IH_NO_ROWPACK")
    device.set_plan_hint(4, 1000, 700, 9, 6, 30, 4)
    try:
        p = device.plan(4, 1000, 700, 9)
        assert p["big_segments"] < p["segments"] and p["tail_segment_rows"] * 4 >= p["segment_rows"] - 3
    finally:
        device.set_plan_hint(4, 1000, 700, 9, 0)
    with pytest.raises(PE):
        device.set_plan_hint(4, 1000, 700, 9, 6, 120, 4)
    with pytest.raises(PE):
        device.set_plan_hint(4, 1000, 700, 9, -1)


def test_plan_cache_follows_knobs_and_hints(monkeypatch):
    """Plans are cached per (IH_* fingerprint, hint generation, shape): a knob
    or hint change between calls takes effect on the next call."""
    from paper_1711_01919_b200 import device

    base = device.plan(8, 1080, 1920, 32)["segments"]
    monkeypatch.setenv("IH_NSEG", "7")
    assert device.plan(8, 1080, 1920, 32)["segments"] == 7
    monkeypatch.setenv("IH_NSEG", "11")
    assert device.plan(8, 1080, 1920, 32)["segments"] == 11
    monkeypatch.delenv("IH_NSEG")
    assert device.plan(8, 1080, 1920, 32)["segments"] == base
    device.set_plan_hint(8, 1080, 1920, 32, 5)
    try:
        assert device.plan(8, 1080, 1920, 32)["segments"] == 5
    finally:
        device.set_plan_hint(8, 1080, 1920, 32, 0)
    assert device.plan(8, 1080, 1920, 32)["segments"] == base


def test_skewed_segment_plans(monkeypatch):
    """Skewed segments: the first pct % of the segments are larger by
    skew/100, the plan still covers every row, and the hint flag form equals
    the environment form."""
    from paper_1711_01919_b200 import device

    monkeypatch.setenv("IH_NSEG", "37")
    monkeypatch.setenv("IH_SKEW_X100", "125")
    p = device.plan(1, 2160, 3840, 16)
    S, nbig, S2, n = p["segment_rows"], p["big_segments"], p["tail_segment_rows"], p["segments"]
    assert nbig == 19 and S2 == S * 100 // 125 and nbig * S + (n - nbig - 1) * S2 < 2160 <= nbig * S + (n - nbig) * S2
    monkeypatch.delenv("IH_SKEW_X100")
    monkeypatch.delenv("IH_NSEG")
    device.set_plan_hint(1, 2160, 3840, 16, 37, 50, 125, skew=True)
    try:
        q = device.plan(1, 2160, 3840, 16)
        assert (q["segment_rows"], q["big_segments"], q["tail_segment_rows"], q["segments"]) == (S, nbig, S2, n)
    finally:
        device.set_plan_hint(1, 2160, 3840, 16, 0)


def test_k2s_plans(monkeypatch):
    """The one-launch small-image kernel: planned for <= 4 bin groups of one
    small frame, forced by IH_SMALL=1, off with IH_SMALL=0, never for column
    tiles or unaligned rows; its workspace holds the flags and aggregates."""
    from paper_1711_01919_b200 import device

    p = device.plan(1, 512, 512, 16)
    assert (p["carry"], p["launches"]) == ("in_kernel", 1)
    assert p["workspace_bytes"] > 0
    assert device.plan(1, 512, 512, 32)["carry"] == "table"
    assert device.plan(1, 512, 512, 16, aligned16=False)["carry"] != "in_kernel"
    assert device.plan(1, 512, 4096, 4)["carry"] != "in_kernel"
    monkeypatch.setenv("IH_SMALL", "1")
    assert device.plan(1, 512, 512, 32)["carry"] == "in_kernel"
    monkeypatch.setenv("IH_SMALL", "0")
    assert device.plan(1, 512, 512, 16)["carry"] != "in_kernel"


def test_bins_per_cta_plans(monkeypatch):
    """Bin pairs (two rows per packed word) for >= 24 bins on aligned rows
    wider than 512 with >= 256 bin pairs over the frames; quads otherwise;
    1-/2-bin slabs pack rows; IH_KB and the hint flags choose explicitly."""
    from paper_1711_01919_b200 import device

    kb = lambda *a, **k: device.plan(*a, **k)["bins_per_cta"]  # noqa: E731
    assert kb(64, 1080, 1920, 32) == 2      # 64 x 16 pairs
    assert kb(16, 1080, 1920, 32) == 2      # 16 x 16 = 256
    assert kb(8, 1080, 1920, 32) == 4       # 8 x 16 = 128: quads
    assert kb(64, 1080, 1920, 16) == 4      # < 24 bins
    assert kb(64, 512, 512, 32) == 4        # 512-wide rows
    assert kb(64, 1080, 1918, 32) == 4      # unaligned output rows
    assert kb(1, 8192, 8192, 256) == 4      # column tiles
    assert kb(64, 1080, 1920, 1) == 1 and kb(64, 1080, 1920, 2) == 2
    q, p = device.plan(8, 1080, 1920, 32), device.plan(64, 1080, 1920, 32)
    monkeypatch.setenv("IH_KB", "2")
    assert kb(8, 1080, 1920, 32) == 2
    monkeypatch.setenv("IH_KB", "4")
    assert kb(64, 1080, 1920, 32) == 4
    monkeypatch.delenv("IH_KB")
    device.set_plan_hint(8, 1080, 1920, 32, q["segments"], kb=2)
    device.set_plan_hint(64, 1080, 1920, 32, p["segments"], kb=4)
    try:
        assert kb(8, 1080, 1920, 32) == 2 and kb(64, 1080, 1920, 32) == 4
    finally:
        device.set_plan_hint(8, 1080, 1920, 32, 0)
        device.set_plan_hint(64, 1080, 1920, 32, 0)
    assert kb(8, 1080, 1920, 32) == 4 and kb(64, 1080, 1920, 32) == 2
