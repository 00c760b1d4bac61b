"""Parity of the CUDA path against the reference (golden fixtures) and the
oracle, bit-exact, through the C ABI.  Needs a B200: run with -m gpu."""

import os
import zlib

import numpy as np
import pytest

from conftest import c1_images
from oracle import oracle as O

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

import paper_1711_01919_b200 as ih  # noqa: E402
from paper_1711_01919_b200 import device  # noqa: E402


def crc_of(t) -> str:
    a = t.cpu().numpy() if hasattr(t, "cpu") else t
    return f"{zlib.crc32(np.ascontiguousarray(a).view(np.uint32).tobytes()):08x}"


@pytest.fixture(autouse=True)
def _clean_env(monkeypatch):
    for k in ("IH_NSEG", "IH_ROWS_PER_BATCH", "IH_TARGET_WARPS", "IH_MIN_SEG_ROWS", "IH_NO_TMA",
              "IH_CARRY_LOOKBACK", "IH_TABLE_SUM_MAX", "IH_NO_COLTILE", "IH_NO_BIG", "IH_COLCOUNTS_SLAB", "IH_K4_MODE", "IH_K5_DIRECT", "IH_TAIL_PCT", "IH_TAIL_DIV", "IH_CARRY_CLUSTER", "IH_NO_RESTAGE", "IH_NO_ROWPACK"):
        monkeypatch.delenv(k, raising=False)


def dev_compute(px, lut, bins, kernel="auto", bin_range=None):
    d = device.upload_image(px)
    return device.integral_histogram(d, lut, bins, bin_range=bin_range, kernel=kernel)


# --------------------------------------------------------------------- C1 / C7
def test_c1_every_strategy_matches_reference(golden_c1):
    """Acceptance C1 (test_acceptance.py:68-83): 200 seeded instances, every
    strategy byte-identical to the reference's compute_sequential."""
    for (w, h, b, tile, px), gold in zip(c1_images(200), golden_c1):
        img = ih.GrayImage(px)
        spec = ih.BinSpec.uniform(b)
        for res in (ih.compute_sequential(img, spec), ih.compute_crossweave(img, spec),
                    ih.compute_sts(img, spec), ih.compute_wavefront(img, spec, tile)):
            assert crc_of(res.counts) == gold["crc"], (w, h, b, tile)


def test_c7_worker_caps_do_not_change_output(golden_c1):
    for (w, h, b, tile, px), gold in list(zip(c1_images(200), golden_c1))[:16]:
        img, spec = ih.GrayImage(px), ih.BinSpec.uniform(b)
        for workers in (1, 2, 8):
            assert crc_of(ih.compute_crossweave(img, spec, workers).counts) == gold["crc"]
            assert crc_of(ih.compute_wavefront(img, spec, tile, workers).counts) == gold["crc"]


# ------------------------------------------------------------ golden small cases
@pytest.mark.parametrize("kernel", ["auto", "single_pass", "crossweave"])
def test_small_cases_exact(golden_small, kernel):
    for name, case in golden_small.items():
        px, lut, bins = case["img"], case["lut"], int(case["bins"])
        got = dev_compute(px, lut, bins, kernel=kernel).cpu().numpy()
        assert np.array_equal(got, case["counts"]), (name, kernel)


def test_small_case_queries(golden_small):
    for name, case in golden_small.items():
        t = dev_compute(case["img"], case["lut"], int(case["bins"]))
        if "regions" in case:
            got = device.region_histograms(t, case["regions"]).cpu().numpy()
            assert np.array_equal(got, case["region_counts"]), name
        for key in case:
            if key.startswith("win_"):
                h, w = (int(x) for x in key[4:].split("x"))
                got = device.window_counts(t, h, w).cpu().numpy()
                assert np.array_equal(got, case[key]), (name, key)


def test_known_answers():
    img = ih.GrayImage(np.array([[0, 255], [128, 0]], dtype=np.uint8))
    t = ih.compute_sequential(img, ih.BinSpec.uniform(2)).counts
    assert t[0, 1, 1] == 2 and t[1, 1, 1] == 2
    img = ih.GrayImage(np.full((3, 5), 200, dtype=np.uint8))
    t = ih.compute_sequential(img, ih.BinSpec.uniform(4)).counts
    hit = (200 * 4) // 256
    assert t[hit, -1, -1] == 15 and not np.delete(t, hit, axis=0).any()
    one = ih.GrayImage(np.array([[77]], dtype=np.uint8))
    for s in (ih.SEQUENTIAL, ih.CROSSWEAVE, ih.SCAN_TRANSPOSE_SCAN, ih.wavefront(1)):
        t = ih.compute(one, ih.BinSpec.uniform(16), s).counts
        assert t.sum() == 1 and t[(77 * 16) // 256, 0, 0] == 1


# ----------------------------------------------- kernel-internal paths vs oracle
SHAPES = [(1, 1), (1, 193), (193, 1), (7, 131), (61, 257), (128, 128), (96, 500),
          (300, 1030), (45, 2049), (33, 4100), (20, 8192)]


@pytest.mark.parametrize("nseg", [0, 2, 3, 7])
@pytest.mark.parametrize("rows_per_batch", [1, 2, 4])
@pytest.mark.parametrize("tma", [True, False])
@pytest.mark.parametrize("carry", ["lookback", "table_sum", "table_prefix", "cluster"])
def test_segments_and_batches(monkeypatch, rng, nseg, rows_per_batch, tma, carry):
    """Force K2 row segmentation (colcounts/colprefix/carry-init path), every
    barrier batch size, and both input paths (TMA smem ring / LDG); compare
    with the oracle bit for bit."""
    if nseg:
        monkeypatch.setenv("IH_NSEG", str(nseg))
    monkeypatch.setenv("IH_ROWS_PER_BATCH", str(rows_per_batch))
    if not tma:
        monkeypatch.setenv("IH_NO_TMA", "1")
    if carry == "lookback":
        monkeypatch.setenv("IH_CARRY_LOOKBACK", "1")
    elif carry == "table_prefix":
        monkeypatch.setenv("IH_TABLE_SUM_MAX", "1")  # always run k2_colprefix
    elif carry == "cluster":
        monkeypatch.setenv("IH_CARRY_CLUSTER", "1")  # DSMEM carries where the plan allows
    for (h, w) in SHAPES:
        bins = int(rng.choice([1, 3, 5, 16, 64]))
        px = rng.integers(0, 256, (h, w), dtype=np.uint8)
        lut = O.np_uniform_table(bins)
        got = dev_compute(px, lut, bins, kernel="single_pass").cpu().numpy()
        assert np.array_equal(got, O.compute_crossweave(px, lut, bins)), (h, w, bins)


@pytest.mark.parametrize("nseg", [0, 40, 200])
@pytest.mark.parametrize("lookback", [False, True])
def test_auto_segmentation_sizes(monkeypatch, rng, nseg, lookback):
    """Real sizes with many segments (look-back chains up to 200 long)."""
    if nseg:
        monkeypatch.setenv("IH_NSEG", str(nseg))
    if lookback:
        monkeypatch.setenv("IH_CARRY_LOOKBACK", "1")
    for (h, w) in [(1080, 1920), (2160, 640), (500, 64)]:
        for bins in (1, 4, 32):
            px = rng.integers(0, 256, (h, w), dtype=np.uint8)
            lut = O.np_uniform_table(bins)
            got = dev_compute(px, lut, bins).cpu().numpy()
            assert np.array_equal(got, O.compute_crossweave(px, lut, bins)), (h, w, bins)


def test_tall_image_sum_mode(rng):
    """H > 65535: u16 prefixes impossible, the scan sums 16-bit count slots."""
    px = rng.integers(0, 256, (70001, 5), dtype=np.uint8)
    lut = O.np_uniform_table(3)
    got = dev_compute(px, lut, 3).cpu().numpy()
    assert np.array_equal(got, O.compute_crossweave(px, lut, 3))


@pytest.mark.parametrize("restage", [True, False])
def test_unaligned_rows_and_odd_widths(monkeypatch, rng, restage):
    """ALIGNED=false (odd pitch / offset) and VEC=false (W % 4 != 0) paths:
    through the device API's 16-byte restaging (TMA path) and, with
    IH_NO_RESTAGE=1, the kernels' own unaligned (LDG) path."""
    if not restage:
        monkeypatch.setenv("IH_NO_RESTAGE", "1")
    for (h, w, bins) in [(37, 101, 16), (64, 255, 7), (19, 1025, 64), (5, 3, 2)]:
        base = rng.integers(0, 256, (h, w + 7), dtype=np.uint8)
        px = np.ascontiguousarray(base[:, 3:3 + w])
        lut = O.np_uniform_table(bins)
        expect = O.compute_crossweave(px, lut, bins)
        dbase = torch.from_numpy(base).cuda()
        view = dbase[:, 3:3 + w]  # pitch w+7, 3-byte offset
        for kernel in ("single_pass", "crossweave"):
            got = device.integral_histogram(view, lut, bins, kernel=kernel).cpu().numpy()
            assert np.array_equal(got, expect), (h, w, bins, kernel)


def test_explicit_tables_and_256_bins(rng):
    for bins in (2, 7, 100, 256):
        tab = rng.integers(0, bins, 256).astype(np.uint8)
        tab[0] = bins - 1
        spec = ih.BinSpec.explicit(tab)
        px = rng.integers(0, 256, (77, 333), dtype=np.uint8)
        for kernel in ("single_pass", "crossweave"):
            got = dev_compute(px, spec.table, spec.bins, kernel=kernel).cpu().numpy()
            assert np.array_equal(got, O.compute_crossweave(px, spec.table, spec.bins))


def test_bin_slabs_match_slices(rng):
    from paper_1711_01919_b200 import sharding

    px = rng.integers(0, 256, (200, 700), dtype=np.uint8)
    lut = O.np_uniform_table(37)
    full = O.compute_crossweave(px, lut, 37)
    for world in (2, 3, 8):
        for lo, hi in sharding.bin_slabs(37, world):
            if hi > lo:
                for kernel in ("single_pass", "crossweave"):
                    got = dev_compute(px, lut, 37, kernel=kernel, bin_range=(lo, hi))
                    assert np.array_equal(got.cpu().numpy(), full[lo:hi]), (world, lo, hi)


def test_frames_batch(rng):
    frames = rng.integers(0, 256, (5, 67, 130), dtype=np.uint8)
    lut = O.np_uniform_table(9)
    t = ih.compute_frames(frames, ih.BinSpec.uniform(9))
    assert t.shape == (5, 9, 67, 130)
    for f in range(5):
        assert np.array_equal(t[f].cpu().numpy(), O.compute_crossweave(frames[f], lut, 9))


def test_wide_image_without_column_tiles_falls_back_to_crossweave(monkeypatch, rng):
    monkeypatch.setenv("IH_NO_COLTILE", "1")
    assert device.plan(1, 3, 10000, 6)["kernel"] == "crossweave"
    px = rng.integers(0, 256, (3, 10000), dtype=np.uint8)
    lut = O.np_uniform_table(6)
    got = dev_compute(px, lut, 6).cpu().numpy()
    assert np.array_equal(got, O.compute_crossweave(px, lut, 6))


COLT_SHAPES = [(1, 2049), (3, 2177), (33, 4100), (70, 3840), (20, 8192), (9, 10000),
               (130, 6001), (2, 30001)]


@pytest.mark.parametrize("nseg", [0, 1, 3, 30])
@pytest.mark.parametrize("tma", [True, False])
@pytest.mark.parametrize("rows_per_batch", [1, 4])
def test_column_tiles(monkeypatch, rng, nseg, tma, rows_per_batch):
    """Column-tiled K2 (W > 2048): k2_rowleft row carries + the carry table summed
    left of each tile, with and without row segments, TMA and LDG inputs,
    ragged last tiles, every width up to 30001 through the single pass."""
    if nseg:
        monkeypatch.setenv("IH_NSEG", str(nseg))
    if not tma:
        monkeypatch.setenv("IH_NO_TMA", "1")
    monkeypatch.setenv("IH_ROWS_PER_BATCH", str(rows_per_batch))
    for (h, w) in COLT_SHAPES:
        bins = int(rng.choice([1, 4, 7, 32, 256]))
        px = rng.integers(0, 256, (h, w), dtype=np.uint8)
        lut = O.np_uniform_table(bins)
        p = device.plan(1, h, w, bins)
        assert p["kernel"] == "single_pass", (h, w)
        got = dev_compute(px, lut, bins, kernel="single_pass").cpu().numpy()
        assert np.array_equal(got, O.compute_crossweave(px, lut, bins)), (h, w, bins)


@pytest.mark.parametrize("slab_counts", [False, True])
def test_colcounts_variants_256_bins(monkeypatch, rng, slab_counts):
    """Carry tables from k2_colcounts_all (one pass, shared atomics, all bins)
    and from the per-32-bin-slab k2_colcounts; 256 bins, explicit LUTs, bin
    slabs whose padding takes the out-of-slab marker."""
    if slab_counts:
        monkeypatch.setenv("IH_COLCOUNTS_SLAB", "1")
    monkeypatch.setenv("IH_NSEG", "5")
    for (h, w) in [(300, 1000), (97, 2500), (64, 130)]:
        px = rng.integers(0, 256, (h, w), dtype=np.uint8)
        for bins, rng_ in [(256, None), (256, (3, 256)), (100, (0, 99)), (33, (1, 33))]:
            lut = O.np_uniform_table(bins) if bins == 256 else rng.integers(0, bins, 256).astype(np.uint8)
            full = O.compute_crossweave(px, lut, bins)
            got = dev_compute(px, lut, bins, kernel="single_pass", bin_range=rng_).cpu().numpy()
            lo, hi = rng_ or (0, bins)
            assert np.array_equal(got, full[lo:hi]), (h, w, bins, rng_)


@pytest.mark.parametrize("tail", ["10:4", "30:2", "50:8"])
@pytest.mark.parametrize("carry", ["table", "prefix", "lookback", "cluster"])
def test_tail_segments(monkeypatch, rng, tail, carry):
    """Non-uniform row segmentation (big segments, then short tail segments
    run last by the segment-major grid) under every carry scheme, with and
    without column tiles and frame batches."""
    pct, div = tail.split(":")
    monkeypatch.setenv("IH_TAIL_PCT", pct)
    monkeypatch.setenv("IH_TAIL_DIV", div)
    monkeypatch.setenv("IH_NSEG", "6")
    if carry == "prefix":
        monkeypatch.setenv("IH_TABLE_SUM_MAX", "1")
    elif carry == "lookback":
        monkeypatch.setenv("IH_CARRY_LOOKBACK", "1")
    elif carry == "cluster":
        monkeypatch.setenv("IH_CARRY_CLUSTER", "1")
    for (F, h, w, bins) in [(1, 500, 700, 16), (3, 257, 300, 5), (1, 300, 4100, 32), (2, 130, 2500, 9)]:
        frames = rng.integers(0, 256, (F, h, w), dtype=np.uint8)
        lut = O.np_uniform_table(bins)
        p = device.plan(F, h, w, bins)
        assert p["segments"] >= 6
        got = device.integral_histogram(torch.from_numpy(frames).cuda(), lut, bins,
                                        kernel="single_pass").cpu().numpy()
        for f in range(F):
            assert np.array_equal(got[f], O.compute_crossweave(frames[f], lut, bins)), (F, h, w, bins, f)


def test_column_tiles_unaligned_slabs_and_frames(rng):
    """Column tiles with an odd pitch / byte offset (LDG rows), bin slabs and a
    frame batch; constant columns stress the row-carry atomics."""
    h, w, bins = 41, 5003, 37
    base = rng.integers(0, 256, (h, w + 5), dtype=np.uint8)
    base[:, :900] = 200  # one bin hit by every pixel of the left tile
    px = np.ascontiguousarray(base[:, 1:1 + w])
    lut = O.np_uniform_table(bins)
    full = O.compute_crossweave(px, lut, bins)
    view = torch.from_numpy(base).cuda()[:, 1:1 + w]
    got = device.integral_histogram(view, lut, bins, kernel="single_pass").cpu().numpy()
    assert np.array_equal(got, full)
    from paper_1711_01919_b200 import sharding
    for lo, hi in sharding.bin_slabs(bins, 4):
        got = dev_compute(px, lut, bins, kernel="single_pass", bin_range=(lo, hi))
        assert np.array_equal(got.cpu().numpy(), full[lo:hi]), (lo, hi)
    frames = rng.integers(0, 256, (3, 50, 4500), dtype=np.uint8)
    t = ih.compute_frames(frames, ih.BinSpec.uniform(9))
    for f in range(3):
        assert np.array_equal(t[f].cpu().numpy(), O.compute_crossweave(frames[f], O.np_uniform_table(9), 9))


# ------------------------------------------------------- BASELINE configs (golden)
@pytest.mark.parametrize("key", ["64x64x16", "512x512x32", "1920x1080x32", "3840x2160x128"])
def test_config_checksums(golden_configs, key):
    w, h, b = (int(x) for x in key.split("x"))
    img = O.synth_image(w, h, 0)
    for kernel in ("auto", "crossweave"):
        assert crc_of(dev_compute(img, O.np_uniform_table(b), b, kernel=kernel)) == \
            golden_configs[key]["crc"], kernel


def test_hd_64_frame_batch(golden_configs):
    frames = np.stack([O.synth_image(1920, 1080, k) for k in range(64)])
    t = ih.compute_frames(frames, ih.BinSpec.uniform(32))
    torch.cuda.synchronize()
    got = [crc_of(t[k]) for k in range(64)]
    assert got == golden_configs["1920x1080x32_frames"]
    # analytic invariants (acceptance C2) on the device for the whole batch
    s = t.view(torch.int32).sum(dim=1, dtype=torch.int64)
    rr = torch.arange(1, 1081, device=t.device)[:, None]
    cc = torch.arange(1, 1921, device=t.device)[None, :]
    assert bool((s == rr * cc).all())


def test_4k_bin_sharded_slabs(golden_configs):
    from paper_1711_01919_b200 import sharding

    img = O.synth_image(3840, 2160, 0)
    lut = O.np_uniform_table(128)
    for world in (2, 4, 8):
        crc = 0
        for lo, hi in sharding.bin_slabs(128, world):
            t = dev_compute(img, lut, 128, bin_range=(lo, hi))
            crc = zlib.crc32(t.cpu().numpy().tobytes(), crc)
        assert f"{crc:08x}" == golden_configs["3840x2160x128"]["crc"], world


# ------------------------------------------------------------- queries / matching
def test_c4_region_queries(rng):
    """Acceptance C4 (test_acceptance.py:121-141) + batched form."""
    for _ in range(10):
        w, h = int(rng.integers(1, 120)), int(rng.integers(1, 90))
        bins = int(rng.choice([1, 2, 3, 16, 64]))
        px = rng.integers(0, 256, (h, w), dtype=np.uint8)
        img, spec = ih.GrayImage(px), ih.BinSpec.uniform(bins)
        t = ih.compute_sequential(img, spec)
        regs = []
        for _ in range(100):
            r0, r1 = sorted(rng.integers(0, h, 2).tolist())
            c0, c1 = sorted(rng.integers(0, w, 2).tolist())
            regs.append((r0, c0, r1, c1))
        got = ih.region_histogram_batch(t, regs)
        dev_t = device.integral_histogram(device.upload_image(px), spec.table, bins)
        pre = torch.empty((len(regs), bins), dtype=torch.uint64, device="cuda")
        assert device.region_histograms(dev_t, regs, out=pre) is pre
        assert np.array_equal(pre.cpu().numpy(), got)
        for k, (r0, c0, r1, c1) in enumerate(regs[:20]):
            one = ih.region_histogram(t, ih.Region(r0, c0, r1, c1)).counts
            assert np.array_equal(one, got[k])
        for k, (r0, c0, r1, c1) in enumerate(regs):
            assert np.array_equal(got[k], O.brute_region_counts(px, spec.table, bins, r0, c0, r1, c1))
    with pytest.raises(ih.BoundsError):
        ih.region_histogram(t, ih.Region(0, 0, h, 0))


def test_window_counts_vs_oracle(rng):
    px = rng.integers(0, 256, (90, 170), dtype=np.uint8)
    lut = O.np_uniform_table(12)
    full = O.compute_crossweave(px, lut, 12)
    t = ih.IntegralHistogram(full)
    for (h, w) in [(1, 1), (8, 8), (64, 64), (90, 170), (13, 1), (1, 170)]:
        assert np.array_equal(ih.window_counts(t, h, w), O.window_counts(full, h, w)), (h, w)
    with pytest.raises(ih.ParameterError):
        ih.window_counts(t, 0, 3)
    with pytest.raises(ih.BoundsError):
        ih.window_counts(t, 91, 3)


@pytest.mark.parametrize("metric", ["intersection", "bhattacharyya"])
def test_likelihood_map_brute(rng, metric):
    """Acceptance C6 (test_acceptance.py:166-190), tolerance 1e-12."""
    px = rng.integers(0, 256, (30, 40), dtype=np.uint8)
    img, spec = ih.GrayImage(px), ih.BinSpec.uniform(16)
    t = ih.compute_sequential(img, spec)
    template = ih.normalize(ih.region_histogram(t, ih.Region(10, 12, 17, 19)))
    lmap = ih.likelihood_map(t, template, 8, 8, metric)
    assert lmap.values.shape == (23, 33)
    for r in range(23):
        for c in range(33):
            q = O.brute_region_counts(px, spec.table, 16, r, c, r + 7, c + 7).astype(np.float64) / 64
            exp = ih.intersection(template, q) if metric == "intersection" else ih.bhattacharyya(template, q)[0]
            assert abs(lmap.values[r, c] - exp) < 1e-12
    assert abs(lmap.values[10, 12] - 1.0) < 1e-12
    r, c, v = ih.best_match(lmap)
    assert (r, c) == (10, 12) or v <= lmap.values[10, 12] + 1e-12


def test_streamed_equals_sequential(rng):
    """Acceptance C5 shape (test_acceptance.py:144-163)."""
    px = rng.integers(0, 256, (256, 256), dtype=np.uint8)
    img, spec = ih.GrayImage(px), ih.BinSpec.uniform(64)
    plan = ih.plan_tiles(256, 256, 64, 80_000)
    assert len(plan.bin_chunks) >= 4 and plan.strips >= 4
    sink = ih.ArraySink(256, 256, 64)
    summary = ih.compute_streamed(img, spec, plan, sink)
    assert np.array_equal(sink.counts, O.compute_crossweave(px, spec.table, 64))
    assert summary.peak_bytes <= 80_000


@pytest.mark.parametrize("budget", [40_000, 200_000, 3_000_000, 50_000_000])
def test_streamed_overlap_paths(rng, budget):
    """f2 overlap: single vs double staging buffers, per-plane strip copies vs
    whole-slab copies, chunk look-ahead; the sink sees every piece in the
    reference's order and peak_bytes is the measured staging, within budget."""
    px = rng.integers(0, 256, (181, 203), dtype=np.uint8)
    img, spec = ih.GrayImage(px), ih.BinSpec.uniform(48)
    plan = ih.plan_tiles(203, 181, 48, budget)
    order = []

    class Sink(ih.ArraySink):
        def write(self, lo, hi, r0, r1, data):
            order.append((lo, r0))
            super().write(lo, hi, r0, r1, data)

    sink = Sink(203, 181, 48)
    summary = ih.compute_streamed(img, spec, plan, sink)
    assert np.array_equal(sink.counts, O.compute_crossweave(px, spec.table, 48))
    assert order == [(lo, r0) for lo, _ in plan.bin_chunks for r0 in range(0, 181, plan.strip_height)]
    assert summary.peak_bytes <= budget
    assert summary.strips == len(plan.bin_chunks) * plan.strips


def test_wavefront_trace_dependency_order(rng):
    px = rng.integers(0, 256, (50, 70), dtype=np.uint8)
    trace = []
    ih.compute_wavefront(ih.GrayImage(px), ih.BinSpec.uniform(4), 16, workers=4, trace=trace)
    ni, nj = -(-50 // 16), -(-70 // 16)
    started = [e[1:] for e in trace if e[0] == "start"]
    assert sorted(started) == sorted((i, j) for i in range(ni) for j in range(nj))
    done = set()
    for ev, i, j in trace:
        if ev == "start":
            assert i == 0 or (i - 1, j) in done
            assert j == 0 or (i, j - 1) in done
        else:
            done.add((i, j))


@pytest.mark.parametrize("shape,tile,bins", [((50, 70), 16, 4), ((1, 1), 1, 1), ((33, 17), 1, 3),
                                             ((61, 97), 7, 16), ((193, 257), 64, 64),
                                             ((40, 40), 1000, 256), ((130, 300), 33, 37)])
def test_wavefront_kernel_real_trace(rng, shape, tile, bins):
    """K7 (the wavefront as scheduled on the device): tensor bit-identical to the
    oracle, and the recorded events are a real interleaving -- a permutation
    of 0..2n-1 in which every tile starts after its upper and left neighbours
    finished (strategies.py:180-181 contract)."""
    H, W = shape
    px = rng.integers(0, 256, shape, dtype=np.uint8)
    lut = O.np_uniform_table(bins)
    counts, ev = device.wavefront(device.upload_image(px), lut, bins, tile)
    assert np.array_equal(counts.cpu().numpy(), O.compute_sequential(px, lut, bins))
    ni, nj = -(-H // tile), -(-W // tile)
    e = ev.cpu().numpy()
    assert e.shape == (ni * nj, 2)
    assert sorted(e.ravel().tolist()) == list(range(2 * ni * nj))
    s, f = e[:, 0].reshape(ni, nj), e[:, 1].reshape(ni, nj)
    assert (f > s).all()
    assert (s[1:, :] > f[:-1, :]).all() and (s[:, 1:] > f[:, :-1]).all()


def test_wavefront_trace_is_recorded_not_synthesised(rng):
    """The trace of a wide image shows tiles of one anti-diagonal overlapping in
    time (a synthesised per-diagonal start*/finish* list never interleaves a
    later diagonal's start before an earlier diagonal's last finish)."""
    px = rng.integers(0, 256, (64, 1024), dtype=np.uint8)
    trace = []
    t = ih.compute_wavefront(ih.GrayImage(px), ih.BinSpec.uniform(8), 8, trace=trace)
    assert np.array_equal(t.counts, O.compute_sequential(px, O.np_uniform_table(8), 8))
    pos = {(k, i, j): n for n, (k, i, j) in enumerate(trace)}
    ni, nj = 8, 128
    diag_last_finish = {}
    for (k, i, j), n in pos.items():
        if k == "finish":
            d = i + j
            diag_last_finish[d] = max(diag_last_finish.get(d, -1), n)
    overlapped = sum(1 for (k, i, j), n in pos.items()
                     if k == "start" and i + j > 0 and n < diag_last_finish[i + j - 1])
    assert overlapped > 0


def test_native_library_is_the_one_loaded():
    from paper_1711_01919_b200 import _native

    maps = open(f"/proc/{os.getpid()}/maps").read()
    assert _native.LIB_PATH in maps


@pytest.mark.parametrize("frames,h,w,bins", [(4, 270, 480, 32), (1, 1080, 1920, 32), (2, 100, 3000, 17)])
def test_cuda_graph_capture_and_streams(frames, h, w, bins, rng):
    """The whole call (row-segment prepass + scan) is stream-ordered and
    graph-capturable: capture once on a side stream, replay with new pixels."""
    lut = O.np_uniform_table(bins)
    imgs = torch.from_numpy(rng.integers(0, 256, (frames, h, w), dtype=np.uint8)).cuda()
    out = device.empty_output(frames, bins, h, w, imgs.device)
    device.integral_histogram(imgs, lut, bins, out=out)  # warm-up: workspace, attributes
    torch.cuda.synchronize()
    side = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=side):
        device.integral_histogram(imgs, lut, bins, out=out)
    for _ in range(2):
        new = rng.integers(0, 256, (frames, h, w), dtype=np.uint8)
        imgs.copy_(torch.from_numpy(new))
        g.replay()
        torch.cuda.synchronize()
        for f in range(frames):
            assert np.array_equal(out[f].cpu().numpy(), O.compute_crossweave(new[f], lut, bins))


def test_autotune_pins_a_measured_segment_count(rng):
    """device.autotune times candidate row-segment counts and pins the fastest;
    the pinned plan still produces the oracle's tensor."""
    res = device.autotune(3, 300, 700, 12)
    try:
        assert str(res["segments"]) in {k.split("/")[0] for k in res["ms"]}
        p = device.plan(3, 300, 700, 12)
        assert p["segments"] >= res["segments"]
        assert (p["big_segments"] < p["segments"]) == (res["tail_pct"] > 0)
        frames = rng.integers(0, 256, (3, 300, 700), dtype=np.uint8)
        t = ih.compute_frames(frames, ih.BinSpec.uniform(12))
        for f in range(3):
            assert np.array_equal(t[f].cpu().numpy(), O.compute_crossweave(frames[f], O.np_uniform_table(12), 12))
    finally:
        device.set_plan_hint(3, 300, 700, 12, 0)


def test_tuning_save_and_load(tmp_path):
    """autotune results persist across processes: save_tuning / load_tuning
    (keyed by GPU model and ABI version)."""
    res = device.autotune(2, 200, 300, 7)
    path = str(tmp_path / "tune.json")
    try:
        assert device.save_tuning(path) >= 1
        want = device.plan(2, 200, 300, 7)
        device.set_plan_hint(2, 200, 300, 7, 0)
        assert device.load_tuning(path) >= 1
        assert device.plan(2, 200, 300, 7) == want
        assert want["big_segments"] >= 1 and res["segments"] >= 1
    finally:
        device.set_plan_hint(2, 200, 300, 7, 0)


def test_plan_describe_matches_launches():
    p = device.plan(64, 1080, 1920, 32)
    assert p["kernel"] == "single_pass" and p["launches"] in (1, 2, 3)
    assert p["segments"] * p["segment_rows"] >= 1080
    assert device.plan(1, 4, 20000, 8)["kernel"] == "single_pass"  # column tiles
    assert device.workspace_bytes(64, 1080, 1920, 32) >= p["workspace_bytes"]


def test_out_argument_and_int32_view(rng):
    px = rng.integers(0, 256, (50, 70), dtype=np.uint8)
    lut = O.np_uniform_table(5)
    out = torch.zeros((1, 5, 50, 70), dtype=torch.int32, device="cuda")
    res = device.integral_histogram(device.upload_image(px), lut, 5, out=out)
    assert res is out
    assert np.array_equal(out[0].cpu().numpy().view(np.uint32), O.compute_crossweave(px, lut, 5))
    with pytest.raises(ih.ShapeError):
        device.integral_histogram(device.upload_image(px), lut, 5,
                                  out=torch.zeros((1, 4, 50, 70), dtype=torch.int32, device="cuda"))


def test_window_count_kernel_variants(monkeypatch, rng):
    """K4 variants (two-output corners, 4-output ILP corners, staged row
    differences, 4 outputs from 16-byte corner loads) against the oracle:
    bit-identical, including odd output widths, w = W, h = H, 1-pixel
    windows and every right-corner word offset (w - 1) % 4."""
    for (H, W, B) in [(70, 1500, 5), (33, 2100, 32), (9, 7, 3), (300, 257, 16), (21, 4, 2), (5, 12, 7)]:
        px = rng.integers(0, 256, (H, W), dtype=np.uint8)
        full = O.compute_crossweave(px, O.np_uniform_table(B), B)
        t = torch.from_numpy(full.view(np.int32)).cuda().view(torch.uint32)
        for (h, w) in [(1, 1), (min(5, H), min(8, W)), (H, W), (H // 2 + 1, W // 3 + 1), (1, W), (H, 1),
                       (min(4, H), min(2, W)), (2, min(3, W)), (H - 1 or 1, max(W - 1, 1))]:
            want = O.window_counts(full, h, w)
            for mode in ("0", "1", "2", "3", "4"):
                monkeypatch.setenv("IH_K4_MODE", mode)
                assert np.array_equal(device.window_counts(t, h, w).cpu().numpy(), want), (H, W, h, w, mode)


def test_likelihood_table_path_bit_identical(monkeypatch, rng):
    """K5 through the per-(bin, count) metric table == K5 computing each term
    directly (IH_K5_DIRECT=1), bit for bit, both metrics, several windows."""
    for (H, W, B) in [(60, 90, 16), (40, 300, 256), (7, 9, 3)]:
        px = rng.integers(0, 256, (H, W), dtype=np.uint8)
        t = torch.from_numpy(O.compute_crossweave(px, O.np_uniform_table(B), B).view(np.int32)).cuda().view(torch.uint32)
        tmpl = rng.random(B)
        tmpl /= tmpl.sum()
        for (h, w) in [(1, 1), (min(8, H), min(8, W)), (H, W), (3, 7)]:
            for m in ("intersection", "bhattacharyya"):
                monkeypatch.delenv("IH_K5_DIRECT", raising=False)
                a = device.likelihood_map(t, tmpl, h, w, m).cpu().numpy()
                monkeypatch.setenv("IH_K5_DIRECT", "1")
                b = device.likelihood_map(t, tmpl, h, w, m).cpu().numpy()
                assert np.array_equal(a.view(np.int64), b.view(np.int64)), (H, W, B, h, w, m)
                monkeypatch.delenv("IH_K5_DIRECT")
                monkeypatch.setenv("IH_K5_PAIRS", "0")  # one placement per thread
                c = device.likelihood_map(t, tmpl, h, w, m).cpu().numpy()
                monkeypatch.delenv("IH_K5_PAIRS")
                assert np.array_equal(a.view(np.int64), c.view(np.int64)), (H, W, B, h, w, m)


@pytest.mark.parametrize("metric", ["intersection", "bhattacharyya"])
def test_fused_likelihood_map_vs_numpy_restatement(rng, metric):
    """K5 against likelihood.py:55-77 restated in numpy (tolerance 1e-12, the
    reference's own, tests/test_likelihood.py:46); also reports exactness."""
    for (H, W, B, h, w) in [(60, 90, 16, 8, 8), (97, 61, 7, 13, 5), (40, 40, 256, 40, 40),
                            (33, 300, 32, 1, 1)]:
        px = rng.integers(0, 256, (H, W), dtype=np.uint8)
        counts = O.compute_crossweave(px, O.np_uniform_table(B), B)
        tmpl = rng.random(B)
        tmpl /= tmpl.sum()
        ih_ = ih.IntegralHistogram(counts)
        got = ih.likelihood_map(ih_, tmpl, h, w, metric).values
        want = O.np_likelihood_map(counts, tmpl, h, w, metric)
        assert got.shape == want.shape
        assert np.abs(got - want).max() < 1e-12, (H, W, B, h, w)
    with pytest.raises(ih.ShapeError):
        ih.likelihood_map(ih_, np.ones(3) / 3, 2, 2)
    with pytest.raises(ih.ParameterError):
        ih.likelihood_map(ih_, tmpl, 2, 2, "nope")
    with pytest.raises(ih.BoundsError):
        ih.likelihood_map(ih_, tmpl, 34, 2)


@pytest.mark.parametrize("piece_bytes", [1 << 30, 3 * 60 * 90 * 4])
def test_frame_pipeline_host_to_host(rng, piece_bytes):
    """pipeline.FramePipeline: pinned H2D, kernels, pinned D2H through a two-slot
    ring, in frame chunks or (small pieces) bin sub-slabs of single frames."""
    from paper_1711_01919_b200 import pipeline

    frames = rng.integers(0, 256, (5, 60, 90), dtype=np.uint8)
    spec = ih.BinSpec.uniform(11)
    pipe = pipeline.FramePipeline(5, 60, 90, spec, chunk=2, bin_range=(2, 9),
                                  max_piece_bytes=piece_bytes)
    h_in = pipeline.pinned_empty((5, 60, 90), dtype=torch.uint8)
    h_in.copy_(torch.from_numpy(frames))
    h_out = pipeline.pinned_empty((5, 7, 60, 90))
    for _ in range(2):
        pipe.run(h_in, h_out)
        for f in range(5):
            want = O.compute_crossweave(frames[f], spec.table, 11)[2:9]
            assert np.array_equal(h_out[f].numpy(), want)


@pytest.mark.parametrize("nseg", [2, 5, 8, 9, 16])
def test_cluster_carries(monkeypatch, rng, nseg):
    """CARRY_CLUSTER: the segments of a strip form one thread-block cluster
    (up to 16 CTAs, non-portable above 8) and read their neighbours' column
    counts from distributed shared memory; frame batches, bin slabs, 256 bins,
    unaligned rows."""
    monkeypatch.setenv("IH_CARRY_CLUSTER", "1")
    monkeypatch.setenv("IH_NSEG", str(nseg))
    for (F, h, w, bins, rng_) in [(1, 512, 512, 32, None), (3, 300, 1000, 7, None),
                                  (1, 200, 2048, 256, (5, 200)), (2, 999, 130, 16, None)]:
        frames = rng.integers(0, 256, (F, h, w), dtype=np.uint8)
        lut = O.np_uniform_table(bins)
        p = device.plan(F, h, w, bins if rng_ is None else rng_[1] - rng_[0])
        assert p["launches"] == 1, p  # no prepass
        got = device.integral_histogram(torch.from_numpy(frames).cuda(), lut, bins, bin_range=rng_,
                                        kernel="single_pass").cpu().numpy()
        lo, hi = rng_ or (0, bins)
        for f in range(F):
            assert np.array_equal(got[f], O.compute_crossweave(frames[f], lut, bins)[lo:hi]), (F, h, w, f)
    base = rng.integers(0, 256, (77, 333 + 3), dtype=np.uint8)
    view = torch.from_numpy(base).cuda()[:, 3:]
    got = device.integral_histogram(view, O.np_uniform_table(9), 9, kernel="single_pass").cpu().numpy()
    assert np.array_equal(got, O.compute_crossweave(np.ascontiguousarray(base[:, 3:]), O.np_uniform_table(9), 9))


@pytest.mark.parametrize("shard", ["bins", "frames"])
@pytest.mark.parametrize("out", ["host", "device", "shards"])
def test_devices_kwarg_single_process(rng, shard, out):
    """multi.integral_histogram_devices (the devices= form): shards over a
    device list (here the one GPU three times, separate streams), every output
    mode, equal to the oracle; compute(..., devices=) and
    compute_frames(..., devices=) use it."""
    from paper_1711_01919_b200 import multi

    frames = rng.integers(0, 256, (4, 90, 300), dtype=np.uint8)
    lut = O.np_uniform_table(11)
    want = np.stack([O.compute_crossweave(f, lut, 11) for f in frames])
    res = multi.integral_histogram_devices(frames, lut, 11, [0, 0, 0], shard=shard, out=out)
    if out == "host":
        got = res
    elif out == "device":
        got = res.cpu().numpy()
    else:
        got = np.zeros_like(want)
        for (f0, f1, b0, b1), t in res:
            if t is not None:
                got[f0:f1, b0:b1] = t.cpu().numpy()
    assert np.array_equal(got, want)
    img = ih.GrayImage(frames[0])
    assert np.array_equal(ih.compute(img, ih.BinSpec.uniform(11), ih.SEQUENTIAL, devices=[0, 0]).counts,
                          want[0])
    t = ih.compute_frames(frames, ih.BinSpec.uniform(11), devices=[0, 0], shard=shard)
    assert np.array_equal(t.cpu().numpy(), want)


def test_graphed_integral_histogram(rng):
    """GraphedIntegralHistogram: capture once, replay with new frames (host or
    device, unaligned width), bit-identical to the oracle each time."""
    for (F, H, W, bins, br) in [(2, 90, 301, 13, None), (1, 1080, 1920, 32, (8, 24))]:
        g = device.GraphedIntegralHistogram(F, H, W, O.np_uniform_table(bins), bins, bin_range=br)
        lo, hi = br or (0, bins)
        for rep in range(3):
            frames = rng.integers(0, 256, (F, H, W), dtype=np.uint8)
            src = frames if rep % 2 == 0 else torch.from_numpy(frames).cuda()
            out = g(src).cpu().numpy()
            for f in range(F):
                want = O.compute_crossweave(frames[f], O.np_uniform_table(bins), bins)[lo:hi]
                assert np.array_equal(out[f], want), (F, H, W, rep, f)


@pytest.mark.parametrize("shard", ["bins", "frames"])
def test_c7_device_count_determinism(rng, shard):
    """acceptance C7 extended to device counts 1/2/4/8 -- the
    assembled tensor is byte-identical for every count (the one GPU stands in
    for each device, on separate streams)."""
    from paper_1711_01919_b200 import multi

    frames = rng.integers(0, 256, (8, 70, 517), dtype=np.uint8)
    lut = O.np_uniform_table(37)
    ref = None
    for g in (1, 2, 4, 8):
        got = multi.integral_histogram_devices(frames, lut, 37, [0] * g, shard=shard, out="host")
        if ref is None:
            ref = got
            for f in range(8):
                assert np.array_equal(got[f], O.compute_crossweave(frames[f], lut, 37))
        assert np.array_equal(got, ref), g


@pytest.mark.parametrize("rowpack", [True, False])
def test_row_packed_one_and_two_bin_slabs(monkeypatch, rng, rowpack):
    """1- and 2-bin slabs pack 4 / 2 rows into the byte lanes of a word (KB =
    1 / 2); against the oracle with segments, tail splits, frame batches, odd
    widths, LDG inputs and bin slabs of larger specs, and with IH_NO_ROWPACK."""
    if not rowpack:
        monkeypatch.setenv("IH_NO_ROWPACK", "1")
    cases = [(1, 300, 1000, 1, None), (3, 97, 130, 2, None), (2, 257, 2048, 37, (5, 6)),
             (1, 1080, 1920, 32, (30, 32)), (4, 33, 7, 2, None), (1, 1, 1, 1, None)]
    for nseg, tail in [("0", None), ("5", "30"), ("3", None)]:
        if nseg != "0":
            monkeypatch.setenv("IH_NSEG", nseg)
        else:
            monkeypatch.delenv("IH_NSEG", raising=False)
        if tail:
            monkeypatch.setenv("IH_TAIL_PCT", tail)
        else:
            monkeypatch.delenv("IH_TAIL_PCT", raising=False)
        for (F, h, w, bins, br) in cases:
            frames = rng.integers(0, 256, (F, h, w + 3), dtype=np.uint8)
            view = torch.from_numpy(frames).cuda()[:, :, 3:]
            lut = O.np_uniform_table(bins)
            lo, hi = br or (0, bins)
            got = device.integral_histogram(view, lut, bins, bin_range=br,
                                            kernel="single_pass").cpu().numpy()
            for f in range(F):
                want = O.compute_crossweave(np.ascontiguousarray(frames[f, :, 3:]), lut, bins)[lo:hi]
                assert np.array_equal(got[f], want), (F, h, w, bins, br, nseg, tail, f)


def test_tall_and_wide_column_tiles(rng):
    """H > 65535 with column tiles: u16 prefix tables are impossible, the scan
    sums count slots, and every tile adds row carries and chunk totals."""
    px = rng.integers(0, 256, (70001, 2100), dtype=np.uint8)
    lut = O.np_uniform_table(2)
    assert device.plan(1, 70001, 2100, 2)["column_tiles"] == 2
    got = dev_compute(px, lut, 2, kernel="single_pass")
    want = O.compute_crossweave(px, lut, 2)
    assert np.array_equal(got.cpu().numpy(), want)


def test_to_host_private_pinned_released(monkeypatch):
    """Results >= PRIVATE_PINNED_MIN_BYTES get their own page-locked block
    (ih_host_alloc) that is freed when the array dies, not a cached one."""
    import gc

    freed = []
    L = device._native.lib()
    real_free = L.ih_host_free
    monkeypatch.setattr(device, "PRIVATE_PINNED_MIN_BYTES", 1 << 20)

    class Spy:
        def __getattr__(self, name):
            return getattr(L, name)

        def ih_host_free(self, p):
            freed.append(p)
            real_free(p)

    monkeypatch.setattr(device._native, "lib", lambda: Spy())
    t = torch.arange(1 << 19, dtype=torch.int32, device="cuda").view(torch.uint32).reshape(512, 1024)
    a = device.to_host(t)
    assert a.dtype == np.uint32 and np.array_equal(a, np.arange(1 << 19, dtype=np.uint32).reshape(512, 1024))
    assert not freed
    v = a[3:5]
    del a
    gc.collect()
    assert not freed and int(v[0, 0]) == 3 * 1024
    del v
    gc.collect()
    assert len(freed) == 1


# ------------------------------------------------ K2s: one-launch small images
def test_k2s_default_plan_and_cfg1(monkeypatch, golden_configs):
    """One image with <= 4 bin groups plans the one-launch kernel by default;
    BASELINE cfg1 (512x512x32, 8 groups: the count-table path by default)
    through K2s reproduces the reference's golden crc."""
    p = device.plan(1, 512, 512, 16)
    assert (p["carry"], p["launches"]) == ("in_kernel", 1), p
    assert device.plan(1, 512, 512, 32)["carry"] == "table"
    px = O.synth_image(512, 512, 0)
    lut16 = O.np_uniform_table(16)
    assert np.array_equal(dev_compute(px, lut16, 16).cpu().numpy(), O.compute_crossweave(px, lut16, 16))
    monkeypatch.setenv("IH_SMALL", "1")
    assert device.plan(1, 512, 512, 32)["carry"] == "in_kernel"
    got = dev_compute(px, O.np_uniform_table(32), 32).cpu().numpy()
    assert crc_of(got) == golden_configs["512x512x32"]["crc"]


def test_k2s_c1_instances(monkeypatch, golden_c1):
    """All 200 acceptance-C1 instances through K2s (forced where it applies)."""
    monkeypatch.setenv("IH_SMALL", "1")
    for (w, h, b, tile, px), gold in zip(c1_images(200), golden_c1):
        got = dev_compute(px, O.np_uniform_table(b), b).cpu().numpy()
        assert crc_of(got) == gold["crc"], (w, h, b)


@pytest.mark.parametrize("nseg", [0, 1, 2, 7, 40, 100000])
def test_k2s_shapes_segments_slabs(monkeypatch, rng, nseg):
    """K2s over widths 1..2048 (4 / 2 / 1 warp-groups, odd widths), heights up
    to 1500, bins 1..256 with slabs and explicit LUTs, frame batches, and
    forced segment counts from 1 to one row per segment."""
    monkeypatch.setenv("IH_SMALL", "1")
    if nseg:
        monkeypatch.setenv("IH_NSEG", str(nseg))
    for (F, h, w, bins) in [(1, 1, 1, 1), (1, 7, 3, 5), (2, 33, 127, 32), (1, 100, 129, 256),
                            (3, 257, 513, 7), (1, 600, 1000, 64), (1, 1500, 2047, 3),
                            (2, 64, 2048, 33), (1, 512, 512, 32)]:
        lut = rng.integers(0, bins, 256).astype(np.uint8) if bins > 4 else O.np_uniform_table(bins)
        lo = int(rng.integers(0, bins))
        hi = int(rng.integers(lo + 1, bins + 1))
        frames = rng.integers(0, 256, (F, h, w), dtype=np.uint8)
        got = device.integral_histogram(device.upload_frames(frames), lut, bins,
                                        bin_range=(lo, hi)).cpu().numpy()
        for f in range(F):
            want = O.compute_crossweave(frames[f], lut, bins)[lo:hi]
            assert np.array_equal(got[f], want), (nseg, F, h, w, bins, lo, hi, f)


@pytest.mark.parametrize("skew,pct", [(115, 50), (130, 50), (150, 30), (300, 70)])
def test_skewed_segments(monkeypatch, rng, skew, pct):
    """Skewed segment sizes (the first pct % of the segments larger by skew/100,
    IH_SKEW_X100 / the autotuner's hint flag) over column tiles, frame batches
    and slabs: bit-exact, and the plan really is skewed."""
    monkeypatch.setenv("IH_SKEW_X100", str(skew))
    monkeypatch.setenv("IH_SKEW_PCT", str(pct))
    for (F, h, w, bins, nseg) in [(1, 2160, 3840, 16, 37), (3, 300, 700, 12, 9), (2, 129, 2100, 5, 4)]:
        monkeypatch.setenv("IH_NSEG", str(nseg))
        p = device.plan(F, h, w, bins)
        assert p["big_segments"] < p["segments"] and p["segment_rows"] > p["tail_segment_rows"], p
        frames = rng.integers(0, 256, (F, h, w), dtype=np.uint8)
        lut = O.np_uniform_table(bins)
        got = device.integral_histogram(device.upload_frames(frames), lut, bins).cpu().numpy()
        for f in range(F):
            assert np.array_equal(got[f], O.compute_crossweave(frames[f], lut, bins)), (F, h, w, bins, f)

