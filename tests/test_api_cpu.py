"""Host-side logic of the drop-in API (no device needed): types, validation
order, strategy set, planning, sharding partitions, and the no-fallback rule."""

import numpy as np
import pytest

import paper_1711_01919_b200 as ih
from conftest import has_cuda
from paper_1711_01919_b200 import sharding


def test_public_names_cover_reference_all():
    for name in ih.REFERENCE_ALL:
        assert hasattr(ih, name), name


class TestBinSpec:
    def test_uniform_examples(self):
        assert ih.map_intensity(0, ih.BinSpec.uniform(16)) == 0
        assert ih.map_intensity(255, ih.BinSpec.uniform(256)) == 255
        assert ih.map_intensity(128, ih.BinSpec.uniform(2)) == 1

    def test_uniform_equals_floor_formula(self):
        for b in (1, 2, 3, 16, 64, 255, 256):
            assert ih.BinSpec.uniform(b).table.tolist() == [(v * b) // 256 for v in range(256)]

    def test_explicit(self):
        tab = np.zeros(256, np.uint8)
        tab[128:] = 1
        spec = ih.BinSpec.explicit(tab)
        assert spec.bins == 2 and ih.map_intensity(127, spec) == 0

    def test_bad_specs(self):
        with pytest.raises(ih.ShapeError):
            ih.BinSpec.uniform(0)
        with pytest.raises(ih.ShapeError):
            ih.BinSpec.uniform(257)
        with pytest.raises(ih.ShapeError):
            ih.BinSpec(2, np.full(256, 2))
        with pytest.raises(ih.ShapeError):
            ih.BinSpec(2, np.zeros(255))
        with pytest.raises(ValueError):
            ih.map_intensity(256, ih.BinSpec.uniform(4))


class TestTypes:
    def test_image(self):
        with pytest.raises(ih.ShapeError):
            ih.GrayImage(np.zeros((2, 2), np.float32))
        with pytest.raises(ih.ShapeError):
            ih.GrayImage(np.zeros((0, 3), np.uint8))
        with pytest.raises(ih.ShapeError):
            ih.GrayImage.from_bytes(2, 2, b"\0" * 3)
        img = ih.GrayImage.from_bytes(3, 2, bytes(range(6)))
        assert (img.width, img.height) == (3, 2)
        assert not img.pixels.flags.writeable

    def test_capacity(self):
        class Fake:
            width, height = 1 << 16, (1 << 16) + 1

        with pytest.raises(ih.CapacityError):
            ih.GrayImage.check_capacity(Fake())

    def test_region(self):
        with pytest.raises(ih.BoundsError):
            ih.Region(2, 0, 1, 0)
        with pytest.raises(ih.BoundsError):
            ih.Region(-1, 0, 0, 0)
        assert ih.Region(1, 2, 3, 5).area == 12
        with pytest.raises(ih.BoundsError):
            ih.Region(0, 0, 4, 3).check_within(4, 4)

    def test_integral_histogram_host(self):
        t = ih.IntegralHistogram(np.ones((2, 3, 4), np.uint32))
        assert (t.bins, t.height, t.width) == (2, 3, 4)
        with pytest.raises(ih.ShapeError):
            ih.IntegralHistogram(np.ones((2, 3), np.uint32))
        with pytest.raises(ih.ShapeError):
            ih.IntegralHistogram(np.ones((2, 3, 4), np.int64))

    def test_metrics(self):
        assert ih.normalize(ih.Histogram(np.array([1, 3]))).tolist() == [0.25, 0.75]
        with pytest.raises(ValueError):
            ih.normalize(ih.Histogram(np.zeros(4)))
        p = np.array([0.5, 0.5])
        assert ih.intersection(p, p) == 1.0
        assert ih.bhattacharyya(p, p)[0] == pytest.approx(1.0)
        with pytest.raises(ih.ShapeError):
            ih.intersection(p, np.ones(3) / 3)


class TestStrategy:
    def test_validation(self):
        with pytest.raises(ih.ParameterError):
            ih.Strategy("wavefront", 0)
        with pytest.raises(ih.ParameterError):
            ih.Strategy("nope")
        with pytest.raises(ih.ParameterError):
            ih.Strategy("sequential", 3)
        assert ih.wavefront().tile == 64

    def test_error_order_before_device(self):
        img = ih.GrayImage(np.zeros((4, 4), np.uint8))
        spec = ih.BinSpec.uniform(2)
        with pytest.raises(ih.ParameterError):
            ih.compute_wavefront(img, spec, 0)
        with pytest.raises(ih.ParameterError):
            ih.resolve_workers(-1)

    @pytest.mark.skipif(has_cuda(), reason="checks the no-GPU behaviour")
    def test_no_cpu_fallback(self):
        img = ih.GrayImage(np.zeros((4, 4), np.uint8))
        for fn in (ih.compute_sequential, ih.compute_crossweave, ih.compute_sts):
            with pytest.raises(ih.DeviceError):
                fn(img, ih.BinSpec.uniform(2))
        with pytest.raises(ih.DeviceError):
            ih.compute_wavefront(img, ih.BinSpec.uniform(2), 2, 0, [])
        with pytest.raises(ih.DeviceError):
            ih.region_histogram(ih.IntegralHistogram(np.ones((1, 2, 2), np.uint32)),
                                ih.Region(0, 0, 1, 1))


class TestPlanning:
    def test_plan_tiles(self):
        plan = ih.plan_tiles(1024, 1024, 64, 64 * 2**20)
        assert len(plan.bin_chunks) >= 4 and plan.strip_height == 1024
        small = ih.plan_tiles(256, 256, 64, 80_000)
        assert len(small.bin_chunks) == 64 and small.strips >= 4
        assert small.peak_bytes <= 80_000
        with pytest.raises(ih.CapacityError):
            ih.plan_tiles(256, 256, 4, 10)
        with pytest.raises(ih.ParameterError):
            ih.TilePlan(4, 4, 4, 1 << 20, ((0, 2), (3, 4)), 4)
        with pytest.raises(ih.ParameterError):
            ih.TilePlan(4, 4, 4, 1 << 20, ((0, 2),), 4)

    def test_bin_slabs(self):
        assert sharding.bin_slabs(256, 8) == [(32 * g, 32 * g + 32) for g in range(8)]
        assert sharding.bin_slabs(128, 2) == [(0, 64), (64, 128)]
        s = sharding.bin_slabs(3, 8)
        assert s[:3] == [(0, 1), (1, 2), (2, 3)] and all(lo == hi for lo, hi in s[3:])
        for bins in range(1, 40):
            for world in range(1, 10):
                s = sharding.bin_slabs(bins, world)
                assert s[0][0] == 0 and s[-1][1] == bins
                assert all(a[1] == b[0] for a, b in zip(s, s[1:]))

    def test_frame_shards(self):
        assert sharding.frame_shards(64, 8) == [(8 * g, 8 * g + 8) for g in range(8)]
        s = sharding.frame_shards(10, 4)
        assert [hi - lo for lo, hi in s] == [3, 3, 2, 2] and s[-1][1] == 10
