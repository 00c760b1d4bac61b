"""Input-robustness fixes: device-side region validation, misaligned window
outputs, explicit streams, host-resident queries, partial pwrites."""

import os

import numpy as np
import pytest

from oracle import oracle as O


def test_pwrite_all_loops_over_partial_writes(tmp_path, monkeypatch):
    """TensorFileSink must finish a plane even when one pwrite moves fewer
    bytes than asked (Linux caps a write at 0x7ffff000 bytes)."""
    from paper_1711_01919_b200 import formats

    real = os.pwrite
    calls = []

    def short_pwrite(fd, buf, off):
        calls.append(len(buf))
        return real(fd, bytes(buf[:7]), off)  # at most 7 bytes per call

    monkeypatch.setattr(formats.os, "pwrite", short_pwrite)
    data = np.arange(3 * 5 * 4, dtype=np.uint32).reshape(3, 5, 4)
    path = tmp_path / "t.ihst"
    with formats.TensorFileSink(path, 4, 5, 3) as sink:
        sink.write(0, 3, 0, 5, data)
    monkeypatch.setattr(formats.os, "pwrite", real)
    raw = path.read_bytes()
    got = np.frombuffer(raw, dtype="<u4", offset=formats.IHST_HEADER_BYTES).reshape(3, 5, 4)
    assert np.array_equal(got, data)
    assert len(calls) > 3 * 2


gpu = pytest.mark.gpu


@gpu
def test_device_regions_are_validated():
    import torch

    from paper_1711_01919_b200 import BoundsError, ParameterError, device

    px = np.random.default_rng(1).integers(0, 256, (40, 50), dtype=np.uint8)
    t = device.integral_histogram(device.upload_image(px), O.np_uniform_table(8), 8)
    ok = torch.tensor([[0, 0, 39, 49], [3, 4, 10, 20]], dtype=torch.int64, device="cuda")
    got = device.region_histograms(t, ok).cpu().numpy().view(np.uint64)
    counts = O.compute_sequential(px, O.np_uniform_table(8), 8)
    assert np.array_equal(got, O.region_histograms(counts, ok.cpu().numpy()))
    for bad, exc in (([5, 0, 4, 3], BoundsError),        # r0 > r1: degenerate
                     ([-1, 0, 4, 3], BoundsError),       # negative
                     ([0, 0, 40, 3], BoundsError),       # outside (H = 40)
                     ([0, 0, 3, 50], BoundsError),       # outside (W = 50)
                     ([0, 0, 1 << 33, 3], BoundsError)):  # outside, and not int32
        with pytest.raises(exc):
            device.region_histograms(t, torch.tensor([bad], dtype=torch.int64, device="cuda"))
    with pytest.raises(ParameterError):
        device.region_histograms(t, torch.zeros((1, 4), dtype=torch.float32, device="cuda"))


@gpu
def test_kernel_never_reads_outside_for_invalid_regions():
    """validate=False (or a C caller): invalid regions give zero rows, no fault."""
    import torch

    from paper_1711_01919_b200 import device

    px = np.random.default_rng(2).integers(0, 256, (16, 16), dtype=np.uint8)
    t = device.integral_histogram(device.upload_image(px), O.np_uniform_table(4), 4)
    regs = torch.tensor([[0, 0, 1 << 30, 1 << 30], [3, 3, 1, 1], [0, 0, 15, 15]],
                        dtype=torch.int32, device="cuda")
    got = device.region_histograms(t, regs, validate=False).cpu().numpy().view(np.uint64)
    torch.cuda.synchronize()
    assert (got[0] == 0).all() and (got[1] == 0).all() and int(got[2].sum()) == 256


@gpu
@pytest.mark.parametrize("mode", ["0", "1", "2", "3", "4"])
def test_window_counts_misaligned_out(monkeypatch, mode):
    """An int64 out view at an odd element offset (8- but not 16-byte aligned),
    for every K4 kernel (IH_K4_MODE; the 16-byte-pair modes fall back)."""
    import torch

    from paper_1711_01919_b200 import device

    monkeypatch.setenv("IH_K4_MODE", mode)
    px = np.random.default_rng(3).integers(0, 256, (30, 41), dtype=np.uint8)
    t = device.integral_histogram(device.upload_image(px), O.np_uniform_table(5), 5)
    for h, w in ((4, 6), (1, 40), (7, 7)):  # odd and even output row lengths
        shape = (5, 30 - h + 1, 41 - w + 1)
        n = int(np.prod(shape))
        buf = torch.zeros(n + 1, dtype=torch.int64, device="cuda")
        out = buf[1:].view(shape)
        assert out.data_ptr() % 16 == 8
        device.window_counts(t, h, w, out=out)
        want = O.window_counts(O.compute_sequential(px, O.np_uniform_table(5), 5), h, w)
        assert np.array_equal(out.cpu().numpy(), want), (h, w)


@gpu
def test_integral_histogram_misaligned_out_is_rejected():
    """A uint32 out view 4 bytes past a 16-byte boundary with W % 4 == 0 (the
    kernels' 16-byte stores would fault) is refused before any launch; the
    same view is fine for an odd width (alignment-adaptive stores), and the
    context stays usable."""
    import torch

    from paper_1711_01919_b200 import device
    from paper_1711_01919_b200.errors import ParameterError, ShapeError

    table = O.np_uniform_table(8)
    for W, ok in ((64, False), (61, True)):
        px = np.random.default_rng(W).integers(0, 256, (33, W), dtype=np.uint8)
        img = device.upload_image(px)
        n = 8 * 33 * W
        buf = torch.zeros(n + 1, dtype=torch.uint32, device="cuda")
        out = buf[1:].view(8, 33, W)
        assert out.data_ptr() % 16 == 4
        if ok:
            device.integral_histogram(img, table, 8, out=out)
            assert np.array_equal(out.cpu().numpy(), O.compute_sequential(px, table, 8))
        else:
            with pytest.raises(ParameterError, match="16-byte aligned"):
                device.integral_histogram(img, table, 8, out=out)
            with pytest.raises(ParameterError, match="16-byte aligned"):
                device.scan(img, table, 8, out)
        with pytest.raises(ShapeError):
            device.scan(img, table, 8, buf[: n // 2])  # too small: refused, not written past
    # the context is intact
    px = np.random.default_rng(0).integers(0, 256, (16, 16), dtype=np.uint8)
    t = device.integral_histogram(device.upload_image(px), table, 8)
    torch.cuda.synchronize()
    assert np.array_equal(t.cpu().numpy(), O.compute_sequential(px, table, 8))


@gpu
def test_concurrent_calls_on_threads_and_streams():
    """Two host threads, each on its own CUDA stream with its own bin table,
    calling integral_histogram with the default workspace: every result is the
    oracle's (per-(device, stream) scratch, atomic table-pointer cache)."""
    import threading

    import torch

    from paper_1711_01919_b200 import device

    px = np.random.default_rng(11).integers(0, 256, (96, 200), dtype=np.uint8)
    img = device.upload_image(px)
    want = {b: O.compute_sequential(px, O.np_uniform_table(b), b) for b in (7, 32)}
    errors = []

    def worker(bins):
        try:
            s = torch.cuda.Stream()
            table = O.np_uniform_table(bins)
            with torch.cuda.stream(s):
                for _ in range(40):
                    t = device.integral_histogram(img, table, bins)
                    s.synchronize()
                    if not np.array_equal(t.cpu().numpy(), want[bins]):
                        errors.append(bins)
                        return
        except Exception as e:  # surfaced below
            errors.append(repr(e))

    torch.cuda.synchronize()
    th = [threading.Thread(target=worker, args=(b,)) for b in (7, 32)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errors, errors


@gpu
def test_default_workspace_grows_under_queued_work():
    """Calls on an explicit side stream whose default workspace must grow
    while earlier calls are still queued: the old buffer is not recycled
    under them (each result equals the oracle)."""
    import torch

    from paper_1711_01919_b200 import device

    s = torch.cuda.Stream()
    table = O.np_uniform_table(16)
    rng = np.random.default_rng(21)
    shapes = [(40, 300), (300, 1000), (900, 1900), (1080, 1920)]  # growing workspaces
    pxs = [rng.integers(0, 256, sh, dtype=np.uint8) for sh in shapes]
    imgs = [device.upload_image(p) for p in pxs]
    torch.cuda.synchronize()
    outs = []
    for _ in range(3):
        for img in imgs:
            outs.append(device.integral_histogram(img, table, 16, stream=s))
    s.synchronize()
    for k, t in enumerate(outs):
        px = pxs[k % len(pxs)]
        assert np.array_equal(t.cpu().numpy(), O.compute_sequential(px, table, 16)), k


@gpu
def test_explicit_stream_queries():
    import torch

    from paper_1711_01919_b200 import device

    px = np.random.default_rng(4).integers(0, 256, (64, 64), dtype=np.uint8)
    lut = O.np_uniform_table(16)
    t = device.integral_histogram(device.upload_image(px), lut, 16)
    counts = O.compute_sequential(px, lut, 16)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    regs = np.array([[0, 0, 63, 63], [5, 6, 30, 40]] * 100)
    q = device.region_histograms(t, regs, stream=s)
    w = device.window_counts(t, 8, 8, stream=s)
    s.synchronize()
    assert np.array_equal(q.cpu().numpy().view(np.uint64), O.region_histograms(counts, regs))
    assert np.array_equal(w.cpu().numpy(), O.window_counts(counts, 8, 8))


@gpu
def test_host_resident_region_query_uploads_corners_only():
    """region_histogram on a host tensor (e.g. read from IHST) answers from the
    4 x B corner values; the full tensor is never uploaded."""
    import paper_1711_01919_b200 as ih

    px = np.random.default_rng(5).integers(0, 256, (37, 53), dtype=np.uint8)
    lut = O.np_uniform_table(7)
    counts = O.compute_sequential(px, lut, 7)
    host_ih = ih.IntegralHistogram(counts)
    for reg in ((0, 0, 36, 52), (0, 5, 10, 5), (4, 0, 4, 52), (3, 7, 20, 31)):
        got = ih.region_histogram(host_ih, ih.Region(*reg)).counts
        assert np.array_equal(got, O.region_histograms(counts, [reg])[0])
    assert host_ih._dev is None
