"""BASELINE cfg4 at full size on one B200: 8192x8192, 256 bins (68.7 GB tensor).

Checked against the reference's own per-plane crc32 (SURVEY.md Appendix A,
computed with the reference's compute_streamed) and the whole-tensor crc, plus
the size-independent invariant sum_b H_b(r, c) = (r+1)(c+1) on the device.
Both the single-GPU tensor and the 8-way bin-shard slabs (32 bins each, the
per-GPU share of the 8-GPU run) are verified.  Then batched region queries
(Q = 65,536, drawn as acceptance C4 does) against the oracle's four-corner
formula on the host copy of a few planes.
"""

import zlib

import numpy as np
import pytest

from oracle import oracle as O

pytestmark = [pytest.mark.gpu, pytest.mark.slow]
torch = pytest.importorskip("torch")

from paper_1711_01919_b200 import device, sharding  # noqa: E402


def _free_gb():
    free, _ = torch.cuda.mem_get_info()
    return free / 1e9


@pytest.fixture(scope="module")
def img8k():
    return O.synth_image(8192, 8192, 0)


def _plane_crcs(t, pinned):
    crcs = []
    for b in range(t.shape[0]):
        pinned.copy_(t[b].view(torch.int32))
        crcs.append(zlib.crc32(memoryview(pinned.numpy())))
    return crcs


def test_8k_256_single_gpu(img8k, golden_configs):
    if _free_gb() < 75:
        pytest.skip("needs ~70 GB of free device memory")
    gold = golden_configs["8192x8192x256"]
    d = device.upload_image(img8k)
    t = device.integral_histogram(d, O.np_uniform_table(256), 256)
    torch.cuda.synchronize()
    # invariant on device: sum over bins == (r+1)(c+1)
    s = torch.zeros((8192, 8192), dtype=torch.int64, device=t.device)
    for b0 in range(0, 256, 32):
        s += t[b0:b0 + 32].view(torch.int32).sum(dim=0, dtype=torch.int64)
    rr = torch.arange(1, 8193, device=t.device, dtype=torch.int64)[:, None]
    cc = torch.arange(1, 8193, device=t.device, dtype=torch.int64)[None, :]
    assert bool((s == rr * cc).all())
    del s
    pinned = torch.empty((8192, 8192), dtype=torch.int32, pin_memory=True)
    crcs = _plane_crcs(t, pinned)
    assert [f"{c:08x}" for c in crcs] == gold["plane_crc"]
    whole = 0
    for b in range(256):
        pinned.copy_(t[b].view(torch.int32))
        whole = zlib.crc32(memoryview(pinned.numpy()), whole)
    assert f"{whole:08x}" == gold["crc"]

    # batched region queries, Q = 65,536 (acceptance-C4 style draws)
    rng = np.random.default_rng(20260823 + 4)
    Q = 65536
    r = np.sort(rng.integers(0, 8192, (Q, 2)), axis=1)
    c = np.sort(rng.integers(0, 8192, (Q, 2)), axis=1)
    regs = np.stack([r[:, 0], c[:, 0], r[:, 1], c[:, 1]], axis=1).astype(np.int32)
    got = device.region_histograms(t, regs).cpu().numpy()
    assert got.shape == (Q, 256)
    assert np.array_equal(got.sum(axis=1, dtype=np.int64),
                          (regs[:, 2] - regs[:, 0] + 1).astype(np.int64)
                          * (regs[:, 3] - regs[:, 1] + 1))
    for b in (0, 100, 255):
        pinned.copy_(t[b].view(torch.int32))
        plane = pinned.numpy().view(np.uint32)[None]
        expect = O.region_histograms(plane, regs[:2048])[:, 0]
        assert np.array_equal(got[:2048, b], expect), b
    # every bin of the first 8,192 queries: the four corners of each query are
    # gathered from the tensor by torch indexing (independent of K3) and
    # combined with the oracle's inclusion-exclusion (core.py:184-194)
    nq = 8192
    rg = torch.from_numpy(regs[:nq].astype(np.int64)).to(t.device)
    tv = t.view(torch.int32)
    corner = []
    for rr, cc in ((rg[:, 2], rg[:, 3]), (rg[:, 0] - 1, rg[:, 3]), (rg[:, 2], rg[:, 1] - 1),
                   (rg[:, 0] - 1, rg[:, 1] - 1)):
        ok = (rr >= 0) & (cc >= 0)
        v = tv[:, rr.clamp(min=0), cc.clamp(min=0)].to(torch.int64) & 0xffffffff
        corner.append((v * ok.to(torch.int64)).cpu().numpy())  # (256, nq)
    expect_all = (corner[0] - corner[1] - corner[2] + corner[3]).T
    assert np.array_equal(got[:nq].astype(np.int64), expect_all)


def test_8k_256_eight_bin_shards(img8k, golden_configs):
    """The 8-GPU decomposition, slab by slab on one device (32 bins each)."""
    gold = golden_configs["8192x8192x256"]["plane_crc"]
    d = device.upload_image(img8k)
    lut = O.np_uniform_table(256)
    pinned = torch.empty((8192, 8192), dtype=torch.int32, pin_memory=True)
    for g, (lo, hi) in enumerate(sharding.bin_slabs(256, 8)):
        t = device.integral_histogram(d, lut, 256, bin_range=(lo, hi))
        crcs = _plane_crcs(t, pinned)
        assert [f"{x:08x}" for x in crcs] == gold[lo:hi], g
        del t
