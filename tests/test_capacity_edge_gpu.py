"""The reference's capacity limit, exactly at the edge: W * H = 2^32 - 1 pixels
(core.py:53-57 accepts it; one more pixel raises CapacityError).

Every count is then <= 2^32 - 1, so the u32 tensor is exact, but any 32-bit
index product (r * W + c, plane offsets, segment/tile strides) inside a kernel
would wrap.  Two shapes: 65535 wide x 65537 tall (column tiles, > 65535 rows:
the raw-count carry path) and 65537 wide (W % 4 == 1: unaligned output rows)
x 65535 tall.  One 1-bin slab of a 2-bin table (17.2 GB of output) each,
checked against the oracle's streamed per-plane crc32 (oracle/ih_oracle.c,
iho_plane_crc32) plus an on-device total.
"""

import zlib

import numpy as np
import pytest

from oracle import oracle as O

pytestmark = [pytest.mark.gpu, pytest.mark.slow]
torch = pytest.importorskip("torch")

from paper_1711_01919_b200 import device  # noqa: E402
from paper_1711_01919_b200.errors import CapacityError  # noqa: E402


def _device_plane_crc32(plane, rows_per_chunk=2048):
    """crc32 of a (H, W) uint32 device plane, streamed through one pinned buffer."""
    H, W = plane.shape
    buf = torch.empty((rows_per_chunk, W), dtype=torch.int32, pin_memory=True)
    crc = 0
    for r0 in range(0, H, rows_per_chunk):
        n = min(rows_per_chunk, H - r0)
        buf[:n].copy_(plane[r0:r0 + n].view(torch.int32))
        crc = zlib.crc32(memoryview(buf[:n].numpy()), crc)
    return crc


def _free_gb():
    free, _ = torch.cuda.mem_get_info()
    return free / 1e9


@pytest.mark.parametrize("W,H", [(65535, 65537), (65537, 65535)])
def test_capacity_edge(W, H):
    assert W * H == 2**32 - 1
    if _free_gb() < 30:
        pytest.skip("needs ~25 GB of free device memory")
    rng = np.random.default_rng(np.random.SeedSequence([7, W, H]))
    img = rng.integers(0, 256, size=(H, W), dtype=np.uint8)
    lut = O.np_uniform_table(2)  # bin 0: values < 128
    d = device.upload_image(img)
    t = device.integral_histogram(d, lut, 2, bin_range=(0, 1))
    assert t.shape == (1, H, W)
    total = int((d < 128).sum())
    assert int(t[0, H - 1, W - 1].view(torch.int32).item()) & 0xffffffff == total
    got = _device_plane_crc32(t[0])
    del t
    torch.cuda.empty_cache()
    assert got == O.plane_crc32(img, lut, 0)


def test_capacity_edge_plus_one_raises():
    """One pixel over the edge is the reference's CapacityError, before any device work."""
    d = torch.empty((65536, 65536), dtype=torch.uint8, device="cuda")
    with pytest.raises(CapacityError):
        device.integral_histogram(d, O.np_uniform_table(2), 2)
