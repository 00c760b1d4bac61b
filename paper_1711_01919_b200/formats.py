"""File formats: binary PGM images and the "IHST" integral-histogram container.

Byte-for-byte compatible with the reference's formats (pkg/src/inthist/imgio.py):

    IHST: 16-byte little-endian header  magic b"IHST" | version u16 = 1 |
          bins u16 | width u32 | height u32, then `bins` planes of
          height x width u32, row-major, bin 0 first (imgio.py:1-14, :26-28).
    PGM:  "P5" binary graymap, maxval 255 only (imgio.py:34-77).

The B200-specific piece is ``save_ihst``: a device-resident tensor is streamed
to the file in plane groups through two pinned host buffers, the D2H copy of
group k+1 overlapping the positional write of group k, so a 68.7 GB tensor
never needs a second full host copy.
"""

from __future__ import annotations

import os
import struct
import threading

import numpy as np

from .domain import GrayImage, IntegralHistogram
from .errors import FormatError

IHST_MAGIC = b"IHST"
IHST_VERSION = 1
_HDR = struct.Struct("<4sHHII")
IHST_HEADER_BYTES = _HDR.size  # 16
_PGM_SPACE = frozenset(b" \t\r\n\x0b\x0c")


# ----------------------------------------------------------------------- PGM
def _pgm_header(data: bytes) -> tuple[int, int, int, int]:
    """(width, height, maxval, offset of the first pixel byte)."""
    if not data.startswith(b"P5"):
        raise FormatError("not a binary PGM: magic is not P5")
    n, pos = len(data), 2
    if pos >= n or (data[pos] not in _PGM_SPACE and data[pos] != ord("#")):
        raise FormatError("malformed PGM header after magic")
    values = []
    while len(values) < 3:
        while pos < n and (data[pos] in _PGM_SPACE or data[pos] == ord("#")):
            if data[pos] == ord("#"):  # comment runs to the end of the line
                eol = data.find(b"\n", pos)
                pos = n if eol < 0 else eol + 1
            else:
                pos += 1
        end = pos
        while end < n and data[end] not in _PGM_SPACE:
            end += 1
        field = data[pos:end]
        if not field.isdigit():
            raise FormatError("malformed PGM header: expected an integer field")
        values.append(int(field))
        pos = end
    width, height, maxval = values
    if maxval != 255:
        raise FormatError(f"unsupported PGM maxval {maxval} (must be 255)")
    if width < 1 or height < 1:
        raise FormatError("PGM extents must be positive")
    if pos >= n or data[pos] not in _PGM_SPACE:
        raise FormatError("malformed PGM header: missing separator before pixels")
    return width, height, maxval, pos + 1  # exactly one separator byte


def read_pgm(data: bytes) -> GrayImage:
    """Parse a P5 PGM byte string into a GrayImage."""
    width, height, _, start = _pgm_header(data)
    need = width * height
    raster = data[start:start + need]
    if len(raster) < need:
        raise FormatError(f"truncated PGM: expected {need} pixel bytes, got {len(raster)}")
    return GrayImage.from_bytes(width, height, raster)


def write_pgm(img: GrayImage) -> bytes:
    """Binary PGM (P5) bytes of an image (reference imgio.py:75-77)."""
    return b"P5\n%d %d\n255\n" % (img.width, img.height) + img.pixels.tobytes()


def write_map_pgm(values) -> bytes:
    """Render fractions in [0, 1] as a P5 image, v -> floor(v * 255 + 0.5)."""
    grid = np.asarray(values, dtype=np.float64)
    if grid.ndim != 2 or grid.size == 0:
        raise ValueError("map must be a non-empty 2D grid")
    if grid.min() < 0.0 or grid.max() > 1.0:
        raise ValueError("map values must lie in [0, 1]")
    px = np.floor(grid * 255.0 + 0.5).astype(np.uint8)
    return b"P5\n%d %d\n255\n" % (grid.shape[1], grid.shape[0]) + px.tobytes()


# ---------------------------------------------------------------------- IHST
def ihst_header(bins: int, width: int, height: int) -> bytes:
    """The 16-byte IHST header `<4sHHII` (reference imgio.py:28)."""
    return _HDR.pack(IHST_MAGIC, IHST_VERSION, bins, width, height)


def serialize_ih(ih: IntegralHistogram) -> bytes:
    """Header + little-endian u32 planes (host copy of the tensor)."""
    body = np.ascontiguousarray(ih.counts).astype("<u4", copy=False)
    return ihst_header(ih.bins, ih.width, ih.height) + body.tobytes()


def deserialize_ih(data: bytes) -> IntegralHistogram:
    """IHST bytes -> IntegralHistogram, with the reference's format checks (imgio.py:97-117)."""
    if len(data) < IHST_HEADER_BYTES:
        raise FormatError("tensor file shorter than its header")
    magic, version, bins, width, height = _HDR.unpack_from(data)
    if magic != IHST_MAGIC:
        raise FormatError(f"bad tensor magic {magic!r}")
    if version != IHST_VERSION:
        raise FormatError(f"unsupported tensor version {version}")
    if min(bins, width, height) < 1:
        raise FormatError("tensor extents must be positive")
    want = IHST_HEADER_BYTES + 4 * bins * width * height
    if len(data) != want:
        raise FormatError(f"tensor length mismatch: expected {want} bytes, got {len(data)}")
    planes = np.frombuffer(data, dtype="<u4", offset=IHST_HEADER_BYTES)
    return IntegralHistogram(planes.astype(np.uint32).reshape(bins, height, width))


def _pwrite_all(fd: int, buf: memoryview, offset: int) -> None:
    """pwrite until every byte is written: one Linux write moves at most
    0x7ffff000 bytes, so a multi-GB plane needs several calls."""
    done, n = 0, len(buf)
    while done < n:
        k = os.pwrite(fd, buf[done:], offset + done)
        if k <= 0:
            raise OSError(f"pwrite wrote {k} bytes at offset {offset + done}")
        done += k


class TensorFileSink:
    """TensorSink writing (bin range, row range) pieces at their final offsets
    of an IHST file; thread-safe, usable with ``compute_streamed``."""

    def __init__(self, path, width: int, height: int, bins: int):
        self.width, self.height, self.bins = width, height, bins
        self._fd = os.open(os.fspath(path), os.O_WRONLY | os.O_CREAT | os.O_TRUNC, 0o644)
        os.pwrite(self._fd, ihst_header(bins, width, height), 0)
        os.ftruncate(self._fd, IHST_HEADER_BYTES + 4 * width * height * bins)
        self._lock = threading.Lock()

    def _offset(self, b: int, row: int) -> int:
        return IHST_HEADER_BYTES + 4 * (b * self.height + row) * self.width

    def write(self, bin_start, bin_stop, row_start, row_stop, data):
        """TensorSink.write: place a (bins, rows, W) chunk at its final file offset (reference imgio.py:134-139)."""
        blocks = np.asarray(data)
        with self._lock:
            for k, b in enumerate(range(bin_start, bin_stop)):
                rows = np.ascontiguousarray(blocks[k]).astype("<u4", copy=False)
                _pwrite_all(self._fd, memoryview(rows).cast("B"), self._offset(b, row_start))

    def close(self):
        """Close the file (reference imgio.py:141-142)."""
        if self._fd is not None:
            os.close(self._fd)
            self._fd = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()


def save_ihst(path, ih: IntegralHistogram, group_bytes: int = 1 << 28) -> int:
    """Write ``ih`` as an IHST file; returns the file size.

    A tensor resident on the device (made by this package) is streamed plane
    group by plane group: pinned D2H of group k+1 on a copy stream overlaps
    the ``pwrite`` of group k.  Host tensors are written directly.
    """
    size = IHST_HEADER_BYTES + 4 * ih.bins * ih.height * ih.width
    dev = getattr(ih, "_dev", None)
    with TensorFileSink(path, ih.width, ih.height, ih.bins) as sink:
        if dev is None:
            sink.write(0, ih.bins, 0, ih.height, ih.counts)
            return size
        import torch

        plane = ih.height * ih.width
        per = max(1, min(ih.bins, group_bytes // (4 * plane)))
        bufs = [torch.empty((per, ih.height, ih.width), dtype=torch.int32, pin_memory=True)
                for _ in range(2)]
        copy = torch.cuda.Stream(dev.device)
        copy.wait_stream(torch.cuda.current_stream(dev.device))
        src = dev.view(torch.int32)
        groups = [(b, min(ih.bins, b + per)) for b in range(0, ih.bins, per)]
        done = [None, None]
        for k, (b0, b1) in enumerate(groups):
            slot = k % 2
            with torch.cuda.stream(copy):
                bufs[slot][: b1 - b0].copy_(src[b0:b1], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(copy)
            done[slot] = ev
            if k:  # write the previous group while this one is in flight
                pb0, pb1 = groups[k - 1]
                done[1 - slot].synchronize()
                sink.write(pb0, pb1, 0, ih.height, bufs[1 - slot][: pb1 - pb0].numpy().view(np.uint32))
        lb0, lb1 = groups[-1]
        done[(len(groups) - 1) % 2].synchronize()
        sink.write(lb0, lb1, 0, ih.height, bufs[(len(groups) - 1) % 2][: lb1 - lb0].numpy().view(np.uint32))
    return size
