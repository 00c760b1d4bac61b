"""CPU oracle for the integral-histogram hot path -- TEST INFRASTRUCTURE ONLY.

Two restatements of the reference `inthist` algorithms (paths below are
relative to the reference package ``pkg/src/inthist/``):

* ``libih_oracle.so`` (``ih_oracle.c``, plain C + OpenMP) -- the sequential
  recursion (strategies.py:86-115), the threaded cross-weave
  (strategies.py:118-150), region queries (core.py:179-195), window counts
  (likelihood.py:34-52) and the streamed per-plane crc32 (streaming.py:123-155).
* numpy restatements of the same functions, used to cross-check the C code,
  and of the scan module (scan.py:20-92; pinned by tests/golden/scans.npz).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline
leg may import this module.  The product package never does; it has no CPU
fallback.  Parity of this oracle is pinned to golden vectors produced by the
reference itself (tests/golden/make_golden.py).
"""

from __future__ import annotations

import ctypes
import os
import subprocess
import zlib

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libih_oracle.so")
_lib = None

U32_MAX = 2**32 - 1


def build() -> str:
    """Compile libih_oracle.so with the committed Makefile (gcc, no GPU)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        src = os.path.join(_HERE, "ih_oracle.c")
        if not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(src):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        P = ctypes.c_void_p
        i64, i32, u32 = ctypes.c_int64, ctypes.c_int32, ctypes.c_uint32
        L.iho_compute_sequential.argtypes = [P, i64, i64, i64, P, i32, P]
        L.iho_compute_sequential.restype = None
        L.iho_compute_crossweave.argtypes = [P, i64, i64, i64, P, i32, P, i32]
        L.iho_compute_crossweave.restype = None
        L.iho_plane_crc32.argtypes = [P, i64, i64, i64, P, i32, u32]
        L.iho_plane_crc32.restype = u32
        L.iho_crc32.argtypes = [P, ctypes.c_uint64, u32]
        L.iho_crc32.restype = u32
        L.iho_region_histograms.argtypes = [P, i32, i64, i64, P, i64, P]
        L.iho_region_histograms.restype = None
        L.iho_window_counts.argtypes = [P, i32, i64, i64, i64, i64, P]
        L.iho_window_counts.restype = None
        L.iho_max_threads.argtypes = []
        L.iho_max_threads.restype = ctypes.c_int
        _lib = L
    return _lib


def _ptr(a: np.ndarray):
    return ctypes.c_void_p(a.ctypes.data)


def _prep(pixels, table):
    px = np.ascontiguousarray(pixels, dtype=np.uint8)
    lut = np.ascontiguousarray(table, dtype=np.uint8)
    assert px.ndim == 2 and lut.shape == (256,)
    return px, lut


# ---------------------------------------------------------------- C oracle
def compute_sequential(pixels, table, bins) -> np.ndarray:
    """strategies.py:109-115 -- (bins, H, W) u32 via the fused recursion."""
    px, lut = _prep(pixels, table)
    H, W = px.shape
    out = np.empty((bins, H, W), dtype=np.uint32)
    lib().iho_compute_sequential(_ptr(px), H, W, W, _ptr(lut), bins, _ptr(out))
    return out


def compute_crossweave(pixels, table, bins, workers: int = 0) -> np.ndarray:
    """strategies.py:129-150 -- threaded CW-B (row scans, barrier, column scans)."""
    px, lut = _prep(pixels, table)
    H, W = px.shape
    out = np.empty((bins, H, W), dtype=np.uint32)
    lib().iho_compute_crossweave(_ptr(px), H, W, W, _ptr(lut), bins, _ptr(out), workers)
    return out


def plane_crc32(pixels, table, b: int, crc_in: int = 0) -> int:
    """streaming.py:123-155 with one-bin chunks: crc32 of plane b in O(W) memory."""
    px, lut = _prep(pixels, table)
    H, W = px.shape
    return int(lib().iho_plane_crc32(_ptr(px), H, W, W, _ptr(lut), b, crc_in))


def region_histograms(counts: np.ndarray, regions) -> np.ndarray:
    """core.py:179-195 for a batch of (r0,c0,r1,c1) rows -> (Q, bins) u64."""
    t = np.ascontiguousarray(counts, dtype=np.uint32)
    regs = np.ascontiguousarray(np.asarray(regions, dtype=np.int32).reshape(-1, 4))
    bins, H, W = t.shape
    out = np.empty((regs.shape[0], bins), dtype=np.uint64)
    lib().iho_region_histograms(_ptr(t), bins, H, W, _ptr(regs), regs.shape[0], _ptr(out))
    return out


def window_counts(counts: np.ndarray, h: int, w: int) -> np.ndarray:
    """likelihood.py:34-52 -> (bins, H-h+1, W-w+1) int64."""
    t = np.ascontiguousarray(counts, dtype=np.uint32)
    bins, H, W = t.shape
    out = np.empty((bins, H - h + 1, W - w + 1), dtype=np.int64)
    lib().iho_window_counts(_ptr(t), bins, H, W, h, w, _ptr(out))
    return out


def max_threads() -> int:
    return int(lib().iho_max_threads())


# ------------------------------------------------------------ numpy oracle
def np_uniform_table(bins: int) -> np.ndarray:
    """core.py:83-87 -- floor(v * bins / 256)."""
    return ((np.arange(256) * bins) // 256).astype(np.uint8)


def np_compute(pixels, table, bins) -> np.ndarray:
    """strategies.py:118-150 restated in numpy: one-hot, row cumsum, column cumsum."""
    binned = np.asarray(table, dtype=np.uint8)[np.asarray(pixels, dtype=np.uint8)]
    onehot = (binned[None, :, :] == np.arange(bins, dtype=np.uint8)[:, None, None])
    t = np.cumsum(onehot, axis=2, dtype=np.uint32)
    np.cumsum(t, axis=1, dtype=np.uint32, out=t)
    return t


def np_region_histogram(counts, r0, c0, r1, c1) -> np.ndarray:
    """core.py:179-195 restated: four corners, int64, zero outside."""
    t = counts

    def corner(r, c):
        if r < 0 or c < 0:
            return np.zeros(t.shape[0], dtype=np.int64)
        return t[:, r, c].astype(np.int64)

    h = corner(r1, c1) - corner(r0 - 1, c1) - corner(r1, c0 - 1) + corner(r0 - 1, c0 - 1)
    return h.astype(np.uint64)


def np_window_counts(counts, h, w) -> np.ndarray:
    """likelihood.py:34-52 restated with shifted slabs."""
    t = counts
    _, H, W = t.shape
    out = t[:, h - 1:, w - 1:].astype(np.int64)
    out[:, 1:, :] -= t[:, : H - h, w - 1:]
    out[:, :, 1:] -= t[:, h - 1:, : W - w]
    out[:, 1:, 1:] += t[:, : H - h, : W - w]
    return out


def np_likelihood_map(counts, template, h, w, metric) -> np.ndarray:
    """likelihood.py:55-77 restated: window counts -> q = c / (h*w) -> metric
    per bin -> sum over the bin axis -> clip to [0, 1] (float64 numpy ops)."""
    q = np_window_counts(counts, h, w).astype(np.float64) / float(h * w)
    t = np.asarray(template, dtype=np.float64)[:, None, None]
    vals = np.minimum(t, q).sum(axis=0) if metric == "intersection" else np.sqrt(t * q).sum(axis=0)
    return np.clip(vals, 0.0, 1.0)


def brute_integral_histogram(pixels, table, bins) -> np.ndarray:
    """tests/conftest.py:17-27 restated: O((WH)^2) direct counting (tiny images)."""
    binned = np.asarray(table, dtype=np.uint8)[np.asarray(pixels, dtype=np.uint8)]
    H, W = binned.shape
    out = np.zeros((bins, H, W), dtype=np.uint32)
    for r in range(H):
        for c in range(W):
            out[:, r, c] = np.bincount(binned[: r + 1, : c + 1].ravel(), minlength=bins)[:bins]
    return out


def brute_region_counts(pixels, table, bins, r0, c0, r1, c1) -> np.ndarray:
    """tests/conftest.py:11-14 restated: bincount over an inclusive rectangle."""
    patch = np.asarray(table)[np.asarray(pixels)[r0 : r1 + 1, c0 : c1 + 1]]
    return np.bincount(patch.ravel(), minlength=bins).astype(np.uint64)


def tensor_checksum(counts: np.ndarray) -> str:
    """bench.py:65-66 -- crc32 of the little-endian u32 bytes."""
    return f"{zlib.crc32(np.ascontiguousarray(counts).astype('<u4', copy=False).tobytes()):08x}"


def synth_image(width: int, height: int, seed: int) -> np.ndarray:
    """bench.py:59-62 -- deterministic uniform u8 image for (seed, W, H)."""
    rng = np.random.default_rng(np.random.SeedSequence([seed, width, height]))
    return rng.integers(0, 256, size=(height, width), dtype=np.uint8)


class ScanOverflow(ArithmeticError):
    """A 1-D prefix above 2^32-1 (the reference raises ScanOverflowError, scan.py:27-30)."""


def _np_u32_prefixes(sums: np.ndarray) -> np.ndarray:
    if sums.size and int(sums.max()) > 0xFFFF_FFFF:
        raise ScanOverflow("prefix sum exceeds 32-bit range")
    return sums.astype(np.uint32)


def np_inclusive_scan(seq) -> np.ndarray:
    """scan.py:20-36 restated: elements as uint64 (mod 2^64 sums), u32 result."""
    v = np.asarray(seq).astype(np.uint64).reshape(-1)
    return _np_u32_prefixes(np.cumsum(v, dtype=np.uint64))


def np_exclusive_scan(seq) -> np.ndarray:
    """scan.py:39-44 restated: the inclusive prefixes shifted right by one."""
    v = np.asarray(seq).astype(np.uint64).reshape(-1)
    sums = np.concatenate([np.zeros(1, np.uint64), np.cumsum(v, dtype=np.uint64)])[:v.size]
    return _np_u32_prefixes(sums)


def np_blocked_scan(seq, block: int) -> np.ndarray:
    """scan.py:47-76 restated with explicit phases (block >= 1): per-block
    prefixes, exclusive scan of block totals, offset add."""
    v = np.asarray(seq).astype(np.uint64).reshape(-1)
    if v.size == 0:
        return np.zeros(0, np.uint32)
    pad = (-v.size) % block
    blocks = np.concatenate([v, np.zeros(pad, np.uint64)]).reshape(-1, block)
    local = np.cumsum(blocks, axis=1, dtype=np.uint64)
    offs = np.cumsum(local[:, -1], dtype=np.uint64) - local[:, -1]
    return _np_u32_prefixes((local + offs[:, None]).reshape(-1)[:v.size])


def np_scan_axis(plane, axis: int) -> np.ndarray:
    """scan.py:79-92 restated: per-element u32 cast, wrapping u32 prefix along axis."""
    a = np.asarray(plane)
    return np.cumsum(a.astype(np.uint32), axis=axis, dtype=np.uint32)
