"""Device-resident API over the C ABI: torch CUDA tensors in, torch tensors out.

PyTorch is plumbing here (device memory, streams); every computation is one
of the sm_100a kernels behind include/inthist_b200.h.  All calls are
stream-ordered on the current torch stream of the tensor's device and do not
synchronise the host.

    t = integral_histogram(frames_u8, table, bins)            # (F, B, H, W) uint32
    q = region_histograms(t[0], regions_int32)                # (Q, B) uint64
    w = window_counts(t[0], h, w)                             # (B, H-h+1, W-w+1) int64
"""

from __future__ import annotations

import contextlib
import ctypes
import os

import numpy as np
import torch

from . import _native
from .errors import BoundsError, DeviceError, ParameterError, ShapeError

_workspaces: dict[tuple, torch.Tensor] = {}
_cuda_seen = False  # a CUDA device was visible once (availability cannot go away)
_NULLCTX = contextlib.nullcontext()


def require_cuda(device=None) -> torch.device:
    """The CUDA device to run on; raises DeviceError when none exists (no CPU fallback)."""
    global _cuda_seen
    if not _cuda_seen:
        if not torch.cuda.is_available():
            raise DeviceError("no CUDA device visible: the B200 engine has no CPU fallback")
        _native.lib()
        _cuda_seen = True
    if isinstance(device, torch.device) and device.type == "cuda" and device.index is not None:
        return device  # the common case: a tensor's device
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
    if dev.type != "cuda":
        raise DeviceError(f"expected a CUDA device, got {dev}")
    if dev.index is None:
        dev = torch.device("cuda", torch.cuda.current_device())
    return dev


def _stream_handle(dev: torch.device, stream=None) -> int:
    if stream is not None:
        return int(stream.cuda_stream)
    raw = getattr(torch._C, "_cuda_getCurrentRawStream", None)
    if raw is not None:  # the handle without building a Stream object
        return int(raw(dev.index))
    return int(torch.cuda.current_stream(dev).cuda_stream)


def _on_device(dev: torch.device):
    """Context making `dev` current for the C ABI's launches (a no-op when it
    already is: entering torch.cuda.device costs microseconds per call)."""
    return _NULLCTX if torch.cuda.current_device() == dev.index else torch.cuda.device(dev)


def workspace_(dev: torch.device, nbytes: int, stream: int = 0) -> torch.Tensor:
    """Scratch buffer per (device, stream), grown on demand (caller-owned per
    the ABI).  Calls on one stream are ordered, so they can share it; calls on
    different streams (threads, pipelines) get different buffers."""
    key = (dev.index, int(stream))
    ws = _workspaces.get(key)
    if ws is None or ws.numel() < nbytes:
        if ws is not None:
            # kernels queued on `stream` may still read the old buffer, and the
            # caching allocator only orders its reuse against the stream it was
            # allocated on: wait for them (growth is rare), or, inside a graph
            # capture where a sync is illegal, keep the old buffer alive
            if torch.cuda.is_current_stream_capturing():
                _retired.append(ws)
            else:
                torch.cuda.synchronize(dev)
        ws = torch.empty(max(int(nbytes), 16), dtype=torch.uint8, device=dev)
        _workspaces[key] = ws
    return ws


_retired: list = []  # workspaces outgrown during a graph capture (never freed)


# (last uint8 table array (kept alive), its data pointer): one tuple, replaced
# as a whole, so a thread never pairs one table with another's pointer
_lut_last: tuple = (None, 0)


def _lut_array(table) -> np.ndarray:
    lut = np.ascontiguousarray(np.asarray(table), dtype=np.uint8)
    if lut.shape != (256,):
        raise ShapeError("lookup table must have exactly 256 entries")
    return lut


def _lut_ptr(a: "_Args") -> int:
    """Host address of the call's 256-byte table (read by the C ABI during the
    call).  A table that already is a contiguous uint8 array is used in place,
    so its pointer is cached per table object."""
    global _lut_last
    lut = a.lut
    last = _lut_last
    if last[0] is lut:
        return last[1]
    ptr = lut.ctypes.data
    _lut_last = (lut, ptr)
    return ptr


def _frames_view(images: torch.Tensor):
    if not isinstance(images, torch.Tensor):
        raise ShapeError("images must be a torch tensor")
    if images.dtype != torch.uint8:
        raise ShapeError(f"image dtype must be uint8, got {images.dtype}")
    if images.dim() == 2:
        images = images.unsqueeze(0)
    if images.dim() != 3 or images.numel() == 0:
        raise ShapeError("images must be a non-empty (H, W) or (F, H, W) tensor")
    if images.stride(-1) != 1:
        images = images.contiguous()
    return images


class _Args:
    __slots__ = ("images", "frames", "H", "W", "pitch", "fstride", "lut", "bins", "lo", "hi",
                 "kernel", "dev", "stream")


def _restage_aligned(imgs: torch.Tensor, stream) -> torch.Tensor:
    """Copy frames whose rows are not 16-byte aligned into a 16-byte-pitched
    buffer (stream-ordered): the TMA row ring needs aligned rows, and the
    fallback per-lane loads of unaligned rows run at less than half the speed
    (1 CTA/SM at ~100 registers).  The copy is 1/(4B) of the output bytes."""
    F, H, W = (int(x) for x in imgs.shape)
    pitch = (W + 15) // 16 * 16
    ctx = torch.cuda.stream(stream) if stream is not None else torch.cuda.device(imgs.device)
    with ctx:
        buf = torch.empty((F, H, pitch), dtype=torch.uint8, device=imgs.device)
        buf[:, :, :W].copy_(imgs)
    return buf[:, :, :W]


def _aligned16(imgs: torch.Tensor) -> bool:
    F = int(imgs.shape[0])
    return (imgs.data_ptr() % 16 == 0 and imgs.stride(1) % 16 == 0 and
            (F == 1 or imgs.stride(0) % 16 == 0))


def _prepare_args(images, table, bins, bin_range, kernel, stream) -> _Args:
    imgs = _frames_view(images)
    dev = require_cuda(imgs.device)
    if not _aligned16(imgs) and not os.environ.get("IH_NO_RESTAGE"):
        imgs = _restage_aligned(imgs, stream)
    a = _Args()
    a.images = imgs
    a.frames, a.H, a.W = (int(x) for x in imgs.shape)
    a.pitch = int(imgs.stride(1))
    a.fstride = int(imgs.stride(0)) if a.frames > 1 else a.H * a.pitch
    a.lut = _lut_array(table)
    a.bins = int(bins)
    a.lo, a.hi = (0, a.bins) if bin_range is None else (int(bin_range[0]), int(bin_range[1]))
    if kernel not in _native.KERNELS:
        raise ParameterError(f"unknown kernel {kernel!r}; expected one of {sorted(_native.KERNELS)}")
    a.kernel = _native.KERNELS[kernel]
    a.dev = dev
    a.stream = _stream_handle(dev, stream)
    return a


def workspace_bytes(frames: int, height: int, width: int, slab_bins: int, kernel: str = "auto") -> int:
    """Device scratch bytes integral_histogram needs for this shape (ih_workspace_bytes)."""
    return int(_native.lib().ih_workspace_bytes(frames, height, width, slab_bins,
                                                _native.KERNELS[kernel]))


PLAN_FIELDS = ("kernel", "launches", "segments", "segment_rows", "chunks_per_lane",
               "rows_per_batch", "warps_per_cta", "workspace_bytes", "column_tiles", "tile_width",
               "resident_ctas", "ctas_per_segment", "big_segments", "tail_segment_rows",
               "carry", "bins_per_cta")
CARRIES = {0: "none", 1: "table", 2: "lookback", 3: "cluster", 4: "in_kernel"}


def plan(frames: int, height: int, width: int, slab_bins: int, kernel: str = "auto",
         aligned16: bool = True) -> dict:
    """The launch plan the C ABI would use (ih_plan_describe); no device work."""
    info = (ctypes.c_int64 * len(PLAN_FIELDS))()
    _native.check(_native.lib().ih_plan_describe(frames, height, width, slab_bins,
                                                 _native.KERNELS[kernel], int(aligned16), info))
    d = dict(zip(PLAN_FIELDS, list(info)))
    d["kernel"] = {v: k for k, v in _native.KERNELS.items()}[d["kernel"]]
    d["carry"] = CARRIES.get(d["carry"], str(d["carry"]))
    return d


def set_plan_hint(frames: int, height: int, width: int, slab_bins: int, segments: int,
                  tail_pct: int = 0, tail_div: int = 0, cluster: bool = False,
                  small: bool = False, skew: bool = False, kb: int = 0) -> None:
    """Pin the row-segment count (optional tail split, optional cluster/DSMEM
    carries, or the K2s one-launch kernel with its own segmentation) for one
    problem shape; segments = 0 removes the pin.  ``skew=True`` reads
    (tail_pct, tail_div) as (percent of segments dispatched first, their size
    ratio x 100 to the rest): skewed segments that let the older and the
    younger CTA of an SM finish together.  ``kb`` = 2 / 4 pins bin pairs
    (two rows per packed word) or bin quads where the plan allows either."""
    flags = (1 if cluster else 0) | (2 if small else 0) | (4 if skew else 0) | \
        (8 if kb == 2 else 16 if kb == 4 else 0)
    _native.check(_native.lib().ih_plan_hint(frames, height, width, slab_bins, int(segments),
                                             int(tail_pct), int(tail_div), flags))


_TUNED: dict = {}  # (frames, H, W, slab_bins) -> (segments, tail_pct, tail_div), this process


def save_tuning(path: str) -> int:
    """Write this process's autotune results (plan hints) to a JSON file, keyed
    by the GPU model and the ABI version; returns the number of entries."""
    import json

    name = torch.cuda.get_device_name(0) if torch.cuda.is_available() else "none"
    doc = {"gpu": name, "abi": int(_native.lib().ih_abi_version()),
           "hints": [list(k) + list(v) for k, v in sorted(_TUNED.items())]}
    with open(path, "w") as fh:
        json.dump(doc, fh, indent=1)
    return len(_TUNED)


def load_tuning(path: str) -> int:
    """Apply plan hints saved by save_tuning (skipped, returning 0, when they
    were measured on another GPU model or ABI version)."""
    import json

    with open(path) as fh:
        doc = json.load(fh)
    name = torch.cuda.get_device_name(0) if torch.cuda.is_available() else "none"
    if doc.get("gpu") != name or doc.get("abi") != int(_native.lib().ih_abi_version()):
        return 0
    for row in doc["hints"]:
        frames, height, width, nb, segs, tail_pct, tail_div = row[:7]
        flags = row[7] if len(row) > 7 else 0
        set_plan_hint(frames, height, width, nb, segs, tail_pct, tail_div, skew=bool(flags & 4),
                      kb=2 if flags & 8 else 4 if flags & 16 else 0)
        _TUNED[(frames, height, width, nb)] = (segs, tail_pct, tail_div, flags)
    return len(doc["hints"])


def segment_candidates(frames: int, height: int, width: int, slab_bins: int) -> list:
    """Row-segment counts worth measuring for a shape: the heuristic's choice and
    the counts whose scan grid ends just at (or just below) a whole number of
    waves of resident CTAs, 1..12 waves, segments of >= 32 rows."""
    p = plan(frames, height, width, slab_bins)
    if p["kernel"] != "single_pass":
        return []
    slots, units = max(1, p["resident_ctas"]), max(1, p["ctas_per_segment"])
    max_seg = max(1, -(-height // 32))
    cands = {p["segments"]}
    for waves in range(1, 13):
        n = (waves * slots) // units
        for m in (n, n - 1):
            if 1 <= m <= max_seg:
                cands.add(m)
    return sorted(cands)


def autotune(frames: int, height: int, width: int, bins: int, bin_range=None, device=None,
             candidates=None, reps: int = 5, images=None, out=None, objective: str = "call") -> dict:
    """Measure integral_histogram (prepare + scan, CUDA-graph replay) for each
    candidate row-segment count on random frames of this shape, then tail
    splits (10/20/30 % of the rows in quarter-height segments run last), skewed
    segments and (objective "call") the other bins-per-CTA grouping for the
    best count; pin the fastest with set_plan_hint and return
    {"segments", "tail_pct", "tail_div", "skew", "bins_per_cta",
    "ms": {"count[/t<pct>|/s<skew>][/kb<k>]": ms}}.
    Results are bit-identical for every count; only the speed differs.
    ``images`` / ``out`` (CUDA tensors of the call's shapes) avoid allocating
    a second input and output.  ``objective="scan"`` times the scan kernel
    alone (for pipelines that run the prepass of the next batch concurrently,
    as bench.py does); the default times the whole call."""
    if objective not in ("call", "scan"):
        raise ParameterError(f"unknown objective {objective!r}")
    dev = require_cuda(device)
    lo, hi = (0, bins) if bin_range is None else bin_range
    nb = hi - lo
    if candidates is None:
        candidates = segment_candidates(frames, height, width, nb)
    if not candidates:
        return {"segments": None, "ms": {}}
    if images is None:
        gen = torch.Generator(device=dev).manual_seed(1234)
        images = torch.randint(0, 256, (frames, height, width), dtype=torch.uint8, device=dev,
                               generator=gen)
    imgs = images
    lut = ((np.arange(256) * bins) // 256).astype(np.uint8)
    if out is None:
        out = empty_output(frames, nb, height, width, dev)
    need = 16
    for n in candidates:  # the workspace grows with the segment count
        set_plan_hint(frames, height, width, nb, n)
        need = max(need, workspace_bytes(frames, height, width, nb))
    ws = torch.empty(need, dtype=torch.uint8, device=dev)
    side = torch.cuda.Stream(dev)
    times = {}

    def hint(n, tail_pct=0, tail_div=0, flags=0):
        set_plan_hint(frames, height, width, nb, n, tail_pct, tail_div, skew=bool(flags & 4),
                      kb=2 if flags & 8 else 4 if flags & 16 else 0)

    def measure(n, tail_pct=0, tail_div=0, flags=0):
        hint(n, tail_pct, tail_div, flags)
        need = workspace_bytes(frames, height, width, nb)
        w = ws if ws.numel() >= need else torch.empty(need, dtype=torch.uint8, device=dev)
        for _ in range(2):  # warm: attributes, caches
            integral_histogram(imgs, lut, bins, bin_range=bin_range, out=out, workspace=w)
        torch.cuda.synchronize(dev)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=side):
            if objective == "scan":  # the workspace still holds this plan's tables
                scan(imgs, lut, bins, out, bin_range=bin_range, stream=side, workspace=w)
            else:
                integral_histogram(imgs, lut, bins, bin_range=bin_range, out=out, workspace=w)
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        torch.cuda.synchronize(dev)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize(dev)
        # ~40 ms of replays per candidate (at least `reps`): small shapes get
        # more repetitions, so their choice is not decided by timing noise
        n = max(reps, min(200, int(40.0 / max(e0.elapsed_time(e1), 1e-3))))
        e0.record()
        for _ in range(n):
            g.replay()
        e1.record()
        torch.cuda.synchronize(dev)
        del g
        return e0.elapsed_time(e1) / n

    with torch.cuda.device(dev):
        for n in candidates:
            times[(n, 0, 0, 0)] = measure(n)
        # second stage for the best count: short tail segments (run last), and
        # skewed segments (the first half, dispatched first, larger by 15-50 %)
        n0 = min(times, key=times.get)[0]
        if n0 > 1:
            for tail_pct, tail_div, flags in ((10, 4, 0), (20, 4, 0), (30, 4, 0),
                                              (50, 115, 4), (50, 130, 4), (50, 150, 4)):
                hint(n0, tail_pct, tail_div, flags)
                p = plan(frames, height, width, nb)
                if p["big_segments"] < p["segments"]:  # the split applies to this shape
                    times[(n0, tail_pct, tail_div, flags)] = measure(n0, tail_pct, tail_div, flags)
        # third stage (whole calls only): the other bins-per-CTA grouping
        # (pairs <-> quads) for the best split so far, at every candidate
        # count (halving the bins per CTA doubles the CTAs).  Not for
        # objective="scan": a pipeline overlaps consecutive scans, and the
        # isolated scan time misranks the groupings there (profiles/r02k/:
        # 8 HD frames x 32 bins, pairs 2 % faster alone, 4 % slower per step)
        b = min(times, key=times.get)
        hint(*b)
        kb0 = plan(frames, height, width, nb)["bins_per_cta"]
        if kb0 in (2, 4) and objective == "call":
            other = 16 if kb0 == 2 else 8
            for n in sorted({b[0]} | set(candidates)):
                hint(n, b[1], b[2], (b[3] & 4) | other)
                if plan(frames, height, width, nb)["bins_per_cta"] == 6 - kb0 and \
                        workspace_bytes(frames, height, width, nb) <= ws.numel():
                    times[(n, b[1], b[2], (b[3] & 4) | other)] = measure(n, b[1], b[2], (b[3] & 4) | other)
    best = min(times, key=times.get)
    hint(*best)
    _TUNED[(frames, height, width, nb)] = tuple(best)

    def key(k):
        s = f"{k[0]}/s{k[2]}" if k[3] & 4 else f"{k[0]}" + (f"/t{k[1]}" if k[1] else "")
        return s + ("/kb2" if k[3] & 8 else "/kb4" if k[3] & 16 else "")
    return {"segments": best[0], "tail_pct": best[1], "tail_div": best[2],
            "skew": bool(best[3] & 4),
            "bins_per_cta": 2 if best[3] & 8 else 4 if best[3] & 16 else None,
            "ms": {key(k): round(v, 4) for k, v in times.items()},
            "ranked": [list(k) + [round(v, 4)] for k, v in sorted(times.items(), key=lambda x: x[1])]}


class GraphedIntegralHistogram:
    """Repeated integral histograms of one shape as a captured CUDA graph.

    For serving loops over small frames, where the per-call host work
    (argument checks, planning, launches) is comparable to the kernels: the
    call (prepare + scan) is captured once on static buffers and each
    ``__call__`` is one H2D/D2D copy into the static input plus one graph
    replay.  Returns the static (F, B_slab, H, W) output tensor (overwritten
    by the next call; ``.clone()`` to keep it).  Bit-identical to
    integral_histogram.
    """

    def __init__(self, frames: int, height: int, width: int, table, bins: int, bin_range=None,
                 device=None, kernel: str = "auto"):
        self.dev = require_cuda(device)
        lo, hi = (0, bins) if bin_range is None else bin_range
        pitch = (width + 15) // 16 * 16  # TMA-aligned rows
        self._buf = torch.zeros((frames, height, pitch), dtype=torch.uint8, device=self.dev)
        self.images = self._buf[:, :, :width]
        self.out = empty_output(frames, hi - lo, height, width, self.dev)
        self._ws = torch.empty(max(workspace_bytes(frames, height, width, hi - lo, kernel), 16),
                               dtype=torch.uint8, device=self.dev)
        self._args = (table, bins, bin_range, kernel)
        self.stream = torch.cuda.Stream(self.dev)
        with torch.cuda.device(self.dev):
            integral_histogram(self.images, table, bins, bin_range=bin_range, out=self.out,
                               kernel=kernel, workspace=self._ws)  # warm: attributes
            torch.cuda.synchronize(self.dev)
            self.graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(self.graph, stream=self.stream):
                integral_histogram(self.images, table, bins, bin_range=bin_range, out=self.out,
                                   kernel=kernel, workspace=self._ws)

    def __call__(self, images=None) -> torch.Tensor:
        """``images``: (F, H, W) / (H, W) uint8, host (pinned for async) or
        CUDA; None replays on the current contents of ``self.images``."""
        cur = torch.cuda.current_stream(self.dev)
        if images is not None:
            src = images if isinstance(images, torch.Tensor) else torch.from_numpy(
                np.ascontiguousarray(images, dtype=np.uint8))
            self.images.copy_(src.view(self.images.shape), non_blocking=True)
        self.stream.wait_stream(cur)
        self.graph.replay()
        cur.wait_stream(self.stream)
        return self.out


def empty_output(frames: int, slab_bins: int, height: int, width: int, device) -> torch.Tensor:
    """An uninitialised (F, B_slab, H, W) uint32 output tensor on `device`."""
    return torch.empty((frames, slab_bins, height, width), dtype=torch.uint32, device=device)


def integral_histogram(images: torch.Tensor, table, bins: int, bin_range=None, out=None,
                       kernel: str = "auto", stream=None, workspace=None) -> torch.Tensor:
    """Integral histograms of (F, H, W) or (H, W) uint8 CUDA frames.

    Returns (F, hi-lo, H, W) torch.uint32 (or (hi-lo, H, W) for a 2D input):
    the bin-major tensor of IntegralHistogram.counts (core.py:106-116) for the
    bins [lo, hi) of ``bin_range`` (default: all).  Bit-identical to every
    reference strategy (strategies.py:109-229).  The default scratch buffer is
    per (device, stream), so concurrent calls on different streams do not
    share it; ``workspace`` (a uint8 CUDA tensor of ``workspace_bytes(...)``
    bytes) overrides it.
    """
    squeeze = images.dim() == 2 and out is None
    a = _prepare_args(images, table, bins, bin_range, kernel, stream)
    nb = a.hi - a.lo
    if nb < 1 or a.lo < 0 or a.hi > a.bins:
        raise ShapeError("bin slab must satisfy 0 <= lo < hi <= bins")
    if out is None:  # allocated on the launch stream, so its reuse is ordered after the kernels
        with (torch.cuda.stream(stream) if stream is not None else _NULLCTX):
            out = empty_output(a.frames, nb, a.H, a.W, a.dev)
    else:
        _check_ih_out(out, a, nb)
    ws = _workspace_for(a, workspace)
    L = _native.lib()
    with _on_device(a.dev):  # launches go to the tensors' device
        _native.check(L.ih_integral_histogram(
            a.images.data_ptr(), a.frames, a.H, a.W, a.pitch, a.fstride, _lut_ptr(a),
            a.bins, a.lo, a.hi, out.data_ptr(), ws.data_ptr(), ws.numel() * ws.element_size(),
            a.kernel, a.stream))
    if squeeze and out.dim() == 4:
        return out[0]
    return out


def _check_ih_out(out, a: "_Args", nb: int) -> None:
    """A caller-provided output of integral_histogram / scan: contiguous
    uint32 (or int32) with frames*nb*H*W elements on the images' device.  The
    C ABI also rejects a misaligned pointer (16 bytes when W % 4 == 0)."""
    if not isinstance(out, torch.Tensor) or out.dtype not in (torch.uint32, torch.int32) or \
            not out.is_contiguous():
        raise ShapeError("out must be a contiguous uint32 tensor")
    if out.numel() != a.frames * nb * a.H * a.W or out.device != a.dev:
        raise ShapeError("out has the wrong size or device")


def _workspace_for(a: "_Args", workspace, per_stream: bool = True) -> torch.Tensor:
    """The call's scratch: ``workspace`` if given, else the default buffer of
    (device, stream) -- or of the device alone for the prepare/scan split,
    whose two halves may be issued on different (caller-synchronised)
    streams and must find the same carries."""
    need = _native.lib().ih_workspace_bytes(a.frames, a.H, a.W, a.hi - a.lo, a.kernel)
    if workspace is None:
        return workspace_(a.dev, need, a.stream if per_stream else 0)
    if workspace.numel() * workspace.element_size() < need or not workspace.is_cuda:
        raise ParameterError(f"workspace needs {need} bytes on the device")
    return workspace


def prepare(images, table, bins, bin_range=None, kernel="auto", stream=None,
            workspace=None) -> None:
    """Phase 1 of integral_histogram (row-segment carries into the workspace).

    Reads only the images: with a caller-owned ``workspace`` per in-flight
    batch, the phase for batch k+1 can run on a side stream while batch k's
    scan (write-bound) runs."""
    a = _prepare_args(images, table, bins, bin_range, kernel, stream)
    ws = _workspace_for(a, workspace, per_stream=False)
    with _on_device(a.dev):
        _native.check(_native.lib().ih_ih_prepare(
            a.images.data_ptr(), a.frames, a.H, a.W, a.pitch, a.fstride, _lut_ptr(a),
            a.bins, a.lo, a.hi, ws.data_ptr(), ws.numel() * ws.element_size(), a.kernel,
            a.stream))


def scan(images, table, bins, out, bin_range=None, kernel="auto", stream=None,
         workspace=None) -> torch.Tensor:
    """Phase 2 of integral_histogram (the dominant single-pass kernel)."""
    a = _prepare_args(images, table, bins, bin_range, kernel, stream)
    nb = a.hi - a.lo
    if nb < 1 or a.lo < 0 or a.hi > a.bins:
        raise ShapeError("bin slab must satisfy 0 <= lo < hi <= bins")
    _check_ih_out(out, a, nb)
    ws = _workspace_for(a, workspace, per_stream=False)
    with _on_device(a.dev):
        _native.check(_native.lib().ih_ih_scan(
            a.images.data_ptr(), a.frames, a.H, a.W, a.pitch, a.fstride, _lut_ptr(a),
            a.bins, a.lo, a.hi, out.data_ptr(), ws.data_ptr(), ws.numel() * ws.element_size(),
            a.kernel, a.stream))
    return out


def wavefront(image: torch.Tensor, table, bins: int, tile: int, stream=None):
    """The wavefront tiled scan as scheduled on the device (K7, ih_wavefront).

    ``image``: (H, W) uint8 CUDA tensor.  Returns ``(counts, events)``:
    counts (bins, H, W) uint32 (bit-identical to integral_histogram) and
    events, an (ni*nj, 2) int64 CUDA tensor holding for tile i*nj + j the
    global sequence numbers of its "start" and "finish" (strategies.py:194-208).
    """
    if tile < 1:
        raise ParameterError(f"tile must be >= 1, got {tile}")
    a = _prepare_args(image, table, bins, None, "auto", stream)
    if a.frames != 1:
        raise ShapeError("wavefront takes one (H, W) image")
    ni, nj = -(-a.H // tile), -(-a.W // tile)
    out = empty_output(1, a.bins, a.H, a.W, a.dev)[0]
    L = _native.lib()
    need = int(L.ih_wavefront_workspace_bytes(a.H, a.W, int(tile)))
    ctx = torch.cuda.stream(stream) if stream is not None else torch.cuda.device(a.dev)
    with ctx:
        ws = torch.empty(max(need, 16), dtype=torch.uint8, device=a.dev)
        ev = torch.empty((ni * nj, 2), dtype=torch.int32, device=a.dev)
        _native.check(L.ih_wavefront(a.images.data_ptr(), a.H, a.W, a.pitch, a.lut.ctypes.data,
                                     a.bins, int(tile), out.data_ptr(), ev.data_ptr(),
                                     ws.data_ptr(), need, a.stream))
    return out, ev.to(torch.int64)


def _check_tensor(t: torch.Tensor) -> torch.Tensor:
    if t.dim() != 3 or t.dtype not in (torch.uint32, torch.int32):
        raise ShapeError("tensor must be a 3D uint32 array (bins, height, width)")
    if not t.is_cuda:
        raise DeviceError("integral-histogram tensor must live on a CUDA device")
    return t.contiguous()


_I32_MAX = (1 << 31) - 1


def _validate_device_regions(regs: torch.Tensor, H: int, W: int) -> None:
    """core.py:142 (degenerate) then core.py:158 (outside) for regions already
    on the device: one fused reduction, one small D2H (a sync)."""
    r0, c0, r1, c1 = regs.unbind(1)
    bad = torch.stack([((r0 < 0) | (c0 < 0) | (r0 > r1) | (c0 > c1)).any(),
                       ((r1 >= H) | (c1 >= W)).any(),
                       (regs > _I32_MAX).any()]).cpu().tolist()
    if bad[0]:
        raise BoundsError("degenerate region")
    if bad[1]:
        raise BoundsError(f"region outside {W}x{H} image")
    if bad[2]:
        raise ParameterError("region coordinates must fit in int32")


def region_histograms(t: torch.Tensor, regions, stream=None, out=None,
                      validate: bool = True) -> torch.Tensor:
    """Batched core.py:179-195: (Q, 4) inclusive (r0,c0,r1,c1) -> (Q, nb) uint64.

    Validation follows core.py:142 (degenerate) then core.py:158 (outside)
    for host and device regions alike (device regions: one reduction and a
    sync; ``validate=False`` skips it for regions the caller has already
    checked -- the kernel never reads outside the tensor either way, but an
    out-of-range region then yields unspecified counts).  Uploads and the
    output allocation are ordered on ``stream`` (default: the current stream).
    """
    t = _check_tensor(t)
    nb, H, W = (int(x) for x in t.shape)
    st = stream if stream is not None else torch.cuda.current_stream(t.device)
    with torch.cuda.device(t.device), torch.cuda.stream(st):
        if isinstance(regions, torch.Tensor) and regions.is_cuda:
            if regions.dtype.is_floating_point or regions.dtype == torch.bool:
                raise ParameterError("regions must be an integer tensor")
            r64 = regions.reshape(-1, 4).to(torch.int64)
            if validate and r64.shape[0]:
                _validate_device_regions(r64, H, W)
            regs = r64.to(torch.int32).contiguous()
        else:
            r = np.ascontiguousarray(np.asarray(regions, dtype=np.int64).reshape(-1, 4))
            if r.size:
                if ((r[:, 0] < 0) | (r[:, 1] < 0) | (r[:, 0] > r[:, 2]) | (r[:, 1] > r[:, 3])).any():
                    raise BoundsError("degenerate region")
                if ((r[:, 2] >= H) | (r[:, 3] >= W)).any():
                    raise BoundsError(f"region outside {W}x{H} image")
                if (r > _I32_MAX).any():
                    raise ParameterError("region coordinates must fit in int32")
            regs = torch.from_numpy(r.astype(np.int32)).to(t.device, non_blocking=False)
        Q = int(regs.shape[0])
        if out is None:
            out = torch.empty((Q, nb), dtype=torch.uint64, device=t.device)
        elif out.shape != (Q, nb) or out.dtype not in (torch.uint64, torch.int64) or \
                not out.is_contiguous() or out.device != t.device:
            raise ShapeError(f"out must be a contiguous ({Q}, {nb}) uint64 tensor on {t.device}")
        if Q:
            _native.check(_native.lib().ih_region_histograms(
                t.data_ptr(), nb, H, W, regs.data_ptr(), Q, out.data_ptr(), int(st.cuda_stream)))
    return out


def _check_out(out, shape, dtypes, dev):
    if out.shape != shape or out.dtype not in dtypes or not out.is_contiguous() or out.device != dev:
        raise ShapeError(f"out must be a contiguous {tuple(shape)} {dtypes[0]} tensor on {dev}")
    return out


def window_counts(t: torch.Tensor, h: int, w: int, stream=None, out=None) -> torch.Tensor:
    """likelihood.py:34-52 on the device -> (nb, H-h+1, W-w+1) int64."""
    if h < 1 or w < 1:
        raise ParameterError("window extents must be >= 1")
    t = _check_tensor(t)
    nb, H, W = (int(x) for x in t.shape)
    if h > H or w > W:
        raise BoundsError(f"{h}x{w} window exceeds {W}x{H} image")
    shape = (nb, H - h + 1, W - w + 1)
    st = stream if stream is not None else torch.cuda.current_stream(t.device)
    with torch.cuda.device(t.device), torch.cuda.stream(st):
        out = torch.empty(shape, dtype=torch.int64, device=t.device) if out is None else \
            _check_out(out, shape, (torch.int64,), t.device)
        _native.check(_native.lib().ih_window_counts(
            t.data_ptr(), nb, H, W, int(h), int(w), out.data_ptr(), int(st.cuda_stream)))
    return out


def likelihood_map(t: torch.Tensor, template, h: int, w: int, metric: str = "bhattacharyya",
                   stream=None, out=None) -> torch.Tensor:
    """Fused K5 (likelihood.py:55-77): (H-h+1, W-w+1) float64 map on the device."""
    metrics = {"intersection": 0, "bhattacharyya": 1}
    if metric not in metrics:
        raise ParameterError(f"unknown metric {metric!r}")
    if h < 1 or w < 1:
        raise ParameterError("window extents must be >= 1")
    t = _check_tensor(t)
    nb, H, W = (int(x) for x in t.shape)
    tmpl = np.ascontiguousarray(np.asarray(template, dtype=np.float64))
    if tmpl.shape != (nb,):
        raise ShapeError(f"template has {tmpl.shape} entries, tensor has {nb} bins")
    if h > H or w > W:
        raise BoundsError(f"{h}x{w} window exceeds {W}x{H} image")
    shape = (H - h + 1, W - w + 1)
    with torch.cuda.device(t.device), (torch.cuda.stream(stream) if stream is not None else _NULLCTX):
        out = torch.empty(shape, dtype=torch.float64, device=t.device) if out is None else \
            _check_out(out, shape, (torch.float64,), t.device)
    L = _native.lib()
    nws = int(L.ih_likelihood_workspace_bytes(nb, int(h), int(w)))
    with torch.cuda.device(t.device):
        ws = torch.empty(max(nws, 16), dtype=torch.uint8, device=t.device)  # stream-ordered reuse
        _native.check(L.ih_likelihood_map_ws(
            t.data_ptr(), nb, H, W, int(h), int(w), tmpl.ctypes.data, metrics[metric],
            out.data_ptr(), ws.data_ptr(), nws, _stream_handle(t.device, stream)))
        if stream is not None:
            ws.record_stream(stream)  # freed at return: keep it until `stream` is done
    return out


PINNED_MIN_BYTES = 1 << 20
PRIVATE_PINNED_MIN_BYTES = 1 << 30
_VIEW_AS = {torch.uint32: (torch.int32, np.uint32), torch.uint64: (torch.int64, np.uint64)}


def _private_pinned(shape, dtype: torch.dtype):
    """A host tensor in its own page-locked allocation (ih_host_alloc), freed
    (ih_host_free) when the last numpy/torch view of it is garbage-collected;
    None if the pages cannot be locked."""
    import weakref

    nbytes = int(np.prod(shape)) * torch.empty((), dtype=dtype).element_size()
    L = _native.lib()
    ptr = L.ih_host_alloc(nbytes)
    if not ptr:
        return None
    raw = (ctypes.c_uint8 * nbytes).from_address(ptr)
    weakref.finalize(raw, L.ih_host_free, ptr)
    flat = np.frombuffer(raw, dtype=np.uint8)  # keeps `raw` alive
    return torch.from_numpy(flat).view(dtype).view(shape)


def to_host(t: torch.Tensor) -> np.ndarray:
    """D2H of a device result into a numpy array of the same dtype.

    Results of 1 MB and more land in page-locked memory (~55 GB/s; a fresh
    pageable array page-faults on first touch and the copy runs at ~2 GB/s):
    below 1 GB from torch's caching host allocator (blocks reused across
    calls), from 1 GB up in a private page-locked allocation that is returned
    to the OS when the array dies -- a cached block would pin e.g. 68.7 GB
    for an 8192^2 x 256 result for the life of the process.  The array is a
    view that keeps its block alive.  ``IH_NO_PINNED=1`` disables both.
    """
    src, np_view = t, None
    if t.dtype in _VIEW_AS:
        carrier, np_view = _VIEW_AS[t.dtype]
        src = t.view(carrier)
    nbytes = src.numel() * src.element_size()
    host = None
    if nbytes >= PINNED_MIN_BYTES and os.environ.get("IH_NO_PINNED", "0") == "0":
        if nbytes >= PRIVATE_PINNED_MIN_BYTES:
            host = _private_pinned(tuple(src.shape), src.dtype)
        if host is None:
            host = torch.empty(src.shape, dtype=src.dtype, pin_memory=True)
        host.copy_(src)
        arr = host.numpy()
    else:
        arr = src.cpu().numpy()
    return arr.view(np_view) if np_view is not None else arr


def upload_frames(frames, device=None) -> torch.Tensor:
    """H2D of host (F, H, W) uint8 frames into a 16-byte-pitched device buffer
    (the TMA path for every width).  Returns the (F, H, W) view."""
    dev = require_cuda(device)
    src = frames if isinstance(frames, torch.Tensor) else \
        torch.from_numpy(np.require(frames, dtype=np.uint8, requirements=["C", "W"]))
    F, H, W = (int(x) for x in src.shape)
    if W % 16 == 0:
        return src.to(dev)
    pitch = (W + 15) // 16 * 16
    buf = torch.empty((F, H, pitch), dtype=torch.uint8, device=dev)
    buf[:, :, :W].copy_(src)
    return buf[:, :, :W]


def upload_image(pixels: np.ndarray, device=None) -> torch.Tensor:
    """H2D of a host (H, W) uint8 image into a 16-byte-pitched device buffer
    (aligned 32-bit pixel loads in the kernels for every width).  Returns the
    (H, W) view."""
    dev = require_cuda(device)
    px = np.require(pixels, dtype=np.uint8, requirements=["C", "W"])  # torch needs writable
    H, W = px.shape
    if W % 16 == 0:
        return torch.from_numpy(px).to(dev)
    pitch = (W + 15) // 16 * 16
    buf = torch.empty((H, pitch), dtype=torch.uint8, device=dev)
    buf[:, :W].copy_(torch.from_numpy(px))
    return buf[:, :W]
