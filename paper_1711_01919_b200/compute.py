"""Image -> integral histogram: the drop-in strategy API, routed to the B200.

Same public surface as the reference's strategies module
(pkg/src/inthist/strategies.py:36-229): ``Strategy`` with its closed name set,
the three constants, ``wavefront(tile)``, ``resolve_workers``, ``compute`` and
the four ``compute_*`` functions with their signatures and validation order.

Every strategy runs on the device and returns the identical tensor (the
reference's contract):

  every strategy -> K2, the single-pass tiled 2D scan (the paper's CW-B on
  the GPU, K1 + K1b, is 3-4x slower and stays available as
  device.integral_histogram(kernel="crossweave"))

``workers`` is validated (ParameterError when negative, strategies.py:62-65)
and otherwise has no effect: device parallelism is fixed by the kernels.
There is no CPU fallback: without a CUDA device the calls raise DeviceError.
"""

from __future__ import annotations

import os
from dataclasses import dataclass

import numpy as np

from . import device
from .domain import BinSpec, GrayImage, IntegralHistogram
from .errors import ParameterError

DEFAULT_TILE = 64  # strategies.py:34 (wavefront tile side; a schedule hint here)

STRATEGY_NAMES = ("sequential", "crossweave", "sts", "wavefront")

# strategy name -> kernel family of the C ABI (include/inthist_b200.h ih_kernel)
# Every strategy runs the single pass: on the device they are one computation
# (the reference's strategies differ only in CPU parallelisation),
# and the paper's cross-weave kernels (K1 + K1b, 3-4x the output traffic) are
# 3-4x slower -- a caller who picks crossweave as the reference's fastest CPU
# path should not get the slowest device path.  K1 + K1b stay reachable as
# kernel="crossweave" (device API) / IH_KERNEL_CROSSWEAVE (C ABI).
_KERNEL_OF = {
    "sequential": "auto",
    "sts": "auto",
    "wavefront": "auto",
    "crossweave": "auto",
}


@dataclass(frozen=True)
class Strategy:
    """A named route to the tensor; ``tile`` only for wavefront (strategies.py:39-50)."""

    name: str
    tile: int = 0

    def __post_init__(self):
        if self.name not in STRATEGY_NAMES:
            raise ParameterError(f"unknown strategy {self.name!r}")
        is_wf = self.name == "wavefront"
        if is_wf and self.tile < 1:
            raise ParameterError(f"wavefront tile must be >= 1, got {self.tile}")
        if not is_wf and self.tile:
            raise ParameterError("tile is only meaningful for wavefront")


SEQUENTIAL = Strategy("sequential")
CROSSWEAVE = Strategy("crossweave")
SCAN_TRANSPOSE_SCAN = Strategy("sts")


def wavefront(tile: int = DEFAULT_TILE) -> Strategy:
    """Strategy("wavefront", tile) (reference strategies.py:58-59)."""
    return Strategy("wavefront", tile)


def resolve_workers(workers: int) -> int:
    """Validation of the reference's worker cap (strategies.py:62-65)."""
    if workers < 0:
        raise ParameterError(f"worker count must be >= 0, got {workers}")
    return workers or (os.cpu_count() or 1)


def _on_device(img: GrayImage, spec: BinSpec, kernel: str) -> IntegralHistogram:
    dimg = device.upload_image(img.pixels)
    t = device.integral_histogram(dimg, spec.table, spec.bins, kernel=kernel)
    return IntegralHistogram(device_counts=t)


def compute_sequential(img: GrayImage, spec: BinSpec) -> IntegralHistogram:
    """The reference oracle's entry point (strategies.py:109-115), on K2."""
    img.check_capacity()
    return _on_device(img, spec, _KERNEL_OF["sequential"])


def compute_crossweave(img: GrayImage, spec: BinSpec, workers: int = 0) -> IntegralHistogram:
    """CW-B (strategies.py:129-150): capacity, then workers, then the device pass
    (the single pass; K1 + K1b via device.integral_histogram(kernel="crossweave"))."""
    img.check_capacity()
    resolve_workers(workers)
    return _on_device(img, spec, _KERNEL_OF["crossweave"])


def compute_sts(img: GrayImage, spec: BinSpec, workers: int = 0) -> IntegralHistogram:
    """CW-STS entry point (strategies.py:162-169); same tensor via K2."""
    img.check_capacity()
    resolve_workers(workers)
    return _on_device(img, spec, _KERNEL_OF["sts"])


def compute_wavefront(img: GrayImage, spec: BinSpec, tile: int = DEFAULT_TILE,
                      workers: int = 0, trace: list | None = None) -> IntegralHistogram:
    """WF-TiS entry point (strategies.py:172-216): tile, capacity, workers checks
    in the reference's order, then the device pass.

    Without ``trace`` the tensor comes from K2 (the single pass: its row-segment
    carries replace the wavefront, and it is 10-100x faster).  With ``trace``
    the wavefront itself runs on the device (K7, ih_wavefront): t x t tiles
    claimed in anti-diagonal order, each starting only once the tiles above
    and to the left have finished, and ``trace`` receives the recorded
    ("start"|"finish", i, j) events in the order they happened (device-wide
    sequence numbers, the analog of the reference's lock, :194-208).
    """
    if tile < 1:
        raise ParameterError(f"tile must be >= 1, got {tile}")
    img.check_capacity()
    resolve_workers(workers)
    if trace is None:
        return _on_device(img, spec, _KERNEL_OF["wavefront"])
    counts, ev = device.wavefront(device.upload_image(img.pixels), spec.table, spec.bins, tile)
    nj = -(-img.width // tile)
    seqs = ev.cpu().numpy()
    events = []
    for k, (s0, s1) in enumerate(seqs):
        i, j = divmod(k, nj)
        events.append((int(s0), "start", i, j))
        events.append((int(s1), "finish", i, j))
    events.sort()
    trace.extend((kind, i, j) for _, kind, i, j in events)
    return IntegralHistogram(device_counts=counts)


def compute(img: GrayImage, spec: BinSpec, strategy: Strategy, workers: int = 0,
            devices=None) -> IntegralHistogram:
    """Dispatch by strategy name (strategies.py:219-229); results never differ.

    ``devices`` (an extension; the reference has no such argument): a list of
    CUDA devices over which the bins are sharded (the paper's multi-GPU
    decomposition, multi.integral_histogram_devices); the result is the same
    host tensor."""
    if devices is not None:
        from . import multi

        resolve_workers(workers)
        counts = multi.integral_histogram_devices(img.pixels, spec.table, spec.bins, devices,
                                                  shard="bins", out="host")
        return IntegralHistogram(counts[0])
    name = strategy.name
    if name == "wavefront":
        return compute_wavefront(img, spec, strategy.tile, workers)
    if name == "crossweave":
        return compute_crossweave(img, spec, workers)
    if name == "sts":
        return compute_sts(img, spec, workers)
    return compute_sequential(img, spec)


def compute_frames(frames, spec: BinSpec, bin_range=None, kernel: str = "auto", devices=None,
                   shard: str = "frames"):
    """Batched video path (no reference equivalent; the reference takes one
    GrayImage per call): (F, H, W) uint8 host or CUDA frames -> CUDA tensor
    (F, B, H, W) uint32, or the bins [lo, hi) of ``bin_range``.

    With ``devices`` (host frames), the frames (``shard="frames"``) or the bins
    (``shard="bins"``) are split over those devices and the result is
    assembled on ``devices[0]`` by peer copies."""
    import torch

    if devices is not None:
        from . import multi

        if bin_range is not None:
            raise ParameterError("bin_range and devices= cannot be combined")
        return multi.integral_histogram_devices(frames, spec.table, spec.bins, devices,
                                                shard=shard, out="device")

    if isinstance(frames, np.ndarray):
        frames = torch.from_numpy(np.ascontiguousarray(frames, dtype=np.uint8))
    if not frames.is_cuda:
        frames = device.upload_frames(frames)
    return device.integral_histogram(frames, spec.table, spec.bins, bin_range=bin_range,
                                     kernel=kernel)
