"""Single-process multi-GPU integral histograms (the `devices=` form).

The paper's multi-GPU scheme driven from one process (``bench.py`` uses one
process per GPU instead): every device computes an independent part of the
output and no data-path collective exists.

* ``shard="bins"``   -- device g computes bins ``sharding.bin_slabs(B, G)[g]``
  of every frame; every device receives the whole image(s).
* ``shard="frames"`` -- device g computes all bins of the frames
  ``sharding.frame_shards(F, G)[g]``.

All devices' uploads, kernels and result copies are enqueued (each on its own
stream, host buffers pinned) before anything synchronises, so the devices run
concurrently.  The result is delivered as

* ``out="host"``   -- one (F, B, H, W) uint32 numpy array, each device's D2H
  landing directly at its final offset;
* ``out="device"`` -- one tensor on ``devices[root]``: the other devices' parts
  arrive by peer copies (NVLink on an NVSwitch box);
* ``out="shards"`` -- ``[((f0, f1, b0, b1), tensor), ...]`` left where computed.

Devices may repeat (several shards on one GPU, on separate streams).
"""

from __future__ import annotations

import warnings

import numpy as np
import torch

from . import device as _dev
from . import sharding
from .errors import ParameterError, ShapeError


def _host_frames(images) -> torch.Tensor:
    if isinstance(images, torch.Tensor):
        if images.is_cuda:
            raise ParameterError("devices= takes host images (numpy or CPU tensor)")
        t = images
    else:
        with warnings.catch_warnings():  # read-only pixels (GrayImage): never written here
            warnings.simplefilter("ignore", UserWarning)
            t = torch.from_numpy(np.ascontiguousarray(images))
    if t.dtype != torch.uint8:
        raise ShapeError("images must be uint8")
    if t.dim() == 2:
        t = t.unsqueeze(0)
    if t.dim() != 3 or t.numel() == 0:
        raise ShapeError("images must be a non-empty (H, W) or (F, H, W) array")
    return t.contiguous()


def integral_histogram_devices(images, table, bins: int, devices, shard: str = "bins",
                               out: str = "host", root: int = 0):
    """Integral histograms of host frames on several devices (see module doc).
    Bit-identical to the single-device path for every device count."""
    if shard not in ("bins", "frames"):
        raise ParameterError(f"unknown shard mode {shard!r}")
    if out not in ("host", "device", "shards"):
        raise ParameterError(f"unknown output mode {out!r}")
    devs = [_dev.require_cuda(d) for d in devices]
    if not devs:
        raise ParameterError("devices must name at least one CUDA device")
    src = _host_frames(images)
    F, H, W = (int(x) for x in src.shape)
    G = len(devs)
    if shard == "bins":
        parts = [(0, F, b0, b1) for b0, b1 in sharding.bin_slabs(bins, G)]
    else:
        parts = [(f0, f1, 0, bins) for f0, f1 in sharding.frame_shards(F, G)]
    pinned = src if src.is_pinned() else src.pin_memory()

    host = None
    if out == "host":
        host = torch.empty((F, bins, H, W), dtype=torch.uint32, pin_memory=True)
    full = None
    if out == "device":
        full = _dev.empty_output(F, bins, H, W, devs[root])

    results, events = [], []
    for d, (f0, f1, b0, b1) in zip(devs, parts):
        if f1 <= f0 or b1 <= b0:
            results.append(((f0, f1, b0, b1), None))
            continue
        with torch.cuda.device(d):
            s = torch.cuda.Stream(d)
            with torch.cuda.stream(s):
                d_img = torch.empty((f1 - f0, H, W), dtype=torch.uint8, device=d)
                d_img.copy_(pinned[f0:f1], non_blocking=True)
                ws = torch.empty(max(_dev.workspace_bytes(f1 - f0, H, W, b1 - b0), 16),
                                 dtype=torch.uint8, device=d)
                part = _dev.integral_histogram(d_img, table, bins, bin_range=(b0, b1),
                                               stream=s, workspace=ws)
                if host is not None:
                    host[f0:f1, b0:b1].copy_(part, non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(s)
            events.append((d, s, ev, part, f0, f1, b0, b1))
            results.append(((f0, f1, b0, b1), part))
    if full is not None:
        rs = torch.cuda.current_stream(devs[root])
        for d, s, ev, part, f0, f1, b0, b1 in events:
            rs.wait_event(ev)
            with torch.cuda.stream(rs):
                full[f0:f1, b0:b1].copy_(part, non_blocking=True)  # peer copy across devices
        torch.cuda.synchronize(devs[root])  # copies done before the parts are freed
        return full
    for d, s, ev, *_ in events:
        ev.synchronize()
    if host is not None:
        return host.numpy()
    return results
