"""Host-buffer batch path: host frames in, host integral histograms out.

The end-to-end form of the reference-facing call for a video batch.  The
output dominates the traffic (4*B bytes per input byte), so the pipeline
overlaps the device->host copy of chunk k with the kernel of chunk k+1 on a
separate stream, through a two-slot device ring:

    stream C : H2D(all frames)  K(0)  K(1)  K(2) ...
    stream D :                        D2H(0) D2H(1) ...

Host buffers should be pinned (``pinned_empty``) for full PCIe bandwidth.
"""

from __future__ import annotations

import numpy as np
import torch

from . import device
from .domain import BinSpec


def pinned_empty(shape, dtype=torch.uint32) -> torch.Tensor:
    """Page-locked host tensor (cudaHostAlloc through torch)."""
    return torch.empty(shape, dtype=dtype, pin_memory=True)


class FramePipeline:
    """Reusable device state for repeated host-to-host batches of one shape."""

    def __init__(self, frames: int, height: int, width: int, spec: BinSpec, chunk: int = 4,
                 bin_range=None, device_index=None, kernel: str = "auto"):
        self.dev = device.require_cuda(device_index)
        self.F, self.H, self.W = frames, height, width
        self.spec = spec
        self.lo, self.hi = (0, spec.bins) if bin_range is None else bin_range
        self.nb = self.hi - self.lo
        self.chunk = max(1, min(chunk, frames))
        self.kernel = kernel
        self.d_in = torch.empty((frames, height, width), dtype=torch.uint8, device=self.dev)
        self.ring = [device.empty_output(self.chunk, self.nb, height, width, self.dev)
                     for _ in range(2)]
        self.s_comp = torch.cuda.Stream(self.dev)
        self.s_copy = torch.cuda.Stream(self.dev)
        self.h2d_bytes = frames * height * width
        self.d2h_bytes = frames * self.nb * height * width * 4

    def run(self, host_frames: torch.Tensor, host_out: torch.Tensor) -> torch.Tensor:
        """host_frames (F, H, W) uint8 CPU (pinned), host_out (F, nb, H, W) uint32 CPU (pinned).
        Returns host_out after the last copy completed."""
        F, c = self.F, self.chunk
        slot_free = [None, None]
        with torch.cuda.stream(self.s_comp):
            self.d_in.copy_(host_frames, non_blocking=True)
        for k, f0 in enumerate(range(0, F, c)):
            f1 = min(F, f0 + c)
            slot = k % 2
            buf = self.ring[slot][: f1 - f0]
            if slot_free[slot] is not None:
                self.s_comp.wait_event(slot_free[slot])
            device.integral_histogram(self.d_in[f0:f1], self.spec.table, self.spec.bins,
                                      bin_range=(self.lo, self.hi), out=buf,
                                      kernel=self.kernel, stream=self.s_comp)
            done = torch.cuda.Event()
            done.record(self.s_comp)
            self.s_copy.wait_event(done)
            with torch.cuda.stream(self.s_copy):
                host_out[f0:f1].copy_(buf, non_blocking=True)
            freed = torch.cuda.Event()
            freed.record(self.s_copy)
            slot_free[slot] = freed
        self.s_copy.synchronize()
        return host_out


def compute_frames_host(frames, spec: BinSpec, out=None, chunk: int = 4, bin_range=None):
    """One-shot host batch: (F, H, W) uint8 numpy/torch -> (F, nb, H, W) uint32 numpy."""
    src = torch.from_numpy(np.ascontiguousarray(frames, dtype=np.uint8)) \
        if isinstance(frames, np.ndarray) else frames
    F, H, W = (int(x) for x in src.shape)
    pipe = FramePipeline(F, H, W, spec, chunk=chunk, bin_range=bin_range)
    if out is None:
        out = pinned_empty((F, pipe.nb, H, W))
    pipe.run(src, out)
    return out.numpy()
