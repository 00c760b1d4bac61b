"""Host-buffer batch path: host frames in, host integral histograms out.

The end-to-end form of the reference-facing call for a video batch.  The
output dominates the traffic (4*B bytes per input byte), so the pipeline
overlaps the device->host copy of chunk k with the kernel of chunk k+1 on a
separate stream, through a two-slot device ring:

    stream C : H2D(0) K(0) H2D(1) K(1) H2D(2) K(2) ...
    stream D :                  D2H(0)        D2H(1) ...

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
    """Reusable device state for repeated host-to-host batches of one shape.

    The output is produced in pieces of at most ``max_piece_bytes``: groups of
    ``chunk`` whole frames, or -- for a single frame larger than that (8K x 256
    bins is 68.7 GB) -- bin sub-slabs of one frame.  Each piece lands in one of
    two device ring slots and is copied to its final host offset (both shapes
    are contiguous in the (F, nb, H, W) host buffer) while the next piece is
    computed.
    """

    def __init__(self, frames: int, height: int, width: int, spec: BinSpec, chunk: int = 4,
                 bin_range=None, device_index=None, kernel: str = "auto",
                 max_piece_bytes: int = 2 << 30):
        self.dev = device.require_cuda(device_index)
        self.F, self.H, self.W = frames, height, width
        self.spec = spec
        self.lo, self.hi = (0, spec.bins) if bin_range is None else bin_range
        self.nb = self.hi - self.lo
        self.kernel = kernel
        plane = height * width * 4
        frame_bytes = self.nb * plane
        self.pieces = []
        if frame_bytes <= max_piece_bytes:
            per = max(1, min(chunk, frames, max_piece_bytes // frame_bytes))
            for f0 in range(0, frames, per):
                self.pieces.append((f0, min(frames, f0 + per), self.lo, self.hi))
        else:
            per_b = max(1, max_piece_bytes // plane)
            for f in range(frames):
                for b0 in range(self.lo, self.hi, per_b):
                    self.pieces.append((f, f + 1, b0, min(self.hi, b0 + per_b)))
        slot_elems = max((f1 - f0) * (b1 - b0) for f0, f1, b0, b1 in self.pieces) * height * width
        self.d_in = torch.empty((frames, height, width), dtype=torch.uint8, device=self.dev)
        self.ring = [torch.empty(slot_elems, dtype=torch.uint32, device=self.dev) for _ in range(2)]
        self.s_comp = torch.cuda.Stream(self.dev)
        self.s_copy = torch.cuda.Stream(self.dev)
        self.h2d_bytes = frames * height * width
        self.d2h_bytes = frames * frame_bytes

    def run(self, host_frames: torch.Tensor, host_out: torch.Tensor) -> torch.Tensor:
        """host_frames (F, H, W) uint8 CPU (pinned), host_out (F, nb, H, W) uint32 CPU (pinned).
        Returns host_out after the last copy completed."""
        H, W = self.H, self.W
        slot_free = [None, None]
        uploaded = 0  # frames [0, uploaded) are on the device
        for k, (f0, f1, b0, b1) in enumerate(self.pieces):
            if f1 > uploaded:  # upload a piece's frames just before its kernel: the
                # H2D overlaps the previous piece's D2H (PCIe is full duplex)
                with torch.cuda.stream(self.s_comp):
                    self.d_in[uploaded:f1].copy_(host_frames[uploaded:f1], non_blocking=True)
                uploaded = f1
            slot = k % 2
            n = (f1 - f0) * (b1 - b0) * H * W
            buf = self.ring[slot][:n].view(f1 - f0, b1 - b0, H, W)
            if slot_free[slot] is not None:
                self.s_comp.wait_event(slot_free[slot])
            device.integral_histogram(self.d_in[f0:f1], self.spec.table, self.spec.bins,
                                      bin_range=(b0, b1), out=buf, kernel=self.kernel,
                                      stream=self.s_comp)
            done = torch.cuda.Event()
            done.record(self.s_comp)
            self.s_copy.wait_event(done)
            with torch.cuda.stream(self.s_copy):
                host_out[f0:f1, b0 - self.lo:b1 - self.lo].copy_(buf, non_blocking=True)
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
