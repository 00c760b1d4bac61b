"""Multi-GPU partitioning: bin slabs and frame shards, one process per GPU.

The paper's multi-GPU scheme (BASELINE.json north_star): every GPU computes
an independent part of the output with no data-path collective.

* bin sharding  -- GPU g owns bins [g*ceil(B/G), min(B, (g+1)*ceil(B/G))): a
  contiguous slab of the bin-major (B, H, W) tensor, the same partition as the
  reference's streaming bin chunks (streaming.py:81-82).  Every GPU reads the
  whole image (8 MB at 4K) and writes only its slab.
* frame sharding -- a video batch of F frames split into contiguous runs.

``gather_slabs`` is the optional "single device tensor" step: grouped
point-to-point sends of each rank's slab into the root's full tensor (NCCL
over NVLink on the GPU box, gloo in the CPU tests).  It is never part of the
throughput metric.
"""

from __future__ import annotations

from typing import Callable

import torch


def bin_slabs(bins: int, world: int) -> list[tuple[int, int]]:
    """Contiguous bin ranges per rank; trailing ranks may be empty when world > bins."""
    if bins < 1 or world < 1:
        raise ValueError("bins and world must be >= 1")
    per = -(-bins // world)
    return [(min(bins, g * per), min(bins, (g + 1) * per)) for g in range(world)]


def frame_shards(frames: int, world: int) -> list[tuple[int, int]]:
    """Balanced contiguous frame ranges per rank (sizes differ by at most one)."""
    if frames < 0 or world < 1:
        raise ValueError("frames must be >= 0 and world >= 1")
    base, extra = divmod(frames, world)
    out, lo = [], 0
    for g in range(world):
        hi = lo + base + (1 if g < extra else 0)
        out.append((lo, hi))
        lo = hi
    return out


def local_bin_slab(compute: Callable[[int, int], torch.Tensor], bins: int, rank: int,
                   world: int) -> tuple[tuple[int, int], torch.Tensor | None]:
    """Run ``compute(lo, hi)`` for this rank's slab; None when the slab is empty."""
    lo, hi = bin_slabs(bins, world)[rank]
    return (lo, hi), (compute(lo, hi) if hi > lo else None)


def gather_slabs(slab: torch.Tensor | None, bins: int, height: int, width: int, rank: int,
                 world: int, root: int = 0, group=None) -> torch.Tensor | None:
    """Assemble the (bins, H, W) tensor on ``root`` from every rank's slab.

    Uses batched isend/irecv so the root receives all slabs concurrently
    (NCCL: one grouped call over NVLink).  Returns the full tensor on the
    root, None elsewhere.  Slabs travel as int32 storage (bit-identical to
    uint32); the result is a uint32 view.
    """
    import torch.distributed as dist

    slabs = bin_slabs(bins, world)
    # gloo cannot move CUDA tensors: stage through host memory (tests / 1-GPU runs)
    staged = dist.get_backend(group) != "nccl" and slab is not None and slab.is_cuda
    if staged:
        slab = slab.cpu()
    if rank == root:
        dev = slab.device if slab is not None else torch.device("cpu")
        full = torch.empty((bins, height, width), dtype=torch.int32, device=dev)
        ops = []
        for g, (lo, hi) in enumerate(slabs):
            if hi <= lo:
                continue
            if g == root:
                full[lo:hi].copy_(slab.view(torch.int32))
            else:
                ops.append(dist.P2POp(dist.irecv, full[lo:hi], g, group=group))
        for req in dist.batch_isend_irecv(ops) if ops else []:
            req.wait()
        return full.view(torch.uint32)
    lo, hi = slabs[rank]
    if hi > lo:
        send = slab.view(torch.int32).contiguous()
        for req in dist.batch_isend_irecv([dist.P2POp(dist.isend, send, root, group=group)]):
            req.wait()
    return None
