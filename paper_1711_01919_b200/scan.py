"""Prefix-sum helpers with the reference's semantics (pkg/src/inthist/scan.py:33-103).

Not on any strategy's call path -- the device kernels fuse their scans -- but
part of the public module surface: 1-D inclusive / exclusive / blocked scans
over uint32 with a 2^32-1 overflow guard (ScanOverflowError), per-row and
per-column plane scans and a transpose.  They run on the device through torch
(int64 accumulation); results come back as numpy uint32 like the reference's.
The blocked scan is the three-phase reduce-then-scan skeleton the K2 row-segment
carries use: per-block scans, an exclusive scan of block totals, a uniform add.
"""

from __future__ import annotations

import numpy as np

from .errors import ParameterError, ScanOverflowError

DEFAULT_BLOCK = 256
DEFAULT_TRANSPOSE_TILE = 64
_LIMIT = 0xFFFF_FFFF


def _dev_vec(seq):
    import torch

    from .device import require_cuda

    arr = np.asarray(seq)
    return torch.as_tensor(arr.astype(np.int64).reshape(-1), device=require_cuda())


def _as_u32(t) -> np.ndarray:
    if t.numel() and int(t.max()) > _LIMIT:
        raise ScanOverflowError("prefix sum exceeds 32-bit range")
    return t.cpu().numpy().astype(np.uint32)


def inclusive_scan(seq) -> np.ndarray:
    """out[i] = in[0] + ... + in[i]."""
    v = _dev_vec(seq)
    return _as_u32(v.cumsum(0))


def exclusive_scan(seq) -> np.ndarray:
    """out[0] = 0, out[i] = in[0] + ... + in[i-1]."""
    v = _dev_vec(seq)
    return _as_u32(v.cumsum(0) - v)


def blocked_scan(seq, block: int = DEFAULT_BLOCK) -> np.ndarray:
    """Inclusive scan by blocks: local scans, exclusive scan of the block
    totals, uniform add -- equal to inclusive_scan for every block >= 1."""
    import torch

    if block < 1:
        raise ParameterError(f"block length must be >= 1, got {block}")
    v = _dev_vec(seq)
    n = v.numel()
    if n == 0:
        return np.zeros(0, dtype=np.uint32)
    nblk = -(-n // block)
    padded = torch.zeros(nblk * block, dtype=torch.int64, device=v.device)
    padded[:n] = v
    local = padded.view(nblk, block).cumsum(1)            # phase 1: per-block scans
    offsets = local[:, -1].cumsum(0) - local[:, -1]        # phase 2: exclusive block totals
    return _as_u32((local + offsets[:, None]).reshape(-1)[:n])  # phase 3: uniform add


def _plane_scan(plane, out, dim):
    import torch

    from .device import require_cuda

    a = np.asarray(plane)
    t = torch.as_tensor(a.astype(np.int64), device=require_cuda()).cumsum(dim)
    res = (t & _LIMIT).cpu().numpy().astype(np.uint32)  # u32 wrap like numpy's u32 cumsum
    if out is None:
        return res
    out[...] = res
    return out


def scan_rows(plane, out=None) -> np.ndarray:
    """Inclusive scan of every row (the reference skips the overflow check here)."""
    return _plane_scan(plane, out, 1)


def scan_cols(plane, out=None) -> np.ndarray:
    """Inclusive scan of every column."""
    return _plane_scan(plane, out, 0)


def transpose(plane, tile: int = DEFAULT_TRANSPOSE_TILE) -> np.ndarray:
    """Fresh contiguous transpose; ``tile`` is validated like the reference's
    cache-blocking parameter (the device transpose needs no blocking hint)."""
    import torch

    from .device import require_cuda

    if tile < 1:
        raise ParameterError(f"tile must be >= 1, got {tile}")
    a = np.ascontiguousarray(plane)
    t = torch.as_tensor(a.view(np.int32) if a.dtype == np.uint32 else a, device=require_cuda())
    res = t.t().contiguous().cpu().numpy()
    return res.view(np.uint32) if a.dtype == np.uint32 else res
