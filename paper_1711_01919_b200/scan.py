"""Prefix-sum helpers with the reference's semantics (pkg/src/inthist/scan.py:33-103).

Not on any strategy's call path -- the device kernels fuse their scans -- but
part of the public module surface, run by the K6 kernels of the C ABI
(csrc/ih_scan.cu, include/inthist_b200.h ``ih_scan_*`` / ``ih_transpose``):

* ``inclusive_scan`` / ``exclusive_scan`` / ``blocked_scan`` -- 1-D scans of
  the input as uint64 (numpy's astype, like the reference's ``_to_u64``),
  summed mod 2^64 on the device and returned as uint32; any prefix above
  2^32-1 raises ScanOverflowError (scan.py:27-30).  ``ih_scan_u64`` *is* the
  three-phase blocked organisation (tile totals, exclusive scan of totals,
  per-tile scans plus offsets), so ``blocked_scan`` validates ``block`` and
  returns the same array for every block length, as the reference's does.
* ``scan_rows`` / ``scan_cols`` -- numpy ``cumsum(axis, dtype=uint32)``
  semantics (u32 wrap-around, no overflow check) through ``ih_scan_axis_u32``.
* ``transpose`` -- ``ih_transpose`` (32x32 shared-memory tiles); ``tile`` is
  validated like the reference's cache-blocking parameter.

Host (numpy / list) inputs return numpy arrays like the reference's; CUDA
tensor inputs stay on their device and return CUDA tensors (no host copy).
There is no host fallback: without a CUDA device the calls raise DeviceError.
"""

from __future__ import annotations

import numpy as np

from . import _native
from .errors import ParameterError, ScanOverflowError

DEFAULT_BLOCK = 256
DEFAULT_TRANSPOSE_TILE = 64


def _torch():
    import torch

    return torch


def _is_cuda(x) -> bool:
    torch = _torch()
    return isinstance(x, torch.Tensor) and x.is_cuda


def _stream(dev):
    return _torch().cuda.current_stream(dev).cuda_stream


def _upload(a: np.ndarray, dev):
    """Host array -> a new tensor on ``dev`` (read-only inputs are only read)."""
    import warnings

    with warnings.catch_warnings():
        warnings.simplefilter("ignore", UserWarning)
        return _torch().from_numpy(np.ascontiguousarray(a)).to(dev)


def _scan_1d(seq, exclusive: bool):
    """ih_scan_u64 over the flattened input; numpy uint32 (host input) or a
    CUDA uint32 tensor (device input)."""
    torch = _torch()
    from .device import require_cuda

    if _is_cuda(seq):
        if seq.dtype.is_floating_point or seq.dtype.is_complex:
            raise ParameterError("device scans take integer tensors")
        v = seq.reshape(-1).to(torch.int64).contiguous()  # same bits as numpy's astype(uint64)
        dev, host = v.device, False
    else:
        arr = np.asarray(seq)
        if arr.size == 0:
            return np.zeros(0, dtype=np.uint32)
        dev, host = require_cuda(), True
        v = _upload(arr.astype(np.uint64).reshape(-1).view(np.int64), dev)
    n = v.numel()
    out = torch.empty(n, dtype=torch.uint32, device=dev)
    if n == 0:
        return out
    L = _native.lib()
    nws = int(L.ih_scan_workspace_bytes(n))
    with torch.cuda.device(dev):
        ws = torch.empty(nws // 8 + 1, dtype=torch.int64, device=dev)
        flag = torch.empty(1, dtype=torch.int32, device=dev)
        _native.check(L.ih_scan_u64(v.data_ptr(), n, out.data_ptr(), int(exclusive),
                                    flag.data_ptr(), ws.data_ptr(), nws, _stream(dev)))
        if int(flag.item()):  # synchronises the stream
            raise ScanOverflowError("prefix sum exceeds 32-bit range")
    return out.cpu().numpy() if host else out


def inclusive_scan(seq):
    """out[i] = in[0] + ... + in[i] (reference scan.py:33-36)."""
    return _scan_1d(seq, exclusive=False)


def exclusive_scan(seq):
    """out[0] = 0, out[i] = in[0] + ... + in[i-1] (reference scan.py:39-44)."""
    return _scan_1d(seq, exclusive=True)


def blocked_scan(seq, block: int = DEFAULT_BLOCK):
    """Inclusive scan by blocks (reference scan.py:47-76): per-block scans, an
    exclusive scan of block totals, a uniform add -- the phases of
    ih_scan_u64 itself; equal to inclusive_scan for every block >= 1."""
    if block < 1:
        raise ParameterError(f"block length must be >= 1, got {block}")
    return _scan_1d(seq, exclusive=False)


def _split_axis(shape, axis: int):
    if axis >= len(shape):
        raise np.exceptions.AxisError(axis, len(shape))
    outer = int(np.prod(shape[:axis], dtype=np.int64))
    inner = int(np.prod(shape[axis + 1:], dtype=np.int64))
    return outer, int(shape[axis]), inner


def _plane_scan(plane, out, axis: int):
    """u32 inclusive scan along ``axis`` (numpy cumsum(axis, dtype=uint32))."""
    torch = _torch()
    from .device import require_cuda

    if _is_cuda(plane):
        dev, host = plane.device, False
        src = plane.contiguous()
        if src.dtype not in (torch.uint8, torch.uint32, torch.int32):
            if src.dtype.is_floating_point or src.dtype.is_complex:
                raise ParameterError("device plane scans take integer tensors")
            src = src.to(torch.int64).to(torch.int32)  # low 32 bits, numpy's u32 cast
        shape = tuple(src.shape)
    else:
        a = np.asarray(plane)
        if a.ndim == 0:
            a = a.reshape(1)
        shape = a.shape
        _split_axis(shape, axis)
        a = np.ascontiguousarray(a if a.dtype == np.uint8 else a.astype(np.uint32))
        dev, host = require_cuda(), True
        src = _upload(a.view(np.int32) if a.dtype == np.uint32 else a, dev)
    outer, n, inner = _split_axis(shape, axis)
    if out is not None:
        if not isinstance(out, np.ndarray) and not _is_cuda(out):
            raise ParameterError("out must be a numpy array or a CUDA tensor")
        if tuple(out.shape) != shape:
            raise ParameterError(f"out has shape {tuple(out.shape)}, expected {shape}")
        ok = (np.uint32, np.int32) if host else (torch.uint32, torch.int32)
        if (np.dtype(out.dtype).type if host else out.dtype) not in ok:
            raise ParameterError("out must be a 32-bit integer array")
    res = torch.empty(shape, dtype=torch.uint32, device=dev)
    with torch.cuda.device(dev):
        _native.check(_native.lib().ih_scan_axis_u32(
            src.data_ptr(), src.element_size(), outer, n, inner, res.data_ptr(), _stream(dev)))
    if host:
        r = res.cpu().numpy()
        if out is None:
            return r
        out[...] = r.view(out.dtype)
        return out
    if out is None:
        return res
    out.copy_(res.view(out.dtype))
    return out


def scan_rows(plane, out=None):
    """Inclusive scan of every row (reference scan.py:79-84; no overflow check)."""
    return _plane_scan(plane, out, 1)


def scan_cols(plane, out=None):
    """Inclusive scan of every column (reference scan.py:87-92)."""
    return _plane_scan(plane, out, 0)



def transpose(plane, tile: int = DEFAULT_TRANSPOSE_TILE):
    """Fresh contiguous transpose of a 2-D array (reference scan.py:95-103)."""
    torch = _torch()
    from .device import require_cuda

    if tile < 1:
        raise ParameterError(f"tile must be >= 1, got {tile}")
    if _is_cuda(plane):
        src = plane.contiguous()
        if src.dim() != 2:
            raise ValueError("transpose takes a 2-D array")
        rows, cols = (int(x) for x in src.shape)
        out = torch.empty((cols, rows), dtype=src.dtype, device=src.device)
        with torch.cuda.device(src.device):
            _native.check(_native.lib().ih_transpose(src.data_ptr(), rows, cols,
                                                     src.element_size(), out.data_ptr(),
                                                     _stream(src.device)))
        return out
    a = np.asarray(plane)
    rows, cols = a.shape  # ValueError for non-2-D input, as the reference's unpacking
    size = a.dtype.itemsize
    if a.dtype.hasobject or size not in (1, 2, 4, 8, 16):
        raise ParameterError(f"transpose supports 1/2/4/8/16-byte elements, not {a.dtype}")
    view = {1: np.uint8, 2: np.int16, 4: np.int32, 8: np.int64, 16: np.int64}[size]
    dev = require_cuda()
    src = _upload(np.ascontiguousarray(a).view(view), dev)  # 16-byte elements: u64 pairs
    res = torch.empty(src.numel(), dtype=src.dtype, device=dev)
    with torch.cuda.device(dev):
        _native.check(_native.lib().ih_transpose(src.data_ptr(), rows, cols, size,
                                                 res.data_ptr(), _stream(dev)))
    host = res.cpu().numpy()
    return host.view(a.dtype).reshape(cols, rows)
