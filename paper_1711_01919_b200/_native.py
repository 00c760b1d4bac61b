"""ctypes binding of the C ABI in include/inthist_b200.h (libinthist_b200.so).

This is the reference-side binding a Python caller of the B200 engine uses
(INTEGRATION.md shows the same stub for the reference package).  The library
is loaded from the package directory; if it is missing or cannot be loaded
the import of any compute function fails loudly -- there is no CPU fallback.
"""

from __future__ import annotations

import ctypes
import os

from .errors import BoundsError, CapacityError, DeviceError, ParameterError, ShapeError

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libinthist_b200.so")

IH_OK, IH_ERR_SHAPE, IH_ERR_CAPACITY, IH_ERR_PARAM, IH_ERR_BOUNDS, IH_ERR_CUDA = range(6)
KERNEL_AUTO, KERNEL_SINGLE_PASS, KERNEL_CROSSWEAVE = 0, 1, 2
KERNELS = {"auto": KERNEL_AUTO, "single_pass": KERNEL_SINGLE_PASS, "crossweave": KERNEL_CROSSWEAVE}

_STATUS_EXC = {
    IH_ERR_SHAPE: ShapeError,
    IH_ERR_CAPACITY: CapacityError,
    IH_ERR_PARAM: ParameterError,
    IH_ERR_BOUNDS: BoundsError,
    IH_ERR_CUDA: DeviceError,
}

# Every symbol include/inthist_b200.h declares (checked by tests/test_abi.py).
EXPORTS = (
    "ih_workspace_bytes",
    "ih_integral_histogram",
    "ih_ih_prepare",
    "ih_ih_scan",
    "ih_region_histograms",
    "ih_window_counts",
    "ih_plan_describe",
    "ih_plan_hint",
    "ih_likelihood_map",
    "ih_debug_trace",
    "ih_likelihood_map_ws",
    "ih_likelihood_workspace_bytes",
    "ih_scan_workspace_bytes",
    "ih_scan_u64",
    "ih_scan_axis_u32",
    "ih_transpose",
    "ih_wavefront_workspace_bytes",
    "ih_wavefront",
    "ih_status_string",
    "ih_last_error",
    "ih_abi_version",
    "ih_host_alloc",
    "ih_host_free",
)

_lib = None


def lib() -> ctypes.CDLL:
    """Load (once) and type the C ABI; raise DeviceError if it is missing."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise DeviceError(
            f"B200 extension not built: {LIB_PATH} is missing "
            "(run `python -m paper_1711_01919_b200.build`); there is no CPU fallback"
        )
    try:
        L = ctypes.CDLL(LIB_PATH)
    except OSError as exc:  # pragma: no cover - environment specific
        raise DeviceError(f"cannot load {LIB_PATH}: {exc}") from exc
    P, i64, i32, sz = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_size_t
    L.ih_workspace_bytes.argtypes = [i64, i64, i64, i32, i32]
    L.ih_workspace_bytes.restype = sz
    ih_args = [P, i64, i64, i64, i64, i64, P, i32, i32, i32]
    L.ih_integral_histogram.argtypes = ih_args + [P, P, sz, i32, P]
    L.ih_integral_histogram.restype = ctypes.c_int
    L.ih_ih_prepare.argtypes = ih_args + [P, sz, i32, P]
    L.ih_ih_prepare.restype = ctypes.c_int
    L.ih_ih_scan.argtypes = ih_args + [P, P, sz, i32, P]
    L.ih_ih_scan.restype = ctypes.c_int
    L.ih_region_histograms.argtypes = [P, i32, i64, i64, P, i64, P, P]
    L.ih_region_histograms.restype = ctypes.c_int
    L.ih_window_counts.argtypes = [P, i32, i64, i64, i32, i32, P, P]
    L.ih_window_counts.restype = ctypes.c_int
    L.ih_likelihood_map.argtypes = [P, i32, i64, i64, i32, i32, P, i32, P, P]
    L.ih_likelihood_map.restype = ctypes.c_int
    L.ih_debug_trace.argtypes = [P, ctypes.c_size_t]
    L.ih_debug_trace.restype = None
    L.ih_likelihood_map_ws.argtypes = [P, i32, i64, i64, i32, i32, P, i32, P, P, ctypes.c_size_t, P]
    L.ih_likelihood_map_ws.restype = ctypes.c_int
    L.ih_likelihood_workspace_bytes.argtypes = [i32, i32, i32]
    L.ih_likelihood_workspace_bytes.restype = ctypes.c_size_t
    L.ih_scan_workspace_bytes.argtypes = [i64]
    L.ih_scan_workspace_bytes.restype = sz
    L.ih_scan_u64.argtypes = [P, i64, P, i32, P, P, sz, P]
    L.ih_scan_u64.restype = ctypes.c_int
    L.ih_scan_axis_u32.argtypes = [P, i32, i64, i64, i64, P, P]
    L.ih_scan_axis_u32.restype = ctypes.c_int
    L.ih_transpose.argtypes = [P, i64, i64, i32, P, P]
    L.ih_transpose.restype = ctypes.c_int
    L.ih_plan_describe.argtypes = [i64, i64, i64, i32, i32, i32, P]
    L.ih_plan_describe.restype = ctypes.c_int
    L.ih_plan_hint.argtypes = [i64, i64, i64, i32, i32, i32, i32, i32]
    L.ih_plan_hint.restype = ctypes.c_int
    L.ih_wavefront_workspace_bytes.argtypes = [i64, i64, i32]
    L.ih_wavefront_workspace_bytes.restype = sz
    L.ih_wavefront.argtypes = [P, i64, i64, i64, P, i32, i32, P, P, P, sz, P]
    L.ih_wavefront.restype = ctypes.c_int
    L.ih_status_string.argtypes = [ctypes.c_int]
    L.ih_status_string.restype = ctypes.c_char_p
    L.ih_last_error.argtypes = []
    L.ih_last_error.restype = ctypes.c_char_p
    L.ih_abi_version.argtypes = []
    L.ih_abi_version.restype = i32
    L.ih_host_alloc.argtypes = [sz]
    L.ih_host_alloc.restype = P
    L.ih_host_free.argtypes = [P]
    L.ih_host_free.restype = None
    _lib = L
    return L


def check(status: int) -> None:
    """Map an ih_status onto the reference exception classes."""
    if status == IH_OK:
        return
    L = lib()
    msg = L.ih_last_error().decode(errors="replace")
    exc = _STATUS_EXC.get(status, DeviceError)
    raise exc(f"{L.ih_status_string(status).decode()}: {msg}")
