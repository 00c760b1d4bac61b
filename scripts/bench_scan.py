"""Device time of the K6 scan-module kernels (csrc/ih_scan.cu) with CUDA
events, device-resident inputs; one JSON line per op.  Algorithmic bytes:
ih_scan_u64 12 B/element (u64 in, u32 out), plane scans 8 B/element (u32 in
and out), transpose 2 x element size."""

import json
import sys

import torch

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__file__)))
from paper_1711_01919_b200 import scan as S  # noqa: E402


def timed(fn, reps=20):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def main():
    n = 1 << 28
    x = torch.randint(0, 8, (n,), dtype=torch.int64, device="cuda")
    plane = torch.randint(0, 2**20, (8192, 8192), dtype=torch.int32, device="cuda").view(torch.uint32)
    out = torch.empty_like(plane)
    # the 1-D scan includes its flag read (one sync per call, like the reference's check)
    for name, fn, nbytes in (
        ("inclusive_scan_u64", lambda: S.inclusive_scan(x), 12 * n),
        ("scan_rows_u32", lambda: S.scan_rows(plane, out=out), 8 * plane.numel()),
        ("scan_cols_u32", lambda: S.scan_cols(plane, out=out), 8 * plane.numel()),
        ("transpose_u32", lambda: S.transpose(plane), 8 * plane.numel()),
    ):
        ms = timed(fn)
        print(json.dumps({"op": name, "ms": round(ms, 4), "gbs": round(nbytes / ms / 1e6, 1)}),
              flush=True)


if __name__ == "__main__":
    main()
