"""Measurement of the widened rows f2 (compute_streamed) and f3 (save_ihst):
delivered bytes per second against this box's plain pinned D2H copy, which
bounds both (the tensor leaves the GPU over PCIe).  One JSON line per case.

  f2: compute_streamed of an 8192x8192 image, 256 bins (the 68.7 GB cfg4
      tensor), through plans of several host budgets, into a sink that only
      counts bytes (the reference's TensorSink protocol; the array handed to
      the sink is the page-locked staging buffer).
  f3: save_ihst of a device-resident tensor (HD x 32, and one 32-bin slab of
      cfg4) to a file under /tmp, then the file removed.
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1711_01919_b200 as ih  # noqa: E402
from paper_1711_01919_b200 import device, formats  # noqa: E402


def synth(w, h, seed):
    rng = np.random.default_rng(np.random.SeedSequence([seed, w, h]))
    return rng.integers(0, 256, size=(h, w), dtype=np.uint8)


def d2h_gbs(nbytes=1 << 30):
    src = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    dst = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    dst.copy_(src)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(3):
        dst.copy_(src)
    torch.cuda.synchronize()
    return 3 * nbytes / (time.perf_counter() - t0) / 1e9


class CountingSink:
    """TensorSink that touches nothing but counts the bytes it is handed."""

    def __init__(self):
        self.bytes = 0
        self.pieces = 0

    def write(self, bin_start, bin_stop, row_start, row_stop, data):
        self.bytes += data.nbytes
        self.pieces += 1


def main():
    peak = d2h_gbs()
    print(json.dumps({"case": "pinned_d2h_copy", "gbs": round(peak, 1)}), flush=True)
    W = H = 8192
    img = ih.GrayImage(synth(W, H, 0))
    spec = ih.BinSpec.uniform(256)
    for budget_gb in (2, 5, 10):
        plan = ih.plan_tiles(W, H, 256, budget_gb << 30)
        for call in ("first", "repeat"):  # the first call also page-locks its staging buffers
            sink = CountingSink()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            summary = ih.compute_streamed(img, spec, plan, sink)
            torch.cuda.synchronize()
            dt = time.perf_counter() - t0
            assert sink.bytes == 4 * 256 * W * H
            print(json.dumps({"case": "f2_compute_streamed", "call": call, "tensor": "8192x8192x256",
                              "budget_gb": budget_gb, "chunks": summary.chunks,
                              "strips": summary.strips, "peak_bytes": summary.peak_bytes,
                              "s": round(dt, 3), "gbs": round(sink.bytes / dt / 1e9, 1),
                              "frac_of_d2h_copy": round(sink.bytes / dt / 1e9 / peak, 3)}), flush=True)
    # the file system's own write rate for the same byte counts (host buffer -> file)
    for nbytes in (265420816, 8589934608):
        buf = np.ones(nbytes, dtype=np.uint8)
        path = "/tmp/ih_bench_raw.bin"
        t0 = time.perf_counter()
        with open(path, "wb") as fh:
            fh.write(memoryview(buf))
            fh.flush()
            os.fsync(fh.fileno())
        dt = time.perf_counter() - t0
        os.remove(path)
        print(json.dumps({"case": "host_file_write", "bytes": nbytes, "s_incl_fsync": round(dt, 3),
                          "gbs": round(nbytes / dt / 1e9, 2)}), flush=True)
        del buf
    for name, (w, h, bins, rng_) in {"hd_x32": (1920, 1080, 32, None),
                                     "8k_slab32": (8192, 8192, 256, (0, 32))}.items():
        d = device.upload_image(synth(w, h, 0))
        t = device.integral_histogram(d, ((np.arange(256) * bins) // 256).astype(np.uint8), bins,
                                      bin_range=rng_)
        hist = ih.IntegralHistogram(device_counts=t)
        path = f"/tmp/ih_bench_{name}.ihst"
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        size = formats.save_ihst(path, hist)
        fd = os.open(path, os.O_RDONLY)
        os.fsync(fd)
        os.close(fd)
        dt = time.perf_counter() - t0
        os.remove(path)
        print(json.dumps({"case": "f3_save_ihst", "tensor": name, "bytes": size,
                          "s_incl_fsync": round(dt, 3), "gbs": round(size / dt / 1e9, 2),
                          "frac_of_d2h_copy": round(size / dt / 1e9 / peak, 3)}), flush=True)
        del t, hist, d


if __name__ == "__main__":
    main()
