"""Run each non-K2 kernel of the C ABI a few times at a representative size, for
per-kernel ncu captures (scripts/gpu_kernel_profiles.sh):

  k1_rowscan / k1b_colscan  HD x 32, 8 frames, kernel="crossweave"
  k3_region_histograms      8192^2 x 32-bin shard (and all 256 bins with `k3full`), Q = 65,536
  k4_window_counts_pairs    HD x 32, 64x64 windows
  k5_metric_table / k5_likelihood_map_tabp   HD x 32, 64x64 windows
  k6_* scans / transpose    2^28 u64 1-D scan, 8192^2 u32 plane scans and transpose
  k7_wavefront              1920x1080 x 32, 64x64 tiles

    python scripts/kernels_once.py [k1|k3|k3full|k4|k5|k6|k7 ...]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1711_01919_b200 import device  # noqa: E402
from paper_1711_01919_b200 import scan as S  # noqa: E402


def synth(w, h, seed):
    rng = np.random.default_rng(np.random.SeedSequence([seed, w, h]))
    return rng.integers(0, 256, size=(h, w), dtype=np.uint8)


def lut(bins):
    return ((np.arange(256) * bins) // 256).astype(np.uint8)


def regions(H, W, Q=65536):
    rng = np.random.default_rng(20260823 + 4)
    r = np.sort(rng.integers(0, H, (Q, 2)), axis=1)
    c = np.sort(rng.integers(0, W, (Q, 2)), axis=1)
    return torch.from_numpy(np.stack([r[:, 0], c[:, 0], r[:, 1], c[:, 1]], 1).astype(np.int32)).cuda()


def main(which):
    reps = 3
    if "k1" in which:
        frames = torch.from_numpy(np.stack([synth(1920, 1080, s) for s in range(8)])).cuda()
        for _ in range(reps):
            device.integral_histogram(frames, lut(32), 32, kernel="crossweave")
    if "k3" in which or "k3full" in which:
        img = device.upload_image(synth(8192, 8192, 0))
        nb = 256 if "k3full" in which else 32
        t = device.integral_histogram(img, lut(256), 256, bin_range=(0, nb))
        regs = regions(8192, 8192)
        out = torch.empty((regs.shape[0], nb), dtype=torch.uint64, device="cuda")
        for _ in range(reps):
            device.region_histograms(t, regs, out=out)
        del t
    if "k4" in which or "k5" in which:
        t = device.integral_histogram(device.upload_image(synth(1920, 1080, 0)), lut(32), 32)
        tmpl = np.full(32, 1 / 32)
        for _ in range(reps):
            if "k4" in which:
                device.window_counts(t, 64, 64)
            if "k5" in which:
                device.likelihood_map(t, tmpl, 64, 64, "bhattacharyya")
    if "k6" in which:
        x = torch.randint(0, 8, (1 << 28,), dtype=torch.int64, device="cuda")
        plane = torch.randint(0, 2**20, (8192, 8192), dtype=torch.int32,
                              device="cuda").view(torch.uint32)
        out = torch.empty_like(plane)
        for _ in range(reps):
            S.inclusive_scan(x)
            S.scan_rows(plane, out=out)
            S.scan_cols(plane, out=out)
            S.transpose(plane)
    if "k7" in which:
        img = device.upload_image(synth(1920, 1080, 0))
        for _ in range(reps):
            device.wavefront(img, lut(32), 32, 64)
    torch.cuda.synchronize()


if __name__ == "__main__":
    main(set(sys.argv[1:]) or {"k1", "k3", "k4", "k5", "k6", "k7"})
