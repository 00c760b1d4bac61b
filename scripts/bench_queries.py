"""Time K3 (batched region histograms) and K4 (window counts) at BASELINE scale."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1711_01919_b200 import device

PEAK = 6555.5
def synth(w, h, seed):
    rng = np.random.default_rng(np.random.SeedSequence([seed, w, h]))
    return rng.integers(0, 256, size=(h, w), dtype=np.uint8)

def timeit(fn, reps=10):
    for _ in range(3): fn()
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    torch.cuda.synchronize(); s.record()
    for _ in range(reps): fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / reps

res = []
# cfg4 queries: 8192^2 x 256 bins (one 8-way shard = 32 bins, and all 256), Q = 65536
for bins, nb in ((256, 32), (256, 256)):
    img = device.upload_image(synth(8192, 8192, 0))
    lut = ((np.arange(256) * bins) // 256).astype(np.uint8)
    t = device.integral_histogram(img, lut, bins, bin_range=(0, nb))
    rng = np.random.default_rng(20260823 + 4)
    Q = 65536
    r = np.sort(rng.integers(0, 8192, (Q, 2)), axis=1); c = np.sort(rng.integers(0, 8192, (Q, 2)), axis=1)
    regs = torch.from_numpy(np.stack([r[:, 0], c[:, 0], r[:, 1], c[:, 1]], 1).astype(np.int32)).cuda()
    ms = timeit(lambda: device.region_histograms(t, regs))
    alg = Q * nb * 24
    res.append({"kernel": "k3_region_histograms", "tensor": f"8192x8192x{nb}", "Q": Q, "ms": round(ms, 4),
                "alg_GBs": round(alg / ms / 1e6, 1), "sector_GBs": round(Q * nb * (4 * 32 + 8) / ms / 1e6, 1),
                "queries_per_s": round(Q / ms * 1e3)})
    del t
# K4: HD x 32, 64x64 windows (reference C6/C8 shape)
img = device.upload_image(synth(1920, 1080, 0))
lut = ((np.arange(256) * 32) // 256).astype(np.uint8)
t = device.integral_histogram(img, lut, 32)
for (h, w) in ((64, 64), (8, 8)):
    ms = timeit(lambda: device.window_counts(t, h, w))
    R, C = 1080 - h + 1, 1920 - w + 1
    alg = 32 * R * C * 8 + 32 * 1080 * 1920 * 4  # int64 out + one read of the tensor
    res.append({"kernel": "k4_window_counts", "tensor": "1920x1080x32", "window": f"{h}x{w}", "ms": round(ms, 4),
                "alg_GBs": round(alg / ms / 1e6, 1), "frac": round(alg / ms / 1e6 / PEAK, 3)})
# K5 fused likelihood map vs the unfused path (K4 counts + float64 torch ops)
tmpl = np.random.default_rng(0).random(32); tmpl /= tmpl.sum()
for (h, w) in ((64, 64), (8, 8)):
    ms = timeit(lambda: device.likelihood_map(t, tmpl, h, w, "bhattacharyya"))
    R, C = 1080 - h + 1, 1920 - w + 1
    tt = torch.from_numpy(tmpl).cuda()[:, None, None]
    def unfused():
        q = device.window_counts(t, h, w).to(torch.float64) / float(h * w)
        return torch.sqrt(tt * q).sum(0).clamp_(0, 1)
    ms_u = timeit(unfused, reps=3)
    alg5 = 32 * 1080 * 1920 * 4 + R * C * 8  # one read of the tensor + the f64 map
    res.append({"kernel": "k5_likelihood_map", "tensor": "1920x1080x32", "window": f"{h}x{w}",
                "ms": round(ms, 4), "unfused_ms": round(ms_u, 4), "speedup": round(ms_u / ms, 1),
                "alg_GBs": round(alg5 / ms / 1e6, 1), "frac": round(alg5 / ms / 1e6 / PEAK, 3),
                "placements_per_s": round(R * C / ms * 1e3)})
tag = {k: os.environ[k] for k in ("IH_K4_MODE", "IH_K5_DIRECT") if k in os.environ}
for r_ in res: print(json.dumps({**r_, **tag}), flush=True)
