"""Per-call latency of small integral histograms: eager device API vs the
captured GraphedIntegralHistogram (host wall clock per call, device-resident
frames, synchronised each call)."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1711_01919_b200 import device

for (F, H, W, B) in [(1, 512, 512, 32), (1, 1080, 1920, 32), (1, 64, 64, 16)]:
    lut = ((np.arange(256) * B) // 256).astype(np.uint8)
    img = device.upload_frames(np.random.default_rng(0).integers(0, 256, (F, H, W), dtype=np.uint8))
    out = device.empty_output(F, B, H, W, "cuda")
    g = device.GraphedIntegralHistogram(F, H, W, lut, B)
    res = {"shape": [F, H, W, B]}
    for name, fn in (("eager", lambda: device.integral_histogram(img, lut, B, out=out)),
                     ("graphed", lambda: g(img))):
        for _ in range(20): fn()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(200):
            fn()
            torch.cuda.synchronize()
        res[name + "_us"] = round((time.perf_counter() - t0) / 200 * 1e6, 1)
    assert torch.equal(g(img), device.integral_histogram(img, lut, B))
    print(json.dumps(res), flush=True)
