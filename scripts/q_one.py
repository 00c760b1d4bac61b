"""One K4 + one K5 call on HD x 32 (for ncu)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1711_01919_b200 import device
rng = np.random.default_rng(np.random.SeedSequence([0, 1920, 1080]))
img = device.upload_image(rng.integers(0, 256, size=(1080, 1920), dtype=np.uint8))
lut = ((np.arange(256) * 32) // 256).astype(np.uint8)
t = device.integral_histogram(img, lut, 32)
tmpl = np.full(32, 1 / 32)
for _ in range(2):
    device.window_counts(t, 64, 64)
    device.likelihood_map(t, tmpl, 64, 64, "bhattacharyya")
torch.cuda.synchronize()
