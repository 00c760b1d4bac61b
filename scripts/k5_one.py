"""One K5 likelihood-map call on HD x 32 bins, 64x64 windows (for ncu)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1711_01919_b200 import device
rng = np.random.default_rng(0)
img = device.upload_image(rng.integers(0, 256, (1080, 1920), dtype=np.uint8))
lut = ((np.arange(256) * 32) // 256).astype(np.uint8)
t = device.integral_histogram(img, lut, 32)
tm = rng.random(32); tm /= tm.sum()
out = torch.empty((1017, 1857), dtype=torch.float64, device="cuda")
for _ in range(3):
    device.likelihood_map(t, tm, 64, 64, "bhattacharyya", out=out)
torch.cuda.synchronize()
