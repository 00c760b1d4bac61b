"""Host cost of one eager device.integral_histogram call (512x512x32, device
input, preallocated output): wall time per call over a stream of calls, and
the same call under cProfile to see where the host time goes."""
import cProfile, os, pstats, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1711_01919_b200 import device
img = device.upload_image(np.random.default_rng(0).integers(0, 256, (512, 512), dtype=np.uint8))
lut = ((np.arange(256) * 32) // 256).astype(np.uint8)
out = device.empty_output(1, 32, 512, 512, "cuda")[0]
for _ in range(50): device.integral_histogram(img, lut, 32, out=out)
torch.cuda.synchronize()
n = 2000
t0 = time.perf_counter()
for _ in range(n): device.integral_histogram(img, lut, 32, out=out)
torch.cuda.synchronize()
print(f"eager us/call: {(time.perf_counter() - t0) / n * 1e6:.1f}")
pr = cProfile.Profile(); pr.enable()
for _ in range(500): device.integral_histogram(img, lut, 32, out=out)
pr.disable(); torch.cuda.synchronize()
pstats.Stats(pr).sort_stats("tottime").print_stats(12)
