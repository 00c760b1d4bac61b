"""K3 timing on the 8K x 256 tensor: fresh tensor vs the bench's (F=1) output view,
before/after a stretch of sustained full-bandwidth writes."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1711_01919_b200 import device

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

img = device.upload_image(synth(8192, 8192, 0))
lut = ((np.arange(256) * 256) // 256).astype(np.uint8)
rng = np.random.default_rng(20260823 + 4)
Q = 65536
r = np.sort(rng.integers(0, 8192, (Q, 2)), axis=1); c = np.sort(rng.integers(0, 8192, (Q, 2)), axis=1)
regs = torch.from_numpy(np.stack([r[:, 0], c[:, 0], r[:, 1], c[:, 1]], 1).astype(np.int32)).cuda()
out = device.empty_output(1, 256, 8192, 8192, "cuda")
device.integral_histogram(img.unsqueeze(0), lut, 256, out=out)
res = {"fresh_view_ms": timeit(lambda: device.region_histograms(out[0], regs))}
for _ in range(30):
    device.integral_histogram(img.unsqueeze(0), lut, 256, out=out)
res["after_30_steps_ms"] = timeit(lambda: device.region_histograms(out[0], regs))
torch.cuda.synchronize()
import time; time.sleep(2)
res["after_sleep_ms"] = timeit(lambda: device.region_histograms(out[0], regs))
import subprocess
res["clk"] = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,clocks.mem,power.draw,clocks_throttle_reasons.active", "--format=csv,noheader"], capture_output=True, text=True).stdout.strip()
print(json.dumps(res))
