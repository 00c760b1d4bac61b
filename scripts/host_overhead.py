import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1711_01919_b200 import device, _native
img = torch.zeros((1, 64, 64), dtype=torch.uint8, device="cuda")
lut = np.zeros(256, np.uint8)
out = device.empty_output(1, 4, 64, 64, "cuda")
for name, fn in [("integral_histogram", lambda: device.integral_histogram(img, lut, 4, out=out)),
                 ("plan", lambda: device.plan(1, 1080, 1920, 32))]:
    for _ in range(50): fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(2000): fn()
    dt = (time.perf_counter() - t0) / 2000
    torch.cuda.synchronize()
    print(name, round(dt * 1e6, 1), "us per call (host)", flush=True)
L = _native.lib()
import ctypes
info = (ctypes.c_int64 * 16)()  # ih_plan_describe fills 16 entries (ABI 1.7)
t0 = time.perf_counter()
for _ in range(20000): L.ih_plan_describe(1, 1080, 1920, 32, 0, 1, info)
print("ih_plan_describe raw", round((time.perf_counter() - t0) / 20000 * 1e6, 2), "us")
