"""Drop-in API latency: GrayImage -> compute -> .counts (host numpy), HD x 32."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1711_01919_b200 as ih
from oracle import oracle as O

img = ih.GrayImage(O.synth_image(1920, 1080, 0))
spec = ih.BinSpec.uniform(32)
for mode in ("pinned", "pageable"):
    os.environ["IH_NO_PINNED"] = "1" if mode == "pageable" else "0"
    ts = []
    for i in range(8):
        t0 = time.perf_counter()
        res = ih.compute(img, spec, ih.SEQUENTIAL).counts
        ts.append(time.perf_counter() - t0)
        del res
    print(mode, "ms per call (steady):", [round(1e3 * t, 1) for t in ts], flush=True)
t0 = time.perf_counter(); O.compute_crossweave(img.pixels, spec.table, 32); print("cpu port ms", round(1e3 * (time.perf_counter() - t0), 1))
