"""A few K2s cases checked against the oracle (for compute-sanitizer runs)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from oracle import oracle as O  # noqa: E402
from paper_1711_01919_b200 import device  # noqa: E402

os.environ["IH_SMALL"] = "1"
for (F, h, w, b, n) in [(1, 512, 512, 32, 0), (2, 33, 127, 5, 7), (1, 100, 1000, 64, 0),
                        (1, 64, 2048, 9, 3), (1, 300, 640, 16, 30)]:
    if n:
        os.environ["IH_NSEG"] = str(n)
    else:
        os.environ.pop("IH_NSEG", None)
    fr = np.random.default_rng(F * h + w).integers(0, 256, (F, h, w), dtype=np.uint8)
    lut = O.np_uniform_table(b)
    got = device.integral_histogram(device.upload_frames(fr), lut, b).cpu().numpy()
    for f in range(F):
        assert np.array_equal(got[f], O.compute_crossweave(fr[f], lut, b)), (F, h, w, b, f)
print("k2s sanitizer cases ok")
