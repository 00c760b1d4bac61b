"""device.autotune (whole calls, CUDA-graph timed) for a few shapes; prints
the heuristic plan's time, the best candidate and its fraction of HBM."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1711_01919_b200 import device  # noqa: E402

SHAPES = {"hd1": (1, 1080, 1920, 32), "hd2": (2, 1080, 1920, 32), "hd4": (4, 1080, 1920, 32),
          "512": (1, 512, 512, 32), "4k128/8": (1, 2160, 3840, 16), "8k256/8": (1, 8192, 8192, 32),
          "hd64b2": (64, 1080, 1920, 2), "hd64b4": (64, 1080, 1920, 4)}
for name in sys.argv[1:] or list(SHAPES):
    f, h, w, b = SHAPES[name]
    heur = device.plan(f, h, w, b)
    r = device.autotune(f, h, w, b)
    alg = f * (h * w + 256 + 4 * b * h * w)
    best = min(r["ms"].values())
    print(json.dumps({"wl": name, "heuristic": [heur["segments"], heur["bins_per_cta"], heur["carry"]],
                      "heuristic_ms": r["ms"].get(str(heur["segments"])), "best": [r["segments"], r["bins_per_cta"]],
                      "best_ms": best, "best_frac": round(alg / best / 1e6 / 6550, 3),
                      "top": dict(sorted(r["ms"].items(), key=lambda x: x[1])[:6])}), flush=True)
