"""Autotuner view of the < 4-bin shapes (HD x 64, B = 1 / 2 / 4): every
candidate segment count, tail / skew splits and the other bins-per-CTA
grouping, CUDA-graph timed whole calls; one JSON line per shape."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1711_01919_b200 import device  # noqa: E402

for b in [int(x) for x in (sys.argv[1:] or ["1", "2", "4"])]:
    heur = device.plan(64, 1080, 1920, b)
    r = device.autotune(64, 1080, 1920, b, candidates=sorted(set(device.segment_candidates(64, 1080, 1920, b)) | {3, 5, 7, 9, 12, 16, 20, 24, 28}))
    alg = 64 * (1080 * 1920 + 256 + 4 * b * 1080 * 1920)
    best = min(r["ms"].values())
    print(json.dumps({"bins": b, "kb_env": os.environ.get("IH_KB"), "heuristic": [heur["segments"], heur["bins_per_cta"]],
                      "heuristic_ms": r["ms"].get(str(heur["segments"])), "best": r["segments"], "best_ms": best,
                      "best_frac": round(alg / best / 1e6 / 6550, 3), "ms": r["ms"]}), flush=True)
