"""Run one workload a few times (for ncu launch lists): python scripts/one.py hd1 [kernel]"""
import os, sys
os.environ["SWEEP_ONE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import sweep  # noqa: E402
name = sys.argv[1]
kernel = sys.argv[2] if len(sys.argv) > 2 else "auto"
ms, gbs = sweep.run(name, reps=5, kernel=kernel)
print(name, kernel, round(ms, 4), "ms", round(gbs, 1), "GB/s")
