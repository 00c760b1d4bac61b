"""Extended fuzz run (the test suite's case generator, many more seeds):
random shapes, slabs, LUTs, offsets and plan knobs against the oracle.
usage: fuzz_extended.py N_SEEDS [FIRST_SEED]"""
import os, sys, json
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np, torch
from oracle import oracle as O
from paper_1711_01919_b200 import device
import test_fuzz_gpu as T

n, first = int(sys.argv[1]), int(sys.argv[2]) if len(sys.argv) > 2 else 5000
bad, cases = [], 0
for seed in range(first, first + n):
    rng = np.random.default_rng(seed)
    for _ in range(20):
        H, W, bins, lo, hi, env, offset = T._case(rng)
        for k in T.KNOBS:
            os.environ.pop(k, None)
        os.environ.update(env)
        lut = rng.integers(0, bins, 256).astype(np.uint8) if rng.random() < 0.3 else O.np_uniform_table(bins)
        base = rng.integers(0, 256, (H, W + offset), dtype=np.uint8)
        px = np.ascontiguousarray(base[:, offset:])
        view = torch.from_numpy(base).cuda()[:, offset:]
        kernel = "single_pass" if W <= 8192 or "IH_NO_COLTILE" not in env else "auto"
        cases += 1
        try:
            got = device.integral_histogram(view, lut, bins, bin_range=(lo, hi), kernel=kernel).cpu().numpy()
            ok = np.array_equal(got, O.compute_crossweave(px, lut, bins)[lo:hi])
        except Exception as exc:
            ok = False
            env = dict(env, error=repr(exc)[:200])
        if not ok:
            bad.append({"seed": seed, "H": H, "W": W, "bins": bins, "lo": lo, "hi": hi, "env": env, "offset": offset})
            print(json.dumps(bad[-1]), flush=True)
print(json.dumps({"cases": cases, "failures": len(bad)}))
