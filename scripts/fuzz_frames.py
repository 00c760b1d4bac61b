"""Extended fuzz of frame batches: (F, H, W) views with padded row pitch and
frame stride, bin slabs, explicit LUTs and the full plan-knob generator of
tests/test_fuzz_gpu.py (_case), every frame against the oracle.
usage: fuzz_frames.py N_CASES [FIRST_SEED]"""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np, torch
from oracle import oracle as O
from paper_1711_01919_b200 import device
import test_fuzz_gpu as T

n, first = int(sys.argv[1]), int(sys.argv[2]) if len(sys.argv) > 2 else 80000
fails = 0
for seed in range(first, first + n):
    rng = np.random.default_rng(seed)
    H, W, bins, lo, hi, env, offset = T._case(rng)
    if H * W > 600 * 2100:  # keep F frames of oracle work bounded
        H = min(H, 257)
    F = int(rng.integers(2, 6))
    for k in T.KNOBS:
        os.environ.pop(k, None)
    os.environ.update(env)
    lut = rng.integers(0, bins, 256).astype(np.uint8) if rng.random() < 0.3 else O.np_uniform_table(bins)
    pad_w, pad_h = int(rng.choice([0, 1, 5, 16])), int(rng.choice([0, 1, 2]))
    base = rng.integers(0, 256, (F, H + pad_h, W + pad_w + offset), dtype=np.uint8)
    view = torch.from_numpy(base).cuda()[:, :H, offset:offset + W]
    try:
        got = device.integral_histogram(view, lut, bins, bin_range=(lo, hi)).cpu().numpy()
        bad = [f for f in range(F) if not np.array_equal(
            got[f], O.compute_crossweave(np.ascontiguousarray(base[f, :H, offset:offset + W]), lut, bins)[lo:hi])]
        if bad:
            fails += 1
            print(json.dumps({"seed": seed, "F": F, "H": H, "W": W, "bins": bins, "lo": lo, "hi": hi,
                              "pad": [pad_h, pad_w], "offset": offset, "env": env, "bad_frames": bad}), flush=True)
    except Exception as e:
        fails += 1
        print(json.dumps({"seed": seed, "F": F, "H": H, "W": W, "bins": bins, "env": env,
                          "error": repr(e)[:300]}), flush=True)
for k in T.KNOBS:
    os.environ.pop(k, None)
print(json.dumps({"cases": n, "failures": fails}), flush=True)
