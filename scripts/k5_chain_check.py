"""K5 chain variants vs the default table kernel: bit-identical maps and timing."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1711_01919_b200 import device

def synth(w, h, s):
    return np.random.default_rng(np.random.SeedSequence([s, w, h])).integers(0, 256, (h, w), dtype=np.uint8)

def timeit(fn, reps=20):
    for _ in range(3): fn()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    torch.cuda.synchronize(); e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps

rng = np.random.default_rng(3)
ok = True
for (W, H, B) in [(1920, 1080, 32), (333, 97, 7), (129, 65, 3)]:
    lut = ((np.arange(256) * B) // 256).astype(np.uint8)
    t = device.integral_histogram(device.upload_image(synth(W, H, 0)), lut, B)
    tm = rng.random(B); tm /= tm.sum()
    for (h, w) in [(64, 64), (8, 8), (1, 1), (H, W), (13, 70)]:
        if h > H or w > W: continue
        for metric in ("bhattacharyya", "intersection"):
            os.environ.pop("IH_K5_CHAIN", None)
            ref = device.likelihood_map(t, tm, h, w, metric).cpu().numpy()
            for kc, pp in ((2, 2), (2, 4), (4, 2), (4, 4), (8, 2)):
                os.environ["IH_K5_CHAIN"], os.environ["IH_K5_PAIRS"] = str(kc), str(pp)
                got = device.likelihood_map(t, tm, h, w, metric).cpu().numpy()
                if not np.array_equal(got, ref):
                    ok = False
                    print("MISMATCH", W, H, B, h, w, metric, kc, pp, np.abs(got - ref).max(), flush=True)
            os.environ.pop("IH_K5_PAIRS", None)
print("bit-identical:", ok)
lut = ((np.arange(256) * 32) // 256).astype(np.uint8)
t = device.integral_histogram(device.upload_image(synth(1920, 1080, 0)), lut, 32)
tm = rng.random(32); tm /= tm.sum()
for (h, w) in [(64, 64), (8, 8)]:
    res = {}
    for kc, pp in ((0, 2), (2, 2), (2, 4), (4, 2), (4, 4), (8, 2)):
        os.environ["IH_K5_CHAIN"], os.environ["IH_K5_PAIRS"] = str(kc), str(pp)
        res[f"K{kc}P{pp}"] = round(timeit(lambda: device.likelihood_map(t, tm, h, w, "bhattacharyya")), 4)
    print(json.dumps({"window": f"{h}x{w}", "ms": res}))
