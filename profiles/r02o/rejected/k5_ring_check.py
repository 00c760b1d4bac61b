"""K5 with TMA-staged corner rows (IH_K5_RING=1, ih_k5ring.cu) vs the chain
kernel (IH_K5_RING=0): bit-identical maps over shapes / windows / metrics,
then timing on HD x 32 (64x64 and 8x8 windows) for a few grid sizes."""
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
ok, n = True, 0
for (W, H, B) in [(1920, 1080, 32), (332, 97, 7), (128, 65, 3), (1024, 600, 16), (516, 300, 1), (2000, 130, 64)]:
    lut = ((np.arange(256) * B) // 256).astype(np.uint8)
    t = device.integral_histogram(device.upload_image(synth(W, H, 0)), lut, B)
    tm = rng.random(B); tm /= tm.sum()
    for (h, w) in [(64, 64), (8, 8), (1, 1), (H, W), (13, 70), (3, 511), (40, 1000), (1, W), (H, 1), (2, 2)]:
        if h > H or w > W: continue
        for metric in ("bhattacharyya", "intersection"):
            os.environ["IH_K5_RING"] = "0"
            ref = device.likelihood_map(t, tm, h, w, metric).cpu().numpy()
            os.environ["IH_K5_RING"] = "1"
            got = device.likelihood_map(t, tm, h, w, metric).cpu().numpy()
            n += 1
            if not np.array_equal(got, ref):
                ok = False
                print("MISMATCH", W, H, B, h, w, metric, np.abs(got - ref).max(), flush=True)
print(json.dumps({"bit_identical": ok, "cases": n}), flush=True)
lut = ((np.arange(256) * 32) // 256).astype(np.uint8)
t = device.integral_histogram(device.upload_image(synth(1920, 1080, 0)), lut, 32)
tm = rng.random(32); tm /= tm.sum()
for (h, w) in [(64, 64), (8, 8), (128, 128)]:
    res = {}
    os.environ["IH_K5_RING"] = "0"
    res["chain"] = round(timeit(lambda: device.likelihood_map(t, tm, h, w, "bhattacharyya")), 4)
    os.environ["IH_K5_RING"] = "1"
    for wv in (1, 2, 4):
        os.environ["IH_K5_RING_WAVES"] = str(wv)
        res[f"ring_w{wv}"] = round(timeit(lambda: device.likelihood_map(t, tm, h, w, "bhattacharyya")), 4)
    os.environ.pop("IH_K5_RING_WAVES", None)
    print(json.dumps({"window": f"{h}x{w}", "ms": res}), flush=True)
