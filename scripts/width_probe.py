"""Graph-timed calls for 64 frames x 32 bins at widths around 1366 (W % 4 =
0/1/2/3, W % 16 = 0 or not), 768 rows: where W % 4 != 0 loses its time."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1711_01919_b200 import _native, device
_native.LIB_PATH = os.environ.get("IH_LIB_OVERRIDE", _native.LIB_PATH)  # A/B builds
PEAK = 6555.5
H, F, B = 768, 64, 32
lut = ((np.arange(256) * B) // 256).astype(np.uint8)
for W in [int(x) for x in (sys.argv[1:] or [1360, 1364, 1365, 1366, 1367, 1368, 1376])]:
    g0 = torch.Generator(device="cuda").manual_seed(W)
    pitch = (W + 15) // 16 * 16
    buf = torch.randint(0, 256, (F, H, pitch), dtype=torch.uint8, device="cuda", generator=g0)
    frames = buf[:, :, :W]  # 16-byte pitched rows: no restaging copy inside the call
    out = device.empty_output(F, B, H, W, "cuda")
    for _ in range(3): device.integral_histogram(frames, lut, B, out=out)
    torch.cuda.synchronize()
    s = torch.cuda.Stream(); g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for _ in range(5): device.integral_histogram(frames, lut, B, out=out)
    g.replay()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    torch.cuda.synchronize(); e0.record()
    for _ in range(4): g.replay()
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    alg = F * (H * W + 256 + 4 * B * H * W)
    p = device.plan(F, H, W, B)
    print(json.dumps({"lib": os.path.basename(_native.LIB_PATH), "W": W, "W%4": W % 4, "ms": round(ms, 4), "frac": round(alg / ms / 1e6 / PEAK, 3),
                      "segments": p["segments"], "warps": p["warps_per_cta"], "kb": p["bins_per_cta"]}), flush=True)
