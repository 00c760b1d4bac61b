"""Pure device time of one integral_histogram call via CUDA-graph replay
(removes host/launch latency from small problems)."""
import json, os, sys
os.environ["SWEEP_ONE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import numpy as np, torch
import sweep
from paper_1711_01919_b200 import device

for name in sys.argv[1:]:
    W, H, B, F, br = sweep.WL[name]
    frames = torch.from_numpy(np.stack([sweep.synth(W, H, k) for k in range(min(F, 8))])).cuda()
    if F > 8: frames = frames.repeat((F + 7) // 8, 1, 1)[:F].contiguous()
    lut = ((np.arange(256) * B) // 256).astype(np.uint8)
    nb = B if br is None else br[1] - br[0]
    out = device.empty_output(F, nb, H, W, "cuda")
    for _ in range(3): device.integral_histogram(frames, lut, B, bin_range=br, out=out)
    torch.cuda.synchronize()
    s = torch.cuda.Stream(); g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for _ in range(10): device.integral_histogram(frames, lut, B, bin_range=br, out=out)
    for _ in range(2): g.replay()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    torch.cuda.synchronize(); e0.record()
    for _ in range(5): g.replay()
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 50
    alg = F * (H * W + 256 + 4 * nb * H * W)
    print(json.dumps({"wl": name, "graph_ms_per_call": round(ms, 4), "frac": round(alg / ms / 1e6 / sweep.PEAK, 3),
                      "plan": device.plan(F, H, W, nb)}), flush=True)
