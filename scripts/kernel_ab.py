"""Graph-timed single pass (auto) vs the cross-weave kernels (K1 + K1b) per workload."""
import json, os, sys
os.environ["SWEEP_ONE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import sweep
from paper_1711_01919_b200 import device

for name in sys.argv[1:]:
    W, H, B, F, br = sweep.WL[name]
    frames = device.upload_frames(np.stack([sweep.synth(W, H, k) for k in range(F)]))
    lut = ((np.arange(256) * B) // 256).astype(np.uint8)
    nb = B if br is None else br[1] - br[0]
    out = device.empty_output(F, nb, H, W, "cuda")
    res = {"wl": name}
    for kernel in ("auto", "crossweave"):
        for _ in range(3): device.integral_histogram(frames, lut, B, bin_range=br, out=out, kernel=kernel)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph(); s = torch.cuda.Stream()
        with torch.cuda.graph(g, stream=s):
            device.integral_histogram(frames, lut, B, bin_range=br, out=out, kernel=kernel)
        g.replay(); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        for _ in range(10): g.replay()
        e1.record(); torch.cuda.synchronize()
        res[kernel + "_ms"] = round(e0.elapsed_time(e1) / 10, 4)
    print(json.dumps(res), flush=True)
