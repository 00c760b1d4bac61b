"""Do two k2_scan launches on two streams overlap?  Prepare two workspaces,
then time N pairs of scans (A on stream 1, B on stream 2, different outputs)
against the same scans back to back on one stream.  usage: WORKLOAD"""
import json, os, sys
os.environ["SWEEP_ONE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import sweep
from paper_1711_01919_b200 import device

W, H, B, F, br = sweep.WL[sys.argv[1]]
frames = torch.from_numpy(np.stack([sweep.synth(W, H, k) for k in range(min(F, 8))])).cuda()
if F > 8: frames = frames.repeat((F + 7) // 8, 1, 1)[:F].contiguous()
lut = ((np.arange(256) * B) // 256).astype(np.uint8)
nb = B if br is None else br[1] - br[0]
outs = [device.empty_output(F, nb, H, W, "cuda") for _ in range(2)]
nws = device.workspace_bytes(F, H, W, nb)
wss = [torch.empty(max(nws, 16), dtype=torch.uint8, device="cuda") for _ in range(2)]
for k in range(2):
    device.prepare(frames, lut, B, bin_range=br, workspace=wss[k])
torch.cuda.synchronize()
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def run(pairs, two):
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    torch.cuda.synchronize()
    e0.record()
    s1.wait_stream(torch.cuda.current_stream()); s2.wait_stream(torch.cuda.current_stream())
    for i in range(pairs):
        for k in range(2):
            s = (s1 if k == 0 else s2) if two else s1
            device.scan(frames, lut, B, outs[k], bin_range=br, stream=s, workspace=wss[k])
    torch.cuda.current_stream().wait_stream(s1); torch.cuda.current_stream().wait_stream(s2)
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / (2 * pairs)
run(2, False); run(2, True)
one, two = run(10, False), run(10, True)
print(json.dumps({"wl": sys.argv[1], "ms_per_scan_one_stream": round(one, 4), "ms_per_scan_two_streams": round(two, 4),
                  "plan": device.plan(F, H, W, nb)["segments"]}))
