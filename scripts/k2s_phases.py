"""Phase timeline of the K2s one-launch kernel (ih_debug_trace): per CTA the
times (us after the first CTA start) at which its rows landed, its aggregate
was published, its predecessors' flags were seen, its carries were done, and
it ended.  usage: k2s_phases.py WORKLOAD"""
import json, os, sys
os.environ["SWEEP_ONE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import sweep
from paper_1711_01919_b200 import device, _native

W, H, B, F, br = sweep.WL[sys.argv[1]]
frames = torch.from_numpy(np.stack([sweep.synth(W, H, k) for k in range(F)])).cuda()
lut = ((np.arange(256) * B) // 256).astype(np.uint8)
out = device.empty_output(F, B, H, W, "cuda")
for _ in range(3):
    device.integral_histogram(frames, lut, B, out=out)
p = device.plan(F, H, W, B)
n = F * p["ctas_per_segment"] * p["segments"]
buf = torch.zeros(8 * n, dtype=torch.int64, device="cuda")
torch.cuda.synchronize()
_native.lib().ih_debug_trace(buf.data_ptr(), 2 * n)
device.integral_histogram(frames, lut, B, out=out)
torch.cuda.synchronize()
_native.lib().ih_debug_trace(None, 0)
tr = buf.view(-1, 4).cpu().numpy().astype(np.float64)
main, ph = tr[:n], tr[n:]
t0 = main[:, 0].min()
cols = {"start": main[:, 0], "rows_landed": ph[:, 0], "published": ph[:, 1], "flags_seen": ph[:, 2],
        "carries_done": main[:, 1], "end": main[:, 2]}
res = {"wl": sys.argv[1], "ctas": n, "plan": p}
for k, v in cols.items():
    v = v[v > 0]
    if len(v):
        res[k + "_us_p10_p50_p90"] = [round(float(np.percentile((v - t0) / 1e3, q)), 2) for q in (10, 50, 90)]
print(json.dumps(res))
