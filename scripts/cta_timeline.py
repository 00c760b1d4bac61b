"""Per-CTA timeline of k2_scan (ih_debug_trace): start / prologue-done / end
times per CTA, summarised: ramp, prologue, CTA lifetime spread, tail.
usage: cta_timeline.py WORKLOAD [NSEG]"""
import json, os, sys
os.environ["SWEEP_ONE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import sweep
from paper_1711_01919_b200 import device, _native

name = sys.argv[1]
if len(sys.argv) > 2:
    os.environ["IH_NSEG"] = sys.argv[2]
W, H, B, F, br = sweep.WL[name]
frames = torch.from_numpy(np.stack([sweep.synth(W, H, k) for k in range(min(F, 8))])).cuda()
if F > 8: frames = frames.repeat((F + 7) // 8, 1, 1)[:F].contiguous()
lut = ((np.arange(256) * B) // 256).astype(np.uint8)
nb = B if br is None else br[1] - br[0]
out = device.empty_output(F, nb, H, W, "cuda")
for _ in range(3):
    device.integral_histogram(frames, lut, B, bin_range=br, out=out)
n = 1 << 16
buf = torch.zeros(4 * n, dtype=torch.int64, device="cuda")
device.prepare(frames, lut, B, bin_range=br)
torch.cuda.synchronize()
_native.lib().ih_debug_trace(buf.data_ptr(), n)
device.scan(frames, lut, B, out, bin_range=br)
torch.cuda.synchronize()
_native.lib().ih_debug_trace(None, 0)
tr = buf.view(-1, 4).cpu().numpy()
if os.environ.get("TRACE_OUT"):
    np.save(os.environ["TRACE_OUT"], tr[: (tr[:, 2] > 0).sum()])
tr = tr[tr[:, 2] > 0].astype(np.float64)
t0 = tr[:, 0].min()
start, ready, end = (tr[:, 0] - t0) / 1e3, (tr[:, 1] - t0) / 1e3, (tr[:, 2] - t0) / 1e3
life = end - start
span = end.max()
p = device.plan(F, H, W, nb)
alg = F * (H * W + 256 + 4 * nb * H * W)
res = {"wl": name, "plan_segments": p["segments"], "ctas": len(tr), "span_us": round(span, 1),
       "frac_of_span": round(alg / (span * 1e-6) / 1e9 / 6555.5, 3),
       "prologue_us_median": round(float(np.median(ready - start)), 2),
       "prologue_us_p95": round(float(np.percentile(ready - start, 95)), 2),
       "life_us_median": round(float(np.median(life)), 1), "life_us_min": round(float(life.min()), 1),
       "life_us_max": round(float(life.max()), 1),
       "last_start_us": round(float(start.max()), 1),
       "end_p10_p50_p90_max": [round(float(np.percentile(end, q)), 1) for q in (10, 50, 90, 100)]}
# busy slots over time (2 CTAs per SM resident): fraction of the span with >= 90% of CTAs slots busy
ts = np.linspace(0, span, 400)
busy = [int(((start <= t) & (end > t)).sum()) for t in ts]
res["busy_ctas_profile"] = [busy[i] for i in range(0, 400, 20)]
print(json.dumps(res), flush=True)
