"""Time prepare (k2_colcounts + k2_colprefix) and k2_scan separately for
workload x env-setting combos.  usage: sweep2.py 'hd64:IH_NSEG=1,2,4,8' 'hd1:IH_TARGET_WARPS=2368,4736,9472' ..."""
import json, os, sys
os.environ["SWEEP_ONE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import numpy as np, torch
import sweep
from paper_1711_01919_b200 import device

def timed(name, reps=5):
    W, H, B, F, br = sweep.WL[name]
    frames = torch.from_numpy(np.stack([sweep.synth(W, H, k) for k in range(min(F, 8))])).cuda()
    if F > 8: frames = frames.repeat((F + 7) // 8, 1, 1)[:F].contiguous()
    lut = ((np.arange(256) * B) // 256).astype(np.uint8)
    nb = B if br is None else br[1] - br[0]
    out = device.empty_output(F, nb, H, W, "cuda")
    ev = [torch.cuda.Event(True) for _ in range(3 * reps)]
    for _ in range(3):
        device.prepare(frames, lut, B, bin_range=br); device.scan(frames, lut, B, out, bin_range=br)
    torch.cuda.synchronize()
    for i in range(reps):
        ev[3*i].record(); device.prepare(frames, lut, B, bin_range=br)
        ev[3*i+1].record(); device.scan(frames, lut, B, out, bin_range=br); ev[3*i+2].record()
    torch.cuda.synchronize()
    prep = sum(ev[3*i].elapsed_time(ev[3*i+1]) for i in range(reps)) / reps
    scan = sum(ev[3*i+1].elapsed_time(ev[3*i+2]) for i in range(reps)) / reps
    alg = F * (H * W + 256 + 4 * nb * H * W)
    tot = ev[0].elapsed_time(ev[-1]) / reps
    return prep, scan, tot, alg / tot / 1e6 / sweep.PEAK, alg / scan / 1e6 / sweep.PEAK

for spec in sys.argv[1:]:
    name, _, envs = spec.partition(":")
    combos = [{}]
    for part in filter(None, envs.split(";")):
        k, v = part.split("=")
        combos = [dict(c, **{k: x}) for c in combos for x in v.split(",")]
    for c in combos:
        for k in ("IH_NSEG", "IH_TARGET_WARPS", "IH_ROWS_PER_BATCH", "IH_MIN_SEG_ROWS", "IH_NO_TMA", "IH_CARRY_LOOKBACK", "IH_TABLE_SUM_MAX", "IH_NO_COLTILE", "IH_TAIL_PCT", "IH_TAIL_DIV"):
            os.environ.pop(k, None)
        os.environ.update(c)
        prep, scan, tot, frac, sfrac = timed(name)
        import subprocess
        clk = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,clocks_throttle_reasons.active,temperature.gpu,power.draw",
                              "--format=csv,noheader"], capture_output=True, text=True).stdout.strip()
        print(json.dumps({"wl": name, **c, "clk": clk, "prep_ms": round(prep, 4), "scan_ms": round(scan, 4),
                          "total_ms": round(tot, 4), "frac_total": round(frac, 3), "frac_scan": round(sfrac, 3)}), flush=True)
