"""Tuning sweep of the K2 plan knobs (env vars read per call) on several workloads."""
import json, os, sys, itertools
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1711_01919_b200 import device

PEAK = 6555.5
def synth(w, h, seed):
    rng = np.random.default_rng(np.random.SeedSequence([seed, w, h]))
    return rng.integers(0, 256, size=(h, w), dtype=np.uint8)

WL = {
  "hd64": (1920, 1080, 32, 64, None),
  "hd1": (1920, 1080, 32, 1, None),
  "4k128": (3840, 2160, 128, 1, None),
  "4k128/8": (3840, 2160, 128, 1, (0, 16)),
  "8k256/8": (8192, 8192, 256, 1, (0, 32)),
  "512": (512, 512, 32, 1, None),
  "hd8": (1920, 1080, 32, 8, None),
  "hd16": (1920, 1080, 32, 16, None),
  "hd32": (1920, 1080, 32, 32, None),
  "4k128/2": (3840, 2160, 128, 1, (0, 64)),
  "4k128/4": (3840, 2160, 128, 1, (0, 32)),
  "8k256": (8192, 8192, 256, 1, None),
  "hd2": (1920, 1080, 32, 2, None),
  "hd4": (1920, 1080, 32, 4, None),
  "4k128/16": (3840, 2160, 128, 1, (0, 8)),
  "8k256/2": (8192, 8192, 256, 1, (0, 128)),
  "8k256/4": (8192, 8192, 256, 1, (0, 64)),
  "512x8": (512, 512, 32, 8, None),
  "hd8w1921": (1921, 1080, 32, 8, None),
  "hd8w1922": (1922, 1080, 32, 8, None),
  "hd8w1924": (1924, 1080, 32, 8, None),
  "hd64w1921": (1921, 1080, 32, 64, None),
  "hd64b1": (1920, 1080, 1, 64, None),
  "hd64b2": (1920, 1080, 2, 64, None),
  "hd64b4": (1920, 1080, 4, 64, None),
  "hd64b8": (1920, 1080, 8, 64, None),
  "hd64b16": (1920, 1080, 16, 64, None),
  "hd64b37": (1920, 1080, 37, 64, None),
  "hd64b64": (1920, 1080, 64, 64, None),
  "vga64": (640, 480, 32, 64, None),
  "svga64": (800, 600, 32, 64, None),
  "xga64": (1024, 768, 32, 64, None),
  "hd720x64": (1280, 720, 32, 64, None),
  "wxga64": (1366, 768, 32, 64, None),
  "hdp64": (1600, 900, 32, 64, None),
  "qhd16": (2560, 1440, 32, 16, None),
  "uhd8": (3840, 2160, 32, 8, None),
  "vga1": (640, 480, 32, 1, None),
  "svga1": (800, 600, 32, 1, None),
  "s384": (384, 384, 32, 1, None),
  "s768": (768, 768, 32, 1, None),
  "512b16": (512, 512, 16, 1, None),
  "512b64": (512, 512, 64, 1, None),
}
def run(name, reps=5, kernel="auto"):
    W, H, B, F, br = WL[name]
    frames = torch.from_numpy(np.stack([synth(W, H, k) for k in range(min(F, 8))])).cuda()
    if F > 8: frames = frames.repeat((F + 7) // 8, 1, 1)[:F].contiguous()
    lut = ((np.arange(256) * B) // 256).astype(np.uint8)
    nb = B if br is None else br[1] - br[0]
    out = device.empty_output(F, nb, H, W, "cuda")
    for _ in range(3): device.integral_histogram(frames, lut, B, bin_range=br, out=out, kernel=kernel)
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    torch.cuda.synchronize(); s.record()
    for _ in range(reps): device.integral_histogram(frames, lut, B, bin_range=br, out=out, kernel=kernel)
    e.record(); torch.cuda.synchronize()
    ms = s.elapsed_time(e) / reps
    alg = F * (H * W + 256 + 4 * nb * H * W)
    return ms, alg / ms / 1e6
def main():
  names = sys.argv[1].split(",") if len(sys.argv) > 1 else list(WL)
  for name in names:
      for kern in ("auto", "crossweave"):
          if kern == "crossweave":
              for k in ("IH_ROWS_PER_BATCH", "IH_TARGET_WARPS"): os.environ.pop(k, None)
              ms, gbs = run(name, kernel=kern)
              print(json.dumps({"wl": name, "kernel": kern, "ms": round(ms, 4), "GBs": round(gbs, 1), "frac": round(gbs / PEAK, 3)}), flush=True)
              continue
          for R, tw in itertools.product((1, 2, 4), (148 * 16, 148 * 32, 148 * 64)):
              os.environ["IH_ROWS_PER_BATCH"] = str(R); os.environ["IH_TARGET_WARPS"] = str(tw)
              ms, gbs = run(name)
              print(json.dumps({"wl": name, "R": R, "tw": tw, "ms": round(ms, 4), "GBs": round(gbs, 1), "frac": round(gbs / PEAK, 3)}), flush=True)


if __name__ == "__main__" and os.environ.get("SWEEP_ONE") is None:
    main()
