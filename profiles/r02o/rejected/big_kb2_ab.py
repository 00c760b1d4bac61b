"""A/B for wide rows (W in (2048, 4096]): column-tiled quads (default), the
1024-thread kernel with quads (IH_NO_COLTILE=1) and with bin pairs
(IH_NO_COLTILE=1 IH_BIG_KB2=1 IH_KB=2).  Each config runs in its own process
(knobs are read per call); prints graph-timed ms per call, the plan and an
exact device checksum of the output for bit-identity across configs."""
import json, os, subprocess, sys
HERE = os.path.dirname(os.path.abspath(__file__))
if len(sys.argv) > 1 and sys.argv[1] == "--one":
    os.environ["SWEEP_ONE"] = "1"
    sys.path.insert(0, HERE)
    import numpy as np, torch
    import sweep
    from paper_1711_01919_b200 import device
    for name in sys.argv[2:]:
        W, H, B, F, br = sweep.WL[name]
        frames = torch.from_numpy(np.stack([sweep.synth(W, H, k) for k in range(F)])).cuda()
        lut = ((np.arange(256) * B) // 256).astype(np.uint8)
        nb = B if br is None else br[1] - br[0]
        out = device.empty_output(F, nb, H, W, "cuda")
        for _ in range(3): device.integral_histogram(frames, lut, B, bin_range=br, out=out)
        torch.cuda.synchronize()
        s = torch.cuda.Stream(); g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for _ in range(10): device.integral_histogram(frames, lut, B, bin_range=br, out=out)
        g.replay()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        torch.cuda.synchronize(); e0.record()
        for _ in range(3): g.replay()
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 30
        alg = F * (H * W + 256 + 4 * nb * H * W)
        flat = out.view(-1)
        chk = 0
        step = 1 << 26
        for i in range(0, flat.numel(), step):
            x = flat[i:i + step].to(torch.int64)
            wgt = torch.arange(i, i + x.numel(), device=x.device, dtype=torch.int64) % 1000003 + 1
            chk = (chk + int((x * wgt).sum().item())) % (1 << 61)
        print(json.dumps({"wl": name, "env": {k: v for k, v in os.environ.items() if k.startswith("IH_")},
                          "ms": round(ms, 4), "frac": round(alg / ms / 1e6 / sweep.PEAK, 3), "chk": chk,
                          "plan": device.plan(F, H, W, nb)}), flush=True)
    sys.exit(0)

wls = ["4k128", "4k128/2", "4k128/4", "4k128/8"]
configs = [{}, {"IH_NO_COLTILE": "1"}, {"IH_NO_COLTILE": "1", "IH_BIG_KB2": "1", "IH_KB": "2"}]
for n in (74, 148):
    configs.append({"IH_NO_COLTILE": "1", "IH_BIG_KB2": "1", "IH_KB": "2", "IH_NSEG": str(n)})
for cfg in configs:
    env = {k: v for k, v in os.environ.items() if not k.startswith("IH_")}
    env.update(cfg)
    r = subprocess.run([sys.executable, __file__, "--one", *wls], env=env, capture_output=True, text=True)
    sys.stdout.write(r.stdout); sys.stderr.write(r.stderr[-2000:])
    sys.stdout.flush()
