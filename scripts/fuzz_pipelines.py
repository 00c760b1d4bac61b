"""Fuzz of the host-buffer and graph-replay entry points: pipeline.FramePipeline
(frame pieces and bin sub-slab pieces via a small max_piece_bytes, repeated
runs on one pipeline), compute_frames_host, and GraphedIntegralHistogram
(repeated calls with new host / device inputs) against the oracle.
usage: fuzz_pipelines.py N_CASES [FIRST_SEED]"""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
from oracle import oracle as O
import paper_1711_01919_b200 as ih
from paper_1711_01919_b200 import device, pipeline

n, first = int(sys.argv[1]), int(sys.argv[2]) if len(sys.argv) > 2 else 200000
fails = 0


def report(kind, seed, **kw):
    global fails
    fails += 1
    print(json.dumps({"kind": kind, "seed": seed, **kw}), flush=True)


for seed in range(first, first + n):
    rng = np.random.default_rng(seed)
    try:
        F = int(rng.integers(1, 6))
        H, W = int(rng.integers(1, 200)), int(rng.integers(1, 900))
        bins = int(rng.choice([1, 3, 16, 32, 64]))
        spec = ih.BinSpec.uniform(bins)
        lo = int(rng.integers(0, bins)); hi = int(rng.integers(lo + 1, bins + 1))
        br = None if rng.random() < 0.5 else (lo, hi)
        lo_, hi_ = (0, bins) if br is None else br
        plane = H * W * 4
        mpb = int(rng.choice([plane, 3 * plane, 1 << 30]))  # small: bin sub-slab pieces
        pipe = pipeline.FramePipeline(F, H, W, spec, chunk=int(rng.integers(1, 5)), bin_range=br,
                                      max_piece_bytes=mpb)
        for rep in range(2):
            frames = rng.integers(0, 256, (F, H, W), dtype=np.uint8)
            hf = torch.from_numpy(frames).pin_memory()
            ho = torch.empty((F, hi_ - lo_, H, W), dtype=torch.uint32).pin_memory()
            pipe.run(hf, ho)
            got = ho.numpy()
            for f in range(F):
                want = O.compute_crossweave(frames[f], np.asarray(spec.table), bins)[lo_:hi_]
                if not np.array_equal(got[f], want):
                    report("frame_pipeline", seed, F=F, H=H, W=W, bins=bins, br=br, mpb=mpb, rep=rep, f=f)
                    break
        got = pipeline.compute_frames_host(frames, spec, bin_range=br)
        if not all(np.array_equal(got[f], O.compute_crossweave(frames[f], np.asarray(spec.table), bins)[lo_:hi_])
                   for f in range(F)):
            report("compute_frames_host", seed, F=F, H=H, W=W, bins=bins, br=br)
        g = device.GraphedIntegralHistogram(F, H, W, spec.table, bins, bin_range=br)
        for rep in range(3):
            frames = rng.integers(0, 256, (F, H, W), dtype=np.uint8)
            src = frames if rep % 2 == 0 else torch.from_numpy(frames).cuda()
            out = g(src).cpu().numpy()
            for f in range(F):
                want = O.compute_crossweave(frames[f], np.asarray(spec.table), bins)[lo_:hi_]
                if not np.array_equal(out[f], want):
                    report("graphed", seed, F=F, H=H, W=W, bins=bins, br=br, rep=rep, f=f)
                    break
    except Exception as e:
        report("exception", seed, error=repr(e)[:300])
print(json.dumps({"cases": n, "failures": fails}), flush=True)
