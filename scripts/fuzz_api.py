"""Extended fuzz of the drop-in API (the reference's public names, pkg/src/
inthist/__init__.py:39-75): every strategy and worker count, `devices=` bin
and frame sharding (one GPU listed several times), compute_frames with bin
slabs, the wavefront trace's dependency order, compute_streamed over random
budgets, IHST round trips through bytes and files, host-resident region
queries, likelihood maps and best_match -- against the oracle.
usage: fuzz_api.py N_CASES [FIRST_SEED]"""
import json, os, sys, tempfile
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
from oracle import oracle as O
import paper_1711_01919_b200 as ih
from paper_1711_01919_b200 import formats

n, first = int(sys.argv[1]), int(sys.argv[2]) if len(sys.argv) > 2 else 50000
fails = 0


def report(kind, seed, **kw):
    global fails
    fails += 1
    print(json.dumps({"kind": kind, "seed": seed, **kw}), flush=True)


def case(seed):
    rng = np.random.default_rng(seed)
    H = int(rng.choice([1, 2, int(rng.integers(1, 200))]))
    W = int(rng.choice([1, 3, int(rng.integers(1, 1200))]))
    bins = int(rng.choice([1, 2, 5, 16, 32, 100, 256]))
    px = rng.integers(0, 256, (H, W), dtype=np.uint8)
    if rng.random() < 0.3:
        spec = ih.BinSpec.explicit(rng.integers(0, bins, 256))
        bins = spec.bins
    else:
        spec = ih.BinSpec.uniform(bins)
    want = O.compute_crossweave(px, np.asarray(spec.table), bins)
    img = ih.GrayImage(px)
    workers = int(rng.choice([0, 1, 3, 16]))
    for strat in (ih.SEQUENTIAL, ih.CROSSWEAVE, ih.SCAN_TRANSPOSE_SCAN,
                  ih.wavefront(int(rng.integers(1, 80)))):
        got = ih.compute(img, spec, strat, workers=workers).counts
        if not np.array_equal(got, want):
            report("compute", seed, H=H, W=W, bins=bins, strategy=strat.name)
    ndev = int(rng.integers(1, 5))
    got = ih.compute(img, spec, ih.SEQUENTIAL, devices=[0] * ndev).counts
    if not np.array_equal(got, want):
        report("compute_devices", seed, H=H, W=W, bins=bins, ndev=ndev)
    # frames and bin slabs, optionally over a device list
    F = int(rng.integers(1, 5))
    frames = np.stack([px] + [rng.integers(0, 256, (H, W), dtype=np.uint8) for _ in range(F - 1)])
    lo = int(rng.integers(0, bins))
    hi = int(rng.integers(lo + 1, bins + 1))
    shard = str(rng.choice(["frames", "bins"]))
    devs = [0] * int(rng.integers(1, 4)) if rng.random() < 0.5 else None
    if devs is not None:  # bin_range and devices= are exclusive (compute_frames)
        lo, hi = 0, bins
    t = ih.compute_frames(frames, spec, bin_range=None if devs else (lo, hi), devices=devs,
                          shard=shard)
    g = t.cpu().numpy() if isinstance(t, torch.Tensor) else np.asarray(t)
    for f in range(F):
        wf = want if f == 0 else O.compute_crossweave(frames[f], np.asarray(spec.table), bins)
        if not np.array_equal(g[f], wf[lo:hi]):
            report("compute_frames", seed, H=H, W=W, bins=bins, F=F, lo=lo, hi=hi, shard=shard,
                   devices=None if devs is None else len(devs))
            break
    # wavefront with a recorded trace: dependency order and the tensor
    tile = int(rng.integers(1, 70))
    trace = []
    got = ih.compute_wavefront(img, spec, tile, workers=workers, trace=trace).counts
    if not np.array_equal(got, want):
        report("wavefront_tensor", seed, H=H, W=W, bins=bins, tile=tile)
    ni, nj = -(-H // tile), -(-W // tile)
    started = sorted(e[1:] for e in trace if e[0] == "start")
    ok = started == sorted((i, j) for i in range(ni) for j in range(nj))
    done = set()
    for ev, i, j in trace:
        if ev == "start":
            ok &= (i == 0 or (i - 1, j) in done) and (j == 0 or (i, j - 1) in done)
        else:
            done.add((i, j))
    if not ok:
        report("wavefront_trace", seed, H=H, W=W, tile=tile)
    # streamed delivery over a random budget
    need1 = ih.streamed.working_set_bytes(W, 1, 1) if hasattr(ih, "streamed") else 0
    budget = int(rng.integers(max(need1, 64), max(need1, 64) + 8 * bins * H * W + 1024))
    try:
        plan = ih.plan_tiles(W, H, bins, budget)
        sink = ih.ArraySink(W, H, bins)
        summ = ih.compute_streamed(img, spec, plan, sink)
        if not np.array_equal(sink.counts, want) or summ.chunks < 1 or summ.strips < 1:
            report("compute_streamed", seed, H=H, W=W, bins=bins, budget=budget)
    except ih.CapacityError:
        pass  # a budget below one 1-bin, 1-row strip (the reference raises too)
    # IHST round trips, host-resident queries
    res = ih.compute(img, spec, ih.SEQUENTIAL)
    back = formats.deserialize_ih(formats.serialize_ih(res))
    with tempfile.TemporaryDirectory() as d:
        path = os.path.join(d, "t.ihst")
        formats.save_ihst(path, res, group_bytes=int(rng.choice([4096, 1 << 20, 1 << 28])))
        with open(path, "rb") as fh:
            back2 = formats.deserialize_ih(fh.read())
    if not (np.array_equal(back.counts, want) and np.array_equal(back2.counts, want)):
        report("ihst_roundtrip", seed, H=H, W=W, bins=bins)
    for _ in range(5):
        r0, r1 = sorted(rng.integers(0, H, 2).tolist())
        c0, c1 = sorted(rng.integers(0, W, 2).tolist())
        reg = ih.Region(r0, c0, r1, c1)
        exp = O.region_histograms(want, [(r0, c0, r1, c1)])[0]
        for src in (res, back2):
            if not np.array_equal(np.asarray(ih.region_histogram(src, reg).counts), exp):
                report("region_histogram", seed, H=H, W=W, bins=bins, region=[r0, c0, r1, c1],
                       host=src is back2)
    h, w = int(rng.integers(1, H + 1)), int(rng.integers(1, W + 1))
    tmpl = rng.random(bins)
    tmpl /= tmpl.sum()
    for metric in ("intersection", "bhattacharyya"):
        lm = ih.likelihood_map(res, tmpl, h, w, metric)
        ref = O.np_likelihood_map(want, tmpl, h, w, metric)
        if lm.values.shape != ref.shape or np.abs(lm.values - ref).max() >= 1e-12:
            report("likelihood_map", seed, H=H, W=W, bins=bins, h=h, w=w, metric=metric)
            continue
        r, c, v = ih.best_match(lm)
        if lm.values[r, c] != lm.values.max() or v != lm.values.max():
            report("best_match", seed, H=H, W=W, h=h, w=w, metric=metric)


for seed in range(first, first + n):
    try:
        case(seed)
    except Exception as e:
        report("exception", seed, error=repr(e)[:300])
print(json.dumps({"cases": n, "failures": fails}), flush=True)
