"""Extended fuzz of the query and scan kernels (K3, K4 every mode, K5 every
variant, K6 scans and transpose) against the oracle / numpy restatements of
the reference (core.py:179-195, likelihood.py:34-77, scan.py:33-103).
usage: fuzz_queries_scans.py N_CASES [FIRST_SEED]; prints one JSON line per
failure and a final {"cases": ..., "failures": ...} line."""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
from oracle import oracle as O
from paper_1711_01919_b200 import device
from paper_1711_01919_b200 import scan as S
from paper_1711_01919_b200.errors import ScanOverflowError

n, first = int(sys.argv[1]), int(sys.argv[2]) if len(sys.argv) > 2 else 7000
K4_MODES, K5_VARIANTS = ("0", "1", "2", "3", "4"), (("0", "2"), ("0", "0"), ("0", "4"), ("1", "0"))
fails, cases = 0, 0


def report(kind, seed, **kw):
    global fails
    fails += 1
    print(json.dumps({"kind": kind, "seed": seed, **kw}), flush=True)


def query_case(seed):
    rng = np.random.default_rng(seed)
    H = int(rng.choice([1, 2, 3, int(rng.integers(1, 300))]))
    W = int(rng.choice([1, 2, 5, int(rng.integers(1, 2100))]))
    bins = int(rng.choice([1, 2, 3, 7, 32, 64, 256]))
    px = rng.integers(0, 256, (H, W), dtype=np.uint8)
    lut = rng.integers(0, bins, 256).astype(np.uint8) if rng.random() < 0.3 else O.np_uniform_table(bins)
    full = O.compute_crossweave(px, lut, bins)
    t = device.integral_histogram(device.upload_image(px), lut, bins)
    if not np.array_equal(t.cpu().numpy(), full):
        report("integral_histogram", seed, H=H, W=W, bins=bins)
        return
    q = int(rng.integers(1, 400))
    r = np.sort(rng.integers(0, H, (q, 2)), axis=1)
    c = np.sort(rng.integers(0, W, (q, 2)), axis=1)
    regs = np.stack([r[:, 0], c[:, 0], r[:, 1], c[:, 1]], 1)
    got = device.region_histograms(t, regs).cpu().numpy()
    if not np.array_equal(got, O.region_histograms(full, regs)):
        report("region_histograms", seed, H=H, W=W, bins=bins, q=q)
    h = int(rng.choice([1, H, int(rng.integers(1, H + 1))]))
    w = int(rng.choice([1, W, int(rng.integers(1, W + 1))]))
    want = O.window_counts(full, h, w)
    for mode in K4_MODES:
        os.environ["IH_K4_MODE"] = mode
        odd = rng.random() < 0.3  # an int64 out view 8 bytes past a 16-byte boundary
        shape = want.shape
        if odd:
            buf = torch.zeros(int(np.prod(shape)) + 1, dtype=torch.int64, device="cuda")
            out = buf[1:].view(shape)
            device.window_counts(t, h, w, out=out)
            g = out.cpu().numpy()
        else:
            g = device.window_counts(t, h, w).cpu().numpy()
        if not np.array_equal(g, want):
            report("window_counts", seed, H=H, W=W, bins=bins, h=h, w=w, mode=mode, odd_out=odd)
    os.environ.pop("IH_K4_MODE", None)
    tmpl = rng.random(bins)
    tmpl /= tmpl.sum()
    for metric in ("intersection", "bhattacharyya"):
        ref = O.np_likelihood_map(full, tmpl, h, w, metric)
        base = None
        for direct, chain in K5_VARIANTS:
            os.environ["IH_K5_DIRECT"], os.environ["IH_K5_CHAIN"] = direct, chain
            g = device.likelihood_map(t, tmpl, h, w, metric).cpu().numpy()
            if np.abs(g - ref).max() >= 1e-12 or (base is not None and not np.array_equal(g, base)):
                report("likelihood_map", seed, H=H, W=W, bins=bins, h=h, w=w, metric=metric,
                       direct=direct, chain=chain)
            base = g if base is None else base
    os.environ.pop("IH_K5_DIRECT", None)
    os.environ.pop("IH_K5_CHAIN", None)


def scan_case(seed):
    rng = np.random.default_rng(seed)
    nlen = int(rng.choice([1, 2, 31, 1024, 4097, int(rng.integers(1, 3_000_000))]))
    hi = int(rng.choice([2, 256, 1 << 16, 1 << 31]))
    a = rng.integers(0, hi, nlen, dtype=np.uint64)
    for fn, excl in ((S.inclusive_scan, False), (S.exclusive_scan, True)):
        cs = np.cumsum(a, dtype=np.uint64)
        ref = np.concatenate([[0], cs[:-1]]).astype(np.uint64) if excl else cs
        overflow = bool(len(ref) and ref.max() > 0xFFFFFFFF)
        try:
            g = fn(a)
            if overflow or not np.array_equal(np.asarray(g, dtype=np.uint64), ref):
                report("scan_1d", seed, n=nlen, hi=hi, exclusive=excl, overflow_expected=overflow)
        except ScanOverflowError:
            if not overflow:
                report("scan_1d_spurious_overflow", seed, n=nlen, hi=hi, exclusive=excl)
    rows, cols = int(rng.integers(1, 600)), int(rng.integers(1, 2100))
    dt = np.uint8 if rng.random() < 0.5 else np.uint32
    plane = rng.integers(0, 256 if dt == np.uint8 else 1 << 32, (rows, cols), dtype=np.uint64).astype(dt)
    for fn, axis in ((S.scan_rows, 1), (S.scan_cols, 0)):
        if not np.array_equal(np.asarray(fn(plane)), np.cumsum(plane, axis=axis, dtype=np.uint32)):
            report("scan_axis", seed, rows=rows, cols=cols, dtype=str(np.dtype(dt)), axis=axis)
    tdt = [np.uint8, np.uint16, np.uint32, np.uint64][int(rng.integers(0, 4))]
    m = rng.integers(0, 200, (rows, cols)).astype(tdt)
    if not np.array_equal(np.asarray(S.transpose(m)), m.T):
        report("transpose", seed, rows=rows, cols=cols, dtype=str(np.dtype(tdt)))


for seed in range(first, first + n):
    cases += 1
    try:
        (query_case if seed % 2 == 0 else scan_case)(seed)
    except Exception as e:  # a raised error is a failure too
        report("exception", seed, error=repr(e)[:300])
print(json.dumps({"cases": cases, "failures": fails}), flush=True)
