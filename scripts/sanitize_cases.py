"""Small parity cases for compute-sanitizer: every K2 carry mode / input path,
column tiles (k2_rowleft), both count-table kernels,
K1/K1b, K3, K4, K5, and the K6 scan-module kernels -- each checked against
the oracle / numpy."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from oracle import oracle as O
from paper_1711_01919_b200 import device

rng = np.random.default_rng(7)
cases = [(1, 1, 3), (7, 131, 5), (61, 257, 16), (100, 300, 64), (33, 2049, 7), (40, 4100, 9), (9, 8192, 4),
         (21, 10001, 256), (70, 3840, 128), (50, 1921, 1), (45, 1922, 2), (30, 701, 2)]
envs = [{}, {"IH_NSEG": "3"}, {"IH_NSEG": "5", "IH_TABLE_SUM_MAX": "1"},
        {"IH_NSEG": "4", "IH_CARRY_LOOKBACK": "1"}, {"IH_NO_TMA": "1", "IH_NSEG": "2"},
        {"IH_ROWS_PER_BATCH": "1", "IH_NSEG": "3"}, {"IH_NSEG": "6", "IH_COLCOUNTS_SLAB": "1"},
        {"IH_NSEG": "3", "IH_NO_COLTILE": "1"}, {"IH_NSEG": "4", "IH_TAIL_PCT": "30"},
        {"IH_NSEG": "3", "IH_CARRY_CLUSTER": "1"}, {"IH_NSEG": "2", "IH_STAGED_STORES": "1"},
        {"IH_SMALL": "1"}, {"IH_SMALL": "1", "IH_NSEG": "7"},
        {"IH_NSEG": "5", "IH_SKEW_X100": "130"}, {"IH_NSEG": "4", "IH_COLCOUNTS_G1": "0"},
        {"IH_NSEG": "9", "IH_COUNT_CW": "2"}, {"IH_NSEG": "7", "IH_KB": "2"}]
bad = 0
for env in envs:
    for k in ("IH_NSEG", "IH_TABLE_SUM_MAX", "IH_CARRY_LOOKBACK", "IH_NO_TMA", "IH_ROWS_PER_BATCH",
              "IH_COLCOUNTS_SLAB", "IH_NO_COLTILE", "IH_TAIL_PCT", "IH_CARRY_CLUSTER",
              "IH_STAGED_STORES", "IH_SMALL", "IH_SKEW_X100", "IH_COLCOUNTS_G1", "IH_COUNT_CW",
              "IH_KB"):
        os.environ.pop(k, None)
    os.environ.update(env)
    for (h, w, b) in cases:
        px = rng.integers(0, 256, (h, w), dtype=np.uint8)
        lut = O.np_uniform_table(b)
        want = O.compute_crossweave(px, lut, b)
        for kernel in ("auto", "crossweave"):
            if kernel == "crossweave" and w > 8192:
                continue
            got = device.integral_histogram(device.upload_image(px), lut, b, kernel=kernel).cpu().numpy()
            if not np.array_equal(got, want):
                bad += 1; print("MISMATCH", env, h, w, b, kernel)
t = torch.from_numpy(O.compute_crossweave(rng.integers(0, 256, (50, 70), dtype=np.uint8), O.np_uniform_table(6), 6)).cuda()
regs = [(0, 0, 49, 69), (3, 4, 20, 30), (49, 69, 49, 69)]
assert np.array_equal(device.region_histograms(t, regs).cpu().numpy(), O.region_histograms(t.cpu().numpy(), regs))
assert np.array_equal(device.window_counts(t, 7, 9).cpu().numpy(), O.window_counts(t.cpu().numpy(), 7, 9))
tm = np.ones(6) / 6
d = device.likelihood_map(t, tm, 7, 9, "intersection").cpu().numpy()
assert np.abs(d - O.np_likelihood_map(t.cpu().numpy(), tm, 7, 9, "intersection")).max() < 1e-12
# K6: 1-D scans (aligned / unaligned views, overflow flag), axis scans (u8 / u32,
# vector and scalar rows, middle axis), transposes of every element size
from paper_1711_01919_b200 import scan as S
from paper_1711_01919_b200.errors import ScanOverflowError
v = torch.from_numpy(rng.integers(0, 100, 5001)).cuda()
for off in (0, 1):
    got = S.inclusive_scan(v[off:]).cpu().numpy()
    bad += not np.array_equal(got, np.cumsum(v[off:].cpu().numpy()).astype(np.uint32))
    bad += int(S.exclusive_scan(v[off:]).cpu().numpy()[-1]) != int(got[-2])
try:
    S.inclusive_scan(np.array([2**32 - 1, 1]))
    bad += 1
except ScanOverflowError:
    pass
for shape, dt in (((33, 260), np.uint8), ((33, 259), np.uint8), ((17, 64), np.uint32), ((5, 3, 7), np.uint32)):
    a = rng.integers(0, 200, shape).astype(dt)
    for ax, fn in ((1, S.scan_rows), (0, S.scan_cols)):
        bad += not np.array_equal(fn(a), np.cumsum(a, axis=ax, dtype=np.uint32))
for dt in (np.uint8, np.uint16, np.uint32, np.float64, np.complex128):
    a = (rng.random((37, 45)) * 100).astype(dt)
    bad += not np.array_equal(S.transpose(a), a.T)
# K7: the wavefront with a recorded trace
pxw = rng.integers(0, 256, (50, 70), dtype=np.uint8)
cw, ev = device.wavefront(device.upload_image(pxw), O.np_uniform_table(5), 5, 16)
bad += not np.array_equal(cw.cpu().numpy(), O.compute_crossweave(pxw, O.np_uniform_table(5), 5))
print("sanitize cases done, mismatches:", bad)
