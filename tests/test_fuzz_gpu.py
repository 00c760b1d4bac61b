"""Seeded fuzzing of the K2 planner/kernel space against the oracle: random
shapes (ragged widths across column-tile boundaries, tall and short images),
bin counts and slabs, explicit LUTs, pitches/offsets, and random settings of
every plan knob (segments, tail split, carry scheme, batch rows, TMA/LDG,
column tiles, count kernel, PDL).  Bit-exact or it fails with the case."""

import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

from paper_1711_01919_b200 import device  # noqa: E402

KNOBS = ("IH_NSEG", "IH_TAIL_PCT", "IH_TAIL_DIV", "IH_CARRY_LOOKBACK", "IH_CARRY_CLUSTER",
         "IH_TABLE_SUM_MAX", "IH_ROWS_PER_BATCH", "IH_NO_TMA", "IH_NO_COLTILE", "IH_TILE_CHUNKS",
         "IH_COLCOUNTS_SLAB", "IH_NO_PDL", "IH_MIN_SEG_ROWS", "IH_K4_MODE", "IH_K5_DIRECT",
         "IH_STAGED_STORES", "IH_NO_RESTAGE", "IH_NO_ROWPACK", "IH_SMALL", "IH_SKEW_X100",
         "IH_SKEW_PCT", "IH_COLCOUNTS_G1", "IH_K5_CHAIN", "IH_COUNT_CW", "IH_KB")


def _case(rng):
    H = int(rng.choice([1, 2, 7, 33, 100, 257, 600, 1500]))
    W = int(rng.choice([1, 3, 64, 127, 128, 129, 1000, 2047, 2048, 2049, 3000, 4100, 6000]))
    bins = int(rng.choice([1, 2, 5, 16, 32, 64, 100, 256]))
    lo = int(rng.integers(0, bins))
    hi = int(rng.integers(lo + 1, bins + 1))
    env = {}
    if rng.random() < 0.7:
        env["IH_NSEG"] = str(int(rng.integers(1, 40)))
    if rng.random() < 0.3:
        env["IH_TAIL_PCT"] = str(int(rng.choice([10, 25, 50])))
        env["IH_TAIL_DIV"] = str(int(rng.choice([2, 4, 8])))
    elif rng.random() < 0.3:  # skewed segments: first pct % larger by skew/100
        env["IH_SKEW_X100"] = str(int(rng.choice([110, 130, 200])))
        env["IH_SKEW_PCT"] = str(int(rng.choice([25, 50, 75])))
    carry = rng.choice(["table", "lookback", "cluster", "prefix", "small"])
    if carry == "small":  # K2s, where it applies (aligned rows, W <= 2048)
        env["IH_SMALL"] = "1"
    elif carry == "lookback":
        env["IH_CARRY_LOOKBACK"] = "1"
    elif carry == "cluster":
        env["IH_CARRY_CLUSTER"] = "1"
    elif carry == "prefix":
        env["IH_TABLE_SUM_MAX"] = "1"
    env["IH_ROWS_PER_BATCH"] = str(int(rng.choice([1, 2, 4])))
    if rng.random() < 0.3:
        env["IH_COLCOUNTS_G1"] = "0"  # <= 4-bin slabs: the shared-atomic count kernel
    for k, p in (("IH_NO_TMA", 0.2), ("IH_NO_COLTILE", 0.2), ("IH_COLCOUNTS_SLAB", 0.2),
                 ("IH_NO_PDL", 0.2), ("IH_STAGED_STORES", 0.25)):
        if rng.random() < p:
            env[k] = "1"
    if rng.random() < 0.2:
        env["IH_TILE_CHUNKS"] = str(int(rng.choice([2, 4, 8])))
    if rng.random() < 0.2:
        env["IH_MIN_SEG_ROWS"] = "4"
    offset = int(rng.choice([0, 0, 1, 3]))
    if rng.random() < 0.5:  # unaligned rows: the kernels' own LDG path
        env["IH_NO_RESTAGE"] = "1"
    if rng.random() < 0.3:  # column chunks per count CTA (warps per chunk 8 / cw)
        env["IH_COUNT_CW"] = str(int(rng.choice([1, 2, 4, 8])))
    if rng.random() < 0.2:  # bins per scan CTA where row packing applies
        env["IH_KB"] = str(int(rng.choice([1, 2, 4])))
    return H, W, bins, lo, hi, env, offset


@pytest.mark.parametrize("seed", range(10))
def test_fuzz_plans_against_oracle(monkeypatch, seed):
    rng = np.random.default_rng(1000 + seed)
    for _ in range(20):
        H, W, bins, lo, hi, env, offset = _case(rng)
        for k in KNOBS:
            monkeypatch.delenv(k, raising=False)
        for k, v in env.items():
            monkeypatch.setenv(k, v)
        lut = rng.integers(0, bins, 256).astype(np.uint8) if rng.random() < 0.3 \
            else O.np_uniform_table(bins)
        base = rng.integers(0, 256, (H, W + offset), dtype=np.uint8)
        px = np.ascontiguousarray(base[:, offset:])
        view = torch.from_numpy(base).cuda()[:, offset:]
        kernel = "single_pass" if W <= 8192 or "IH_NO_COLTILE" not in env else "auto"
        try:
            got = device.integral_histogram(view, lut, bins, bin_range=(lo, hi), kernel=kernel)
        except Exception as exc:
            raise AssertionError(f"{exc!r} for {(H, W, bins, lo, hi, env, offset)} "
                                 f"plan {device.plan(1, H, W, hi - lo)}") from exc
        want = O.compute_crossweave(px, lut, bins)[lo:hi]
        assert np.array_equal(got.cpu().numpy(), want), (H, W, bins, lo, hi, env, offset)


@pytest.mark.parametrize("seed", range(4))
def test_fuzz_frame_batches_and_pitches(monkeypatch, seed):
    """Frame batches with padded row pitch and frame stride (views into a
    larger buffer), random plan knobs; every frame equals the oracle."""
    rng = np.random.default_rng(2000 + seed)
    for _ in range(10):
        F = int(rng.integers(1, 6))
        H = int(rng.choice([1, 5, 40, 333]))
        W = int(rng.choice([1, 17, 128, 700, 2100, 4097]))
        bins = int(rng.choice([1, 3, 32, 256]))
        for k in KNOBS:
            monkeypatch.delenv(k, raising=False)
        if rng.random() < 0.6:
            monkeypatch.setenv("IH_NSEG", str(int(rng.integers(1, 12))))
        if rng.random() < 0.3:
            monkeypatch.setenv("IH_TAIL_PCT", "30")
        pad_w, pad_h = int(rng.choice([0, 16, 5])), int(rng.choice([0, 2]))
        base = rng.integers(0, 256, (F, H + pad_h, W + pad_w), dtype=np.uint8)
        view = torch.from_numpy(base).cuda()[:, :H, :W]
        lut = O.np_uniform_table(bins)
        got = device.integral_histogram(view, lut, bins).cpu().numpy()
        for f in range(F):
            want = O.compute_crossweave(np.ascontiguousarray(base[f, :H, :W]), lut, bins)
            assert np.array_equal(got[f], want), (F, H, W, bins, pad_w, pad_h, f)


@pytest.mark.parametrize("seed", range(3))
def test_fuzz_queries(monkeypatch, seed):
    """K3 regions, K4 windows (every kernel variant) and K5 maps (table and
    direct) on random tensors against the oracle / numpy restatement."""
    rng = np.random.default_rng(3000 + seed)
    for _ in range(6):
        H, W = int(rng.integers(1, 200)), int(rng.integers(1, 1500))
        bins = int(rng.choice([1, 4, 17, 64]))
        px = rng.integers(0, 256, (H, W), dtype=np.uint8)
        full = O.compute_crossweave(px, O.np_uniform_table(bins), bins)
        t = torch.from_numpy(full.view(np.int32)).cuda().view(torch.uint32)
        regs = []
        for _ in range(50):
            r0, r1 = sorted(rng.integers(0, H, 2).tolist())
            c0, c1 = sorted(rng.integers(0, W, 2).tolist())
            regs.append((r0, c0, r1, c1))
        assert np.array_equal(device.region_histograms(t, regs).cpu().numpy(),
                              O.region_histograms(full, regs))
        h, w = int(rng.integers(1, H + 1)), int(rng.integers(1, W + 1))
        want = O.window_counts(full, h, w)
        for mode in ("0", "1", "2", "3", "4"):
            monkeypatch.setenv("IH_K4_MODE", mode)
            assert np.array_equal(device.window_counts(t, h, w).cpu().numpy(), want), (H, W, h, w, mode)
        tmpl = rng.random(bins)
        tmpl /= tmpl.sum()
        for metric in ("intersection", "bhattacharyya"):
            ref = O.np_likelihood_map(full, tmpl, h, w, metric)
            base = None
            for direct, chain in (("0", "2"), ("0", "0"), ("0", "4"), ("1", "0")):
                monkeypatch.setenv("IH_K5_DIRECT", direct)
                monkeypatch.setenv("IH_K5_CHAIN", chain)
                got = device.likelihood_map(t, tmpl, h, w, metric).cpu().numpy()
                assert np.abs(got - ref).max() < 1e-12, (H, W, h, w, metric, direct, chain)
                if base is None:
                    base = got
                else:  # every K5 variant computes the same terms in the same order
                    assert np.array_equal(got, base), (H, W, h, w, metric, direct, chain)
