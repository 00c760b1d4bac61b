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
         "IH_COLCOUNTS_SLAB", "IH_NO_PDL", "IH_MIN_SEG_ROWS")


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
    carry = rng.choice(["table", "lookback", "cluster", "prefix"])
    if carry == "lookback":
        env["IH_CARRY_LOOKBACK"] = "1"
    elif carry == "cluster":
        env["IH_CARRY_CLUSTER"] = "1"
    elif carry == "prefix":
        env["IH_TABLE_SUM_MAX"] = "1"
    env["IH_ROWS_PER_BATCH"] = str(int(rng.choice([1, 2, 4])))
    for k, p in (("IH_NO_TMA", 0.2), ("IH_NO_COLTILE", 0.2), ("IH_COLCOUNTS_SLAB", 0.2),
                 ("IH_NO_PDL", 0.2)):
        if rng.random() < p:
            env[k] = "1"
    if rng.random() < 0.2:
        env["IH_TILE_CHUNKS"] = str(int(rng.choice([2, 4, 8])))
    if rng.random() < 0.2:
        env["IH_MIN_SEG_ROWS"] = "4"
    offset = int(rng.choice([0, 0, 1, 3]))
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
