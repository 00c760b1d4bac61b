"""Generate the golden fixtures by running the REFERENCE `inthist` package.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports the reference from /root/reference/pkg/src and writes small
fixtures next to this script.  They pin both the oracle (oracle/) and the
CUDA path to the reference's own outputs.  Nothing on the GPU box reads
/root/reference; only these committed files travel.

Fixtures:
  c1_instances.json   -- the 200 acceptance-C1 instances (test_acceptance.py:48-61,
                         seed 20260823): (W, H, B, tile), crc32 of the image bytes
                         and crc32 of the reference compute_sequential tensor.
  configs.json        -- tensor_checksum (bench.py:65-66) of the BASELINE configs
                         (synth_image seed 0; HD frames seeds 0..63), computed here
                         with the reference; the 8192x8192x256 per-plane values are
                         SURVEY.md Appendix A (reference compute_streamed, 698 s).
  scans.npz           -- the reference scan module (scan.py:33-103) on edge
                         inputs: 1-D scans across the device tile size, u64 wrap,
                         negative ints, overflow at / past the last prefix,
                         plane scans of several dtypes, transposes;
                         ``<case>__raises`` holds the exception name, ``<case>__in_of``
                         the case whose input it shares.
  likelihood.npz      -- reference likelihood_map / best_match (likelihood.py:55-86)
                         on random and structured images: both metrics, square,
                         rectangular, 1x1 and full-image windows, B in {1, 3, 16,
                         64, 256}, templates from normalize(region_histogram(...))
                         (the reference tests' construction) and random ones.
  small_cases.npz     -- full reference tensors for hand-picked edge cases
                         (known answers of tests/test_strategies.py, explicit LUTs,
                         B=256, ragged shapes), plus reference region_histogram
                         and window_counts outputs on them.
"""

from __future__ import annotations

import json
import os
import sys
import zlib

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REF)

import inthist  # noqa: E402  (the reference)
from inthist.bench import synth_image, tensor_checksum  # noqa: E402
from inthist.likelihood import window_counts  # noqa: E402

SEED = 20260823
WIDTHS = [1, 2, 3, 5, 17, 33, 64, 97, 131, 257]
HEIGHTS = [1, 2, 7, 19, 33, 61, 96, 128, 193]
BINS = [1, 2, 3, 16, 64]
TILES = [1, 7, 64]


def c1_instances():
    """test_acceptance.py:48-61 + :68-75 (same RNG stream, same order)."""
    rng = np.random.default_rng(SEED)
    fixed = [(1, 1, 1, 1), (1, 1, 64, 64), (257, 193, 16, 64), (257, 193, 64, 7)]
    inst = list(fixed)
    while len(inst) < 200:
        inst.append((int(rng.choice(WIDTHS)), int(rng.choice(HEIGHTS)),
                     int(rng.choice(BINS)), int(rng.choice(TILES))))
    out = []
    for w, h, b, tile in inst:
        px = rng.integers(0, 256, size=(h, w), dtype=np.uint8)
        ih = inthist.compute_sequential(inthist.GrayImage(px), inthist.BinSpec.uniform(b))
        out.append({"w": w, "h": h, "bins": b, "tile": tile,
                    "img_crc": f"{zlib.crc32(px.tobytes()):08x}",
                    "crc": tensor_checksum(ih)})
    return out


def configs():
    res = {}
    for (w, h, b) in [(64, 64, 16), (512, 512, 32), (1920, 1080, 32), (3840, 2160, 128)]:
        img = synth_image(w, h, 0)
        ih = inthist.compute(img, inthist.BinSpec.uniform(b), inthist.CROSSWEAVE)
        res[f"{w}x{h}x{b}"] = {"seed": 0, "crc": tensor_checksum(ih),
                              "img_crc": f"{zlib.crc32(img.pixels.tobytes()):08x}"}
        if (w, h) == (3840, 2160):  # per-plane crcs for bin-shard checks
            res[f"{w}x{h}x{b}"]["plane_crc"] = [
                f"{zlib.crc32(ih.counts[k].astype('<u4').tobytes()):08x}" for k in range(b)]
        print(w, h, b, res[f"{w}x{h}x{b}"], flush=True)
    spec = inthist.BinSpec.uniform(32)
    frames = []
    for k in range(64):
        ih = inthist.compute(synth_image(1920, 1080, k), spec, inthist.CROSSWEAVE)
        frames.append(tensor_checksum(ih))
    res["1920x1080x32_frames"] = frames
    res["8192x8192x256"] = {
        "seed": 0,
        "source": "SURVEY.md Appendix A (reference compute_streamed, 1-bin chunks)",
        "crc": "b416da31",
        "plane_crc": APPENDIX_A_PLANES.split(),
    }
    return res


APPENDIX_A_PLANES = """
a4def62a 92b94c39 4f2dfcbd 02d3fa73 a3df4740 88d08cdc 34a3d251 ee8209e6 64e6892a fc66f578 c4c1f941 a05a472b b163325e 14df6051 a5e8704c 163f14b7
98c6ee77 afa8e8cb 37f3da33 0d434b37 b3d41091 fb9275ac e5fd589e 17506c2f d4551290 dbd8b564 aff7b50e 1de79817 2919dacd 78f42ceb 17131024 995c6c4e
deef505b 55ed3d38 96cef745 2940c5e1 16701882 3be29c06 ba9f589a 82fbdaac 1df331f2 d1323d11 83702f8d 6791ac60 1fe89d79 0c3e7556 c24abf27 405fd665
b166b92a 0affe75c 5945318d bbb9139e 0d1e95cc 4ffff944 572635db d4e778e4 4424e688 42914ee5 89afd8af 0f66b69d df777d4c 7f7ac588 65f4773a 1115e97d
3fb6b639 c5a2d82c 61bfa510 88144127 20044f27 4694cf27 0dae07c5 7835eea1 f53bd16b 8838ef20 b48559f7 f9a4c1c2 a0def3d4 4d01a1db aa2eb3be c9980e60
b5659310 849380da 09fd7e2e 371b1d40 f9776323 f59595cc e7ec2568 d503ec9d f43d3b96 0600d24e 437bdeda 5baf07b6 453923ab ffcf3919 f0987739 1d0b6b41
394a4216 9cf019c0 130b81f9 7359ccbf bd91e427 862b0a4f e1faa447 a7838aa2 499cf937 239d5e3f 2e664cc2 6be24750 09525504 3bff17c8 c076bea6 b36bcce7
abb8066e 21a20e17 8dbc9aa2 4c6f645e 36a86a31 a72a3b4b 72043292 4e3431a3 bc7f6318 a8755037 d95b8ad5 39ab25ea 6a9e874f 6110048a 5ce43972 a08408ae
555c1a94 7756a7e2 beeffce2 e0045645 7ec4a974 ec45fe5c 873a2ac3 92a0c57f 81740d8c e06034c8 afb5b588 b2a3dee0 6eb56f1e 99f60d4e 32256cc9 c111de02
424f9801 b815ff5e 1ea8c973 8714f7f0 a6593702 88713c7e a8a16769 914e9d1b c3318969 ceb9f1b1 2c1759bc 0b7b5a20 7ec4e3a4 ba35bb1a 5994f301 5cc564e4
b7383b01 afba2789 982ec5bc 0d01df62 9d8a3ba2 f2d7bdba 7cd26741 a36dc522 70ba2514 f3157357 a75e37a9 54e6a218 45e96fc9 164cdf97 8a958288 dfa94281
eff1a8ab 8c765032 f8a88801 3c4f0b30 522d2dce b52be353 72d22f28 1d017ebf 621d6bc7 1b7514a4 1885ba25 01a65450 e431a76f fe187c8a 50e17df6 37b58fa6
b2a9d636 9f10e133 f7a66308 2efb49cd eaf095cf edd4f439 1f9b0802 d0a55af7 362a88ce f59ad5b7 bc8e9c60 5e8a049d ab57542b 1180463c 9de4e442 1e200deb
07356ead 5da65d4f 3d0b0cc6 eb78fdac f673acdc 4daa2ac3 b6c7c826 7ff3bd99 dac93f98 b285cfcf 8f9808be 65c9ea2f 144074c8 3729789e 26d07300 614b6e0e
4f3ac100 e56d38b6 9b6a514e aac0672a cd56db48 b35a6ce7 6fd75e5d e00569d9 445a76a5 95d253b2 4b7ce0f4 fb6fac7b cd056aeb d6cd9fd2 5a49d98e 9b268690
03e6ca96 232dbb23 36959ee3 4825aabf a800a1bc b0e62b0c 04e20e75 09755bf4 9fb7a34c f0f9e8a4 f7f1dca1 69a189ad 74296f72 ae1a2f8f f2be5d59 4ba6753d
"""


def small_cases():
    """Edge cases with full reference tensors + query outputs."""
    rng = np.random.default_rng(SEED + 100)
    cases = {}

    def add(name, px, spec, regions=(), windows=()):
        ih = inthist.compute_sequential(inthist.GrayImage(px), spec)
        cases[f"{name}__img"] = px
        cases[f"{name}__lut"] = np.asarray(spec.table, dtype=np.uint8)
        cases[f"{name}__bins"] = np.array(spec.bins)
        cases[f"{name}__counts"] = ih.counts
        if regions:
            regs = np.array(regions, dtype=np.int32)
            got = np.stack([inthist.region_histogram(ih, inthist.Region(*r)).counts
                            for r in regions])
            cases[f"{name}__regions"] = regs
            cases[f"{name}__region_counts"] = got
        for (h, w) in windows:
            cases[f"{name}__win_{h}x{w}"] = window_counts(ih, h, w)

    add("pix2x2", np.array([[0, 255], [128, 0]], dtype=np.uint8), inthist.BinSpec.uniform(2))
    add("const3x5", np.full((3, 5), 200, dtype=np.uint8), inthist.BinSpec.uniform(4))
    add("one77", np.array([[77]], dtype=np.uint8), inthist.BinSpec.uniform(16))
    add("row1x31", rng.integers(0, 256, (1, 31), dtype=np.uint8), inthist.BinSpec.uniform(4))
    add("col47x1", rng.integers(0, 256, (47, 1), dtype=np.uint8), inthist.BinSpec.uniform(3))
    add("b256_64x64", rng.integers(0, 256, (64, 64), dtype=np.uint8), inthist.BinSpec.uniform(256),
        regions=[(0, 0, 63, 63), (5, 7, 40, 33), (63, 63, 63, 63)], windows=[(8, 8)])
    tab = rng.integers(0, 7, 256)
    add("explicit7_97x61", rng.integers(0, 256, (61, 97), dtype=np.uint8), inthist.BinSpec.explicit(tab),
        regions=[(0, 0, 60, 96), (3, 4, 3, 4), (10, 20, 50, 90)], windows=[(5, 4), (61, 97), (1, 1)])
    tab2 = np.zeros(256, dtype=np.uint8)
    tab2[128:] = 1
    add("explicit_step_33x130", rng.integers(0, 256, (33, 130), dtype=np.uint8), inthist.BinSpec(2, tab2))
    add("ragged_193x257x64", rng.integers(0, 256, (193, 257), dtype=np.uint8), inthist.BinSpec.uniform(64),
        regions=[(int(a), int(b), int(c), int(d)) for a, b, c, d in
                 [(0, 0, 192, 256), (1, 1, 1, 1), (100, 3, 150, 255), (0, 200, 0, 256)]],
        windows=[(64, 64), (7, 13)])
    add("wide1x600", rng.integers(0, 256, (1, 600), dtype=np.uint8), inthist.BinSpec.uniform(5))
    return cases


def scans():
    """Reference scan-module outputs (scan.py:33-103) on edge inputs."""
    from inthist import scan as S

    rng = np.random.default_rng(SEED + 200)
    out, seen = {}, {}

    def run(name, fn, x, *args):
        if id(x) in seen:  # shared input: stored once, referenced by name
            out[f"{name}__in_of"] = np.array(seen[id(x)])
        else:
            seen[id(x)] = name
            out[f"{name}__in"] = np.asarray(x)
        try:
            out[f"{name}__out"] = np.asarray(fn(x, *args))
        except Exception as exc:  # noqa: BLE001 - the class name is the fixture
            out[f"{name}__raises"] = np.array(type(exc).__name__)

    for n in (1, 2, 255, 2047, 2048, 2049, 4096 + 3, 10_007):
        x = rng.integers(0, 1000, n).astype(np.uint16)
        run(f"incl_{n}", S.inclusive_scan, x)
        run(f"excl_{n}", S.exclusive_scan, x)
        run(f"blk7_{n}", S.blocked_scan, x, 7)
    big = np.full(5000, 2**20, dtype=np.int64)  # 2^20 * 4096 = 2^32: overflow at i = 4095
    run("incl_over_mid", S.inclusive_scan, big)
    run("excl_over_mid", S.exclusive_scan, big)
    run("excl_last_only", S.exclusive_scan, np.array([2**32 - 1, 5], dtype=np.int64))
    run("incl_last_only", S.inclusive_scan, np.array([2**32 - 1, 5], dtype=np.int64))
    run("incl_neg_wrap", S.inclusive_scan, np.array([5, -3, 2], dtype=np.int64))
    run("incl_neg_over", S.inclusive_scan, np.array([-1], dtype=np.int64))
    run("incl_huge_elem", S.inclusive_scan, np.array([2**40], dtype=np.int64))
    run("incl_u64_wrap", S.inclusive_scan, np.array([5, 2**64 - 5, 3], dtype=np.uint64))
    run("incl_u64_over", S.inclusive_scan, np.array([2**63, 2**63, 7], dtype=np.uint64))
    run("incl_int8", S.inclusive_scan, np.array([-1, 1, 100], dtype=np.int8))
    run("incl_2d", S.inclusive_scan, rng.integers(0, 50, (13, 17)))
    run("incl_bool", S.inclusive_scan, rng.random(3000) < 0.5)
    for name, plane in (
        ("u32", rng.integers(0, 2**32, (37, 53), dtype=np.uint64).astype(np.uint32)),
        ("u8", rng.integers(0, 256, (65, 300), dtype=np.uint8)),
        ("i64", rng.integers(-2**40, 2**40, (5, 1000), dtype=np.int64)),
        ("bool", rng.random((17, 9)) < 0.3),
        ("tall", rng.integers(0, 2**31, (3000, 3), dtype=np.uint64).astype(np.uint32)),
        ("wide", rng.integers(0, 2**31, (2, 3000), dtype=np.uint64).astype(np.uint32)),
        ("vec", rng.integers(0, 9, 40, dtype=np.uint32)),
    ):
        run(f"rows_{name}", S.scan_rows, plane)
        run(f"cols_{name}", S.scan_cols, plane)
    for name, plane in (
        ("u8", rng.integers(0, 256, (33, 65), dtype=np.uint8)),
        ("u16", rng.integers(0, 2**16, (70, 31), dtype=np.uint16)),
        ("u32", rng.integers(0, 2**32, (100, 3), dtype=np.uint64).astype(np.uint32)),
        ("f64", rng.random((45, 64))),
        ("c128", rng.random((9, 40)) + 1j * rng.random((9, 40))),
        ("one", np.array([[7]], dtype=np.uint32)),
    ):
        run(f"tr_{name}", S.transpose, plane)
    return out


def likelihood():
    """Reference likelihood_map / best_match outputs (likelihood.py:55-86)."""
    from inthist.likelihood import best_match, likelihood_map

    rng = np.random.default_rng(SEED + 300)
    out = {}

    def add(name, px, spec, template, h, w, metric):
        ih = inthist.compute_sequential(inthist.GrayImage(px), spec)
        lm = likelihood_map(ih, template, h, w, metric)
        r, c, v = best_match(lm)
        out[f"{name}__img"] = px
        out[f"{name}__lut"] = np.asarray(spec.table, dtype=np.uint8)
        out[f"{name}__bins"] = np.array(spec.bins)
        out[f"{name}__template"] = np.asarray(template, dtype=np.float64)
        out[f"{name}__hw"] = np.array([h, w])
        out[f"{name}__metric"] = np.array(metric)
        out[f"{name}__map"] = lm.values
        out[f"{name}__best"] = np.array([r, c], dtype=np.int64)
        out[f"{name}__best_value"] = np.array(v)

    def region_template(px, spec, reg):
        ih = inthist.compute_sequential(inthist.GrayImage(px), spec)
        return inthist.normalize(inthist.region_histogram(ih, inthist.Region(*reg)))

    for metric in ("intersection", "bhattacharyya"):
        m = metric[:5]
        px = rng.integers(0, 256, (30, 40), dtype=np.uint8)
        spec = inthist.BinSpec.uniform(16)
        add(f"rnd40x30_b16_{m}", px, spec, region_template(px, spec, (10, 12, 17, 19)), 8, 8, metric)
        px = rng.integers(0, 256, (61, 97), dtype=np.uint8)
        spec = inthist.BinSpec.uniform(64)
        add(f"rect97x61_b64_{m}", px, spec, region_template(px, spec, (3, 5, 22, 13)), 20, 9, metric)
        spec = inthist.BinSpec.uniform(256)
        px = rng.integers(0, 256, (64, 70), dtype=np.uint8)
        add(f"b256_{m}", px, spec, region_template(px, spec, (0, 0, 15, 15)), 16, 16, metric)
        tpl = rng.random(3)
        tpl /= tpl.sum()
        px = rng.integers(0, 256, (25, 33), dtype=np.uint8)
        add(f"randtpl_b3_{m}", px, inthist.BinSpec.uniform(3), tpl, 5, 7, metric)
        add(f"win1x1_b3_{m}", px, inthist.BinSpec.uniform(3), tpl, 1, 1, metric)
        add(f"full_b3_{m}", px, inthist.BinSpec.uniform(3), tpl, 25, 33, metric)
        add(f"b1_{m}", px, inthist.BinSpec.uniform(1), np.array([1.0]), 4, 4, metric)
        # structured: blocks of constant value, so many windows tie (best_match tie rule)
        blk = np.kron(rng.integers(0, 4, (6, 8)), np.ones((8, 8), dtype=np.int64)).astype(np.uint8) * 60
        spec = inthist.BinSpec.uniform(8)
        add(f"blocks64x48_b8_{m}", blk, spec, region_template(blk, spec, (8, 8, 15, 15)), 8, 8, metric)
        tab = rng.integers(0, 5, 256)
        px = rng.integers(0, 256, (40, 50), dtype=np.uint8)
        spec = inthist.BinSpec.explicit(tab)
        add(f"explicit5_{m}", px, spec, region_template(px, spec, (0, 0, 39, 49)), 12, 10, metric)
    return out


def main():
    if "--only-likelihood" in sys.argv:
        np.savez_compressed(os.path.join(HERE, "likelihood.npz"), **likelihood())
        return
    if "--only-scans" in sys.argv:
        np.savez_compressed(os.path.join(HERE, "scans.npz"), **scans())
        return
    np.savez_compressed(os.path.join(HERE, "scans.npz"), **scans())
    np.savez_compressed(os.path.join(HERE, "likelihood.npz"), **likelihood())
    inst = c1_instances()
    with open(os.path.join(HERE, "c1_instances.json"), "w") as fh:
        json.dump(inst, fh, indent=0)
    print("c1 done", flush=True)
    np.savez_compressed(os.path.join(HERE, "small_cases.npz"), **small_cases())
    print("small cases done", flush=True)
    with open(os.path.join(HERE, "configs.json"), "w") as fh:
        json.dump(configs(), fh, indent=1)
    print("configs done", flush=True)


if __name__ == "__main__":
    main()
