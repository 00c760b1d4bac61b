#!/bin/bash
# Final-code sweep: common frame sizes, bin counts, small images, shares
# (graph-timed calls, heuristic plans) + query kernels.
OUT=gpurun_out/${1:-r02_sweep}
mkdir -p $OUT
python scripts/graph_time.py vga64 svga64 xga64 hd720x64 wxga64 hdp64 hd64 qhd16 uhd8 > $OUT/common_sizes.jsonl 2>&1
python scripts/graph_time.py hd64b1 hd64b2 hd64b4 hd64b8 hd64b16 hd64 hd64b37 hd64b64 > $OUT/bin_counts.jsonl 2>&1
python scripts/graph_time.py 512 512b16 512b64 s384 s768 vga1 svga1 hd1 hd2 hd4 hd8 hd16 hd32 512x8 > $OUT/small_and_frames.jsonl 2>&1
python scripts/graph_time.py 4k128 4k128/2 4k128/4 4k128/8 8k256 8k256/2 8k256/4 8k256/8 > $OUT/shards.jsonl 2>&1
python scripts/graph_time.py hd8w1921 hd8w1922 hd8w1924 hd64w1921 > $OUT/odd_widths.jsonl 2>&1
python scripts/bench_queries.py > $OUT/queries.jsonl 2>&1
python3 - <<PY
import json, glob
for f in sorted(glob.glob("$OUT/*.jsonl")):
    print("==", f.split("/")[-1])
    for l in open(f):
        if not l.startswith("{"): continue
        d = json.loads(l)
        if "graph_ms_per_call" in d:
            p = d["plan"]
            print(f"  {d['wl']:10s} {d['graph_ms_per_call']*1000:9.1f} us  frac {d['frac']:.3f}  segs {p['segments']:3d} carry {p['carry']:9s} launches {p['launches']}")
        else:
            print("  ", {k: v for k, v in d.items() if k in ("kernel", "tensor", "window", "ms", "frac", "speedup")})
PY
