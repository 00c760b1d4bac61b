#!/bin/bash
# Quick check after a prepass/scan change: parity + fuzz, per-kernel small-bin
# times, graph-timed bin counts / shards / small images.
OUT=gpurun_out/${1:-quick}
mkdir -p $OUT
timeout 1200 python -m pytest tests/test_parity_gpu.py tests/test_fuzz_gpu.py -q -x > $OUT/pytest.log 2>&1; echo pytest=$?; tail -1 $OUT/pytest.log
bash scripts/gpu_smallbins.sh ${1:-quick}/smallbins > $OUT/smallbins.txt 2>&1
python scripts/graph_time.py hd64b1 hd64b2 hd64b4 hd64b8 hd64b16 hd64 > $OUT/bin_counts.jsonl 2>&1
python scripts/graph_time.py 4k128 4k128/2 4k128/4 4k128/8 8k256/4 8k256/8 hd8 hd1 512 512x8 > $OUT/shards.jsonl 2>&1
python3 - <<PY
import json, glob
for f in sorted(glob.glob("$OUT/*.jsonl")):
    for l in open(f):
        if l.startswith("{"):
            d = json.loads(l); p = d["plan"]
            print(f"  {d['wl']:10s} {d['graph_ms_per_call']*1000:9.1f} us  frac {d['frac']:.3f}  segs {p['segments']:3d} kb {p['bins_per_cta']}")
PY
