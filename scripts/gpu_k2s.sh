#!/bin/bash
# K2s (one-launch small-image kernel): parity, sanitizers, phase timeline,
# graph-timed A/B vs the count-table path, cfg1 bench line.
set -u
TAG=${1:-k2s}
OUT=gpurun_out/$TAG
mkdir -p $OUT
timeout 600 python -m pytest tests/test_parity_gpu.py -q -x -k "k2s or streamed or to_host" > $OUT/pytest_k2s.log 2>&1; echo pytest_k2s=$?; tail -1 $OUT/pytest_k2s.log
timeout 900 python -m pytest tests/test_fuzz_gpu.py -q -x > $OUT/pytest_fuzz.log 2>&1; echo fuzz=$?; tail -1 $OUT/pytest_fuzz.log
for tool in memcheck racecheck synccheck; do
  timeout 600 compute-sanitizer --tool $tool --kernel-name kns=k2_small python scripts/k2s_case.py > $OUT/san_$tool.txt 2>&1; echo san_$tool=$?; tail -1 $OUT/san_$tool.txt
done
for w in 512 hd1 vga1 512b64; do python scripts/k2s_phases.py $w; done > $OUT/phases.jsonl 2>&1
for env in "IH_SMALL=0" "IH_SMALL=1"; do
  env $env timeout 300 python scripts/graph_time.py 512 hd1 vga1 svga1 s384 s768 512b16 512b64 512x8 > $OUT/graph_${env}.jsonl 2>&1; echo graph_$env=$?
done
timeout 300 python scripts/eager_overhead.py > $OUT/eager_overhead_512.txt 2>&1; head -1 $OUT/eager_overhead_512.txt
timeout 600 python bench.py --workload 512 > $OUT/bench512.json 2> $OUT/bench512.err; echo bench512=$?
