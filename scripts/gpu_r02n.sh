#!/bin/bash
# Re-entry check of the restored final code on a fresh box (GPU suite, smoke,
# default bench line, reference arm) plus a segment-count sweep of the
# 4K x 128 8-way share beyond the 32-row minimum segment.
set -u
OUT=gpurun_out/r02n
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem --format=csv > $OUT/gpu.txt 2>&1
timeout 1200 python -m pytest tests -q -m gpu -x > $OUT/pytest_gpu.log 2>&1; echo pytest=$?; tail -1 $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo smoke=$?
timeout 600 python bench.py > $OUT/bench_hd64.json 2> $OUT/bench_hd64.err; echo hd64=$?
timeout 600 python bench.py --impl reference --steps 3 > $OUT/ref_hd64.json 2> $OUT/ref_hd64.err; echo ref=$?
for n in 0 36 48 54 60 72 74 90 108 135 144; do
  if [ $n = 0 ]; then timeout 120 python scripts/graph_time.py 4k128/8 4k128/4 hd8; else
  IH_NSEG=$n timeout 120 python scripts/graph_time.py 4k128/8 4k128/4 hd8; fi | sed "s/^{/{\"nseg\": $n, /"
done > $OUT/nseg_4k8.jsonl 2> $OUT/nseg_4k8.err; echo nseg=$?
cut -c1-200 $OUT/nseg_4k8.jsonl
