#!/bin/bash
# Round-2 batch: GPU tests (incl. capacity edge, streamed overlap, pinned
# release), per-kernel ncu summaries, k2_scan traffic per plan, cfg1 timeline
# and ncu, eager host overhead.
set -u
TAG=${1:-r02c}
OUT=gpurun_out/$TAG
mkdir -p $OUT
timeout 1500 python -m pytest tests -q -m gpu -x > $OUT/pytest.log 2>&1; echo pytest=$?; tail -1 $OUT/pytest.log
timeout 200 python scripts/eager_overhead.py > $OUT/eager_overhead_512.txt 2>&1; echo eager=$?
timeout 200 python scripts/cta_timeline.py 512 > $OUT/cta_timeline_512.json 2>&1; echo timeline=$?
timeout 200 python scripts/cta_timeline.py hd1 > $OUT/cta_timeline_hd1.json 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k2_scan -s 1 -c 1 \
  -o $OUT/k2_scan_512 -f python scripts/one.py 512 > /dev/null 2>&1; echo ncu512=$?
python scripts/ncu_summary.py $OUT/k2_scan_512.ncu-rep > $OUT/k2_scan_512_summary.json 2>/dev/null
KEEP_REPS="k3_shard32" bash scripts/gpu_kernel_profiles.sh $TAG
bash scripts/traffic_capture.sh $TAG; echo traffic=$?
du -sh $OUT
