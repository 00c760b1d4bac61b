#!/bin/bash
# Bins per scan CTA (IH_KB = 1 / 2 / 4, heuristic segment counts) on the shapes
# row packing applies to; then the final-code sweep with the default planner.
OUT=gpurun_out/${1:-kb_sweep}
mkdir -p $OUT
for kb in 1 2 4; do
  IH_KB=$kb timeout 900 python scripts/graph_time.py hd64 hd64b64 hd64b37 hdp64 hd720x64 wxga64 hd16 hd32 hd8 > $OUT/kb$kb.jsonl 2>&1; echo kb$kb=$?
done
timeout 1800 bash scripts/gpu_r02_sweep.sh ${1:-kb_sweep}/sweep > $OUT/sweep_summary.txt 2>&1; echo sweep=$?
