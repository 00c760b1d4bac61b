#!/bin/bash
# Column-tile A/B: parity tests for the tiled path, then CUDA-graph device time
# per workload with column tiles (default) and without (IH_NO_COLTILE=1).
mkdir -p gpurun_out
TAG=${1:-ct}
timeout 900 python -m pytest tests/test_parity_gpu.py -q -x -k "column_tile or config_checksums or 4k_bin or segments_and or small_cases or plan_describe" > gpurun_out/pytest_${TAG}.log 2>&1; echo pytest=$?
WLS="4k128 4k128/2 4k128/4 4k128/8 8k256/8 8k256 hd64 hd1"
timeout 600 python scripts/graph_time.py $WLS > gpurun_out/graph_${TAG}_colt.jsonl 2>&1; echo colt=$?
IH_NO_COLTILE=1 timeout 600 python scripts/graph_time.py $WLS > gpurun_out/graph_${TAG}_nocolt.jsonl 2>&1; echo nocolt=$?
