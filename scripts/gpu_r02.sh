#!/bin/bash
# Round-2 evidence pass: GPU tests, smoke, reference suite, bench lines, launch list.
mkdir -p gpurun_out
TAG=${1:-r02a}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu_${TAG}.txt 2>&1
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_${TAG}.log 2>&1; echo pytest=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_${TAG}.log 2>&1; echo smoke=$?
timeout 900 scripts/reftests/run.sh run gpurun_out/reftests_${TAG} > /dev/null 2>&1; echo reftests=$?
timeout 600 python bench.py > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err; echo bench=$?
timeout 600 python bench.py --workload 512 > gpurun_out/bench512_${TAG}.json 2> gpurun_out/bench512_${TAG}.err; echo bench512=$?
timeout 600 python bench.py --impl reference --steps 3 > gpurun_out/benchref_${TAG}.json 2> gpurun_out/benchref_${TAG}.err; echo benchref=$?
timeout 300 python bench.py --gpus 2 > gpurun_out/bench_g2_${TAG}.json 2> gpurun_out/bench_g2_${TAG}.err; echo bench_g2=$?
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_${TAG}.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo launches=$?
