#!/bin/bash
# One GPU session: bench line, ncu launch list of the same command, one
# ncu --set full capture of the dominant kernel.  Outputs under gpurun_out/.
set -u
mkdir -p gpurun_out
TAG=${1:-r01}
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err
echo bench=$?
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_${TAG}.csv \
  python bench.py --steps 10 --warmup 3 --e2e-steps 0 --no-cpu-baseline > /dev/null 2>&1
echo ncu_launches=$?
timeout 400 ncu --set full --clock-control none --import-source on -k regex:k2_scan -s 3 -c 1 \
  -o gpurun_out/prof_k2_${TAG} -f \
  python bench.py --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline > /dev/null 2>&1
echo ncu_full=$?
