#!/bin/bash
# tests + bench + 2-rank path test (gloo, both ranks on GPU 0) + launch lists of single-image configs
mkdir -p gpurun_out
TAG=${1:-x}
timeout 1200 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_${TAG}.log 2>&1; echo pytest=$?
timeout 600 python bench.py > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err; echo bench=$?
IH_BENCH_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 2 --steps 5 --warmup 3 --e2e-steps 1 > gpurun_out/bench2_${TAG}.json 2> gpurun_out/bench2_${TAG}.err; echo bench2=$?
for wl in hd1 4k128 4k128/8 8k256/8 512; do
  n=$(echo $wl | tr '/' '_')
  timeout 200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}_${n}.csv python scripts/one.py $wl > /dev/null 2>&1
done
echo launches=$?
