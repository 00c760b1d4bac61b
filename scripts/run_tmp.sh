mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py -q -x -k "autotune or plan_describe or graph" > gpurun_out/pytest_at.log 2>&1; echo pytest=$?
timeout 900 python bench.py --e2e-steps 1 > gpurun_out/bench_at_hd64.json 2> gpurun_out/bench_at_hd64.err; echo b1=$?
for fr in 32 16 8; do timeout 900 python bench.py --frames $fr --e2e-steps 0 --no-cpu-baseline > gpurun_out/bench_at_hd$fr.json 2>> gpurun_out/bench_at.err; done
timeout 900 python bench.py --workload 4k128 --e2e-steps 0 --no-cpu-baseline > gpurun_out/bench_at_4k128.json 2>> gpurun_out/bench_at.err
timeout 900 python bench.py --workload 8k256 --e2e-steps 0 --no-cpu-baseline > gpurun_out/bench_at_8k256.json 2>> gpurun_out/bench_at.err
echo done
