mkdir -p gpurun_out
timeout 900 python bench.py --e2e-steps 0 --no-cpu-baseline > gpurun_out/bench_w_hd64.json 2> gpurun_out/bench_w.err; echo b1=$?
timeout 900 python bench.py --workload 8k256 --e2e-steps 0 --no-cpu-baseline > gpurun_out/bench_w_8k256.json 2>> gpurun_out/bench_w.err
echo done
