mkdir -p gpurun_out
for fr in 64 16 8; do timeout 900 python bench.py --frames $fr --e2e-steps 0 --no-cpu-baseline > gpurun_out/bench_r_hd$fr.json 2>> gpurun_out/bench_r.err; done
timeout 900 python bench.py --workload 4k128 --e2e-steps 0 --no-cpu-baseline > gpurun_out/bench_r_4k128.json 2>> gpurun_out/bench_r.err
echo done
