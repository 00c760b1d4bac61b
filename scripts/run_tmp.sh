mkdir -p gpurun_out
for fr in 8 16 32 64; do
  timeout 900 python bench.py --frames $fr --e2e-steps 0 --no-cpu-baseline > gpurun_out/bench_ts0_hd$fr.json 2>> gpurun_out/bench_ts.err
  IH_TABLE_SUM_MAX=1 timeout 900 python bench.py --frames $fr --e2e-steps 0 --no-cpu-baseline > gpurun_out/bench_ts1_hd$fr.json 2>> gpurun_out/bench_ts.err
done
echo done
