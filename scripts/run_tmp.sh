mkdir -p gpurun_out
for i in 1 2 3; do timeout 900 python bench.py --e2e-steps 0 --no-cpu-baseline > gpurun_out/bench_v$i.json 2>> gpurun_out/bench_v.err; done
for i in 1 2; do IH_NSEG=5 timeout 900 python bench.py --e2e-steps 0 --no-cpu-baseline --no-autotune > gpurun_out/bench_v5_$i.json 2>> gpurun_out/bench_v.err; done
for i in 1 2; do IH_NSEG=3 timeout 900 python bench.py --e2e-steps 0 --no-cpu-baseline --no-autotune > gpurun_out/bench_v3_$i.json 2>> gpurun_out/bench_v.err; done
nvidia-smi --query-gpu=name,serial,pci.bus_id,clocks.max.mem,memory.total --format=csv > gpurun_out/gpuinfo.txt
echo done
