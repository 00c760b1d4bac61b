mkdir -p gpurun_out
timeout 900 python -m pytest tests/ -q -x -m gpu > gpurun_out/pytest_ct6.log 2>&1; echo pytest=$?
timeout 900 python scripts/sweep2.py 'hd64' 'hd32' 'hd16' 'hd8' 'hd1' '512' '4k128' '4k128/2' '4k128/4' '4k128/8' '8k256/8' '8k256' > gpurun_out/sweep_ct6.jsonl 2>&1; echo sweep=$?
timeout 600 python bench.py > gpurun_out/bench_ct6_hd64.json 2> gpurun_out/bench_ct6_hd64.err; echo bench=$?
timeout 600 python bench.py --workload 4k128 > gpurun_out/bench_ct6_4k128.json 2> gpurun_out/bench_ct6_4k128.err; echo bench4k=$?
timeout 900 python bench.py --workload 8k256 > gpurun_out/bench_ct6_8k256.json 2> gpurun_out/bench_ct6_8k256.err; echo bench8k=$?
