mkdir -p gpurun_out
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_fin_4k128.csv python bench.py --workload 4k128 --steps 5 --warmup 3 --e2e-steps 0 --no-cpu-baseline > /dev/null 2>&1; echo a=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_fin_8k256.csv python bench.py --workload 8k256 --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline > /dev/null 2>&1; echo b=$?
timeout 400 ncu --set full --clock-control none --import-source on -k regex:"k2_scan|k2_rowleft|k2_colcounts_all|k2_colprefix" -c 4 -o gpurun_out/prof_fin_4k128 -f python scripts/one.py 4k128 > /dev/null 2>&1; echo c=$?
timeout 600 python scripts/bench_queries.py > gpurun_out/queries_fin.jsonl 2>&1; echo d=$?
