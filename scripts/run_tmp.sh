mkdir -p gpurun_out
timeout 1200 python -m pytest tests/ -q -x -m gpu > gpurun_out/pytest_ck.log 2>&1; echo pytest=$?
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_ck.log 2>&1; echo smoke=$?
timeout 900 python bench.py > gpurun_out/bench_ck.json 2> gpurun_out/bench_ck.err; echo bench=$?
timeout 600 python bench.py --impl reference > gpurun_out/bench_ck_ref.json 2>> gpurun_out/bench_ck.err; echo ref=$?
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_ck.csv python bench.py --steps 10 --warmup 3 --e2e-steps 0 --no-cpu-baseline --no-autotune > /dev/null 2>&1; echo ncul=$?
IH_NSEG=5 timeout 400 ncu --set full --clock-control none --import-source on -k regex:"k2_scan|k2_colcounts_all" -s 6 -c 2 -o gpurun_out/prof_ck -f python bench.py --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline --no-autotune > /dev/null 2>&1; echo ncuf=$?
echo done
