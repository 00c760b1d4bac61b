#!/bin/bash
# Regenerate the round-1 evidence on one B200 (under gpurun: outputs land in
# gpurun_out/repro/; copy what you want to keep into profiles/).
#   /usr/local/graft/bin/gpurun --timeout 3000 -- 'bash scripts/reproduce_round1.sh'
set -u
O=gpurun_out/repro
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo build=$?
timeout 1500 python -m pytest tests -q -m gpu > $O/pytest_gpu.log 2>&1; echo pytest=$?
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke=$?
# headline line (cfg2) and the reference arm on the same box
timeout 900 python bench.py > $O/bench_hd64.json 2> $O/bench.err; echo bench=$?
timeout 600 python bench.py --impl reference > $O/bench_reference.json 2>> $O/bench.err; echo ref=$?
# cfg3 / cfg4 lines and the per-GPU shares of the N = 2/4/8 frame-sharded run
timeout 900 python bench.py --workload 4k128 > $O/bench_4k128.json 2>> $O/bench.err
timeout 1200 python bench.py --workload 8k256 > $O/bench_8k256.json 2>> $O/bench.err
for fr in 32 16 8; do
  timeout 900 python bench.py --frames $fr --e2e-steps 0 --no-cpu-baseline > $O/bench_hd$fr.json 2>> $O/bench.err
done
# query kernels, graph-timed sweeps
timeout 600 python scripts/bench_queries.py > $O/queries.jsonl 2>&1
timeout 900 python scripts/graph_time.py hd64 hd8 hd1 512 4k128 4k128/8 8k256/8 > $O/graph_time.jsonl 2>&1
# ncu: launch list of the bench command + one full capture of the scan kernel
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $O/launches_bench.csv python bench.py --steps 10 --warmup 3 --e2e-steps 0 \
  --no-cpu-baseline --no-autotune > /dev/null 2>&1; echo ncu_launches=$?
IH_NSEG=5 timeout 400 ncu --set full --clock-control none --import-source on \
  -k regex:"k2_scan|k2_colcounts_all" -s 6 -c 2 -o $O/prof_hd64 -f \
  python bench.py --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline --no-autotune \
  > /dev/null 2>&1; echo ncu_full=$?
python scripts/ncu_summary.py $O/prof_hd64.ncu-rep > $O/ncu_full_hd64.json 2>/dev/null
# sanitizers over every kernel path
for tool in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $tool python scripts/sanitize_cases.py > $O/san_$tool.txt 2>&1
done
echo done
