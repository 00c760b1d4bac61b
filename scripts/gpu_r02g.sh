#!/bin/bash
# Round-2 final-code evidence: full GPU suite, smoke, sanitizers over every
# kernel path, hd64 bench + launch list + ncu --set full of k2_scan.
set -u
TAG=${1:-r02g}
OUT=gpurun_out/$TAG
mkdir -p $OUT
timeout 1800 python -m pytest tests -q -m gpu > $OUT/pytest_gpu.log 2>&1; echo pytest=$?; tail -1 $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo smoke=$?
for tool in memcheck racecheck synccheck; do
  timeout 1800 compute-sanitizer --tool $tool python scripts/sanitize_cases.py > $OUT/san_$tool.txt 2>&1; echo san_$tool=$?; tail -2 $OUT/san_$tool.txt
done
python bench.py > $OUT/bench_hd64.json 2> $OUT/bench_hd64.err; echo bench=$?
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches_hd64.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1; echo launches=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k2_scan -s 40 -c 1 -o $OUT/k2_scan_hd64 -f python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1; echo ncu_full=$?
python scripts/ncu_summary.py $OUT/k2_scan_hd64.ncu-rep > $OUT/k2_scan_hd64_summary.json 2>/dev/null
ncu -i $OUT/k2_scan_hd64.ncu-rep --page source --csv > $OUT/k2_scan_hd64_source.csv 2>/dev/null
rm -f $OUT/k2_scan_hd64.ncu-rep
du -sh $OUT
