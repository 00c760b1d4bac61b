#!/bin/bash
# Full GPU suite, smoke and the three sanitizers over every kernel path.
OUT=gpurun_out/${1:-full}
mkdir -p $OUT
timeout 1800 python -m pytest tests -q -m gpu > $OUT/pytest_gpu.log 2>&1; echo pytest=$?; tail -1 $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo smoke=$?
for tool in memcheck racecheck synccheck; do
  timeout 1800 compute-sanitizer --tool $tool python scripts/sanitize_cases.py > $OUT/san_$tool.txt 2>&1; echo san_$tool=$?; tail -2 $OUT/san_$tool.txt
done
