#!/bin/bash
# Last check of the round's final code: GPU suite, smoke, the driver's bench
# command and reference arm, cfg1 line and its host-overhead breakdown, and
# the --gpus 2 refusal on a one-GPU box.
set -u
OUT=gpurun_out/r02r
mkdir -p $OUT
timeout 1200 python -m pytest tests -q -m gpu > $OUT/pytest_gpu.log 2>&1; echo pytest=$?; tail -1 $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo smoke=$?
timeout 600 python bench.py --gpus 1 --steps 20 --warmup 5 > $OUT/bench_hd64.json 2> $OUT/bench_hd64.err; echo hd64=$?
timeout 600 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > $OUT/ref_hd64.json 2> $OUT/ref_hd64.err; echo ref=$?
timeout 600 python bench.py --workload 512 > $OUT/bench_512.json 2> $OUT/bench_512.err; echo w512=$?
timeout 300 python scripts/eager_breakdown.py > $OUT/eager_breakdown.jsonl 2>&1; echo eager=$?
timeout 120 python bench.py --gpus 2 --steps 3 --warmup 3 > $OUT/gpus2.out 2>&1; echo gpus2=$?
tail -2 $OUT/gpus2.out
cat $OUT/eager_breakdown.jsonl
python3 - <<PY
import json
for f in ["$OUT/bench_hd64.json", "$OUT/ref_hd64.json", "$OUT/bench_512.json"]:
    d = json.loads(open(f).read().strip().splitlines()[-1])
    print(f.split("/")[-1], round(d.get("value", 0), 1), "step", round(d.get("hbm_frac_step", 0) or 0, 3),
          "scan", round((d.get("roofline") or {}).get("frac", 0) or 0, 3),
          "e2e", round((d.get("e2e") or {}).get("value") or 0, 1), "eager", d.get("eager"), "clk", (d.get("clocks") or {}).get("sm_mhz"))
PY
