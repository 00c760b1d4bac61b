#!/bin/bash
# Final-code check after the round-2 re-entry changes: GPU suite, smoke, the
# driver's bench command, reference arm, cfg1 line, launch list and an ncu
# --set full capture of k2_scan.
set -u
OUT=gpurun_out/r02q
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem --format=csv > $OUT/gpu.txt 2>&1
timeout 1200 python -m pytest tests -q -m gpu > $OUT/pytest_gpu.log 2>&1; echo pytest=$?; tail -1 $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo smoke=$?
timeout 600 python bench.py --gpus 1 --steps 20 --warmup 5 > $OUT/bench_hd64.json 2> $OUT/bench_hd64.err; echo hd64=$?
timeout 600 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > $OUT/ref_hd64.json 2> $OUT/ref_hd64.err; echo ref=$?
timeout 600 python bench.py --workload 512 > $OUT/bench_512.json 2> $OUT/bench_512.err; echo w512=$?
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches_hd64.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1; echo launches=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k2_scan -s 40 -c 1 -o $OUT/k2_scan_hd64 -f python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1; echo ncu_full=$?
python scripts/ncu_summary.py $OUT/k2_scan_hd64.ncu-rep > $OUT/k2_scan_hd64_summary.json 2>/dev/null; echo summary=$?
rm -f $OUT/k2_scan_hd64.ncu-rep
python scripts/launch_table.py $OUT/launches_hd64.csv > $OUT/launches_hd64_table.txt 2>&1
python3 - <<PY
import json, glob
for f in sorted(glob.glob("$OUT/bench*.json")) + ["$OUT/ref_hd64.json"]:
    try: d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e: print(f, "ERR", e); continue
    print(f.split("/")[-1], round(d.get("value", 0), 1), "step", round(d.get("hbm_frac_step", 0) or 0, 3),
          "scan", round((d.get("roofline") or {}).get("frac", 0) or 0, 3), "traffic", (d.get("roofline") or {}).get("traffic"),
          "e2e", round((d.get("e2e") or {}).get("value") or 0, 1), "clk", (d.get("clocks") or {}).get("sm_mhz"))
PY
cat $OUT/k2_scan_hd64_summary.json | head -12
