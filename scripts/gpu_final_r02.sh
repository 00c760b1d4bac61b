#!/bin/bash
# Round-2 final-code evidence in one box session: GPU suite + smoke, every
# BASELINE workload's bench line, the reference arm, per-GPU shares, the
# bench's ncu launch list and a --set full capture of k2_scan, the reference
# test suite against the drop-in.
set -u
TAG=${1:-r02m}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem --format=csv > $OUT/gpu.txt 2>&1
timeout 1800 python -m pytest tests -q -m gpu > $OUT/pytest_gpu.log 2>&1; echo pytest=$?; tail -1 $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo smoke=$?
python bench.py --csv $OUT/bench.csv > $OUT/bench_hd64.json 2> $OUT/bench_hd64.err; echo hd64=$?
python bench.py > $OUT/bench_hd64_b.json 2> $OUT/bench_hd64_b.err; echo hd64b=$?
python bench.py --workload 512 --csv $OUT/bench.csv > $OUT/bench_512.json 2> $OUT/bench_512.err; echo 512=$?
python bench.py --workload 4k128 --csv $OUT/bench.csv > $OUT/bench_4k128.json 2> $OUT/bench_4k128.err; echo 4k128=$?
python bench.py --workload 8k256 --steps 10 --csv $OUT/bench.csv > $OUT/bench_8k256.json 2> $OUT/bench_8k256.err; echo 8k256=$?
python bench.py --impl reference --steps 3 > $OUT/ref_hd64.json 2> $OUT/ref_hd64.err; echo ref=$?
for wl in hd64 4k128 8k256; do
  for n in 2 4 8; do
    python bench.py --workload $wl --share-of $n --steps 10 --e2e-steps 0 --no-cpu-baseline > $OUT/share_${wl}_${n}.json 2> $OUT/share_${wl}_${n}.err; echo share_${wl}_${n}=$?
  done
done
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches_hd64.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1; echo launches=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k2_scan -s 40 -c 1 -o $OUT/k2_scan_hd64 -f python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1; echo ncu_full=$?
python scripts/ncu_summary.py $OUT/k2_scan_hd64.ncu-rep > $OUT/k2_scan_hd64_summary.json 2>/dev/null
rm -f $OUT/k2_scan_hd64.ncu-rep
timeout 900 scripts/reftests/run.sh run $OUT/reftests > /dev/null 2>&1; echo reftests=$?
python3 - <<PY
import json, glob
for f in sorted(glob.glob("$OUT/*.json")):
    if "summary" in f: continue
    try: d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e: print(f, "ERR", e); continue
    sh = d.get("emulated_share", {})
    print(f.split("/")[-1], round(d.get("value", 0), 1), "step", round(d.get("hbm_frac_step", 0) or 0, 3),
          "scan", round((d.get("roofline") or {}).get("frac", 0) or 0, 3),
          "per_gpu", round(sh.get("per_gpu_hbm_frac_step", 0), 3) if sh else "",
          "e2e", round((d.get("e2e") or {}).get("value") or 0, 1), "clk", (d.get("clocks") or {}).get("sm_mhz"))
PY
du -sh $OUT
