#!/bin/bash
# Round-2 bench evidence: every BASELINE workload's line, the reference arm,
# and rank-0 per-GPU shares of 2/4/8-GPU runs (one GPU here).
set -u
TAG=${1:-r02e}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem --format=csv > $OUT/gpu.txt 2>&1
python bench.py --csv $OUT/bench.csv > $OUT/bench_hd64.json 2> $OUT/bench_hd64.err; echo hd64=$?
python bench.py --workload 512 --csv $OUT/bench.csv > $OUT/bench_512.json 2> $OUT/bench_512.err; echo 512=$?
python bench.py --workload 4k128 --csv $OUT/bench.csv > $OUT/bench_4k128.json 2> $OUT/bench_4k128.err; echo 4k128=$?
python bench.py --workload 8k256 --steps 10 --csv $OUT/bench.csv > $OUT/bench_8k256.json 2> $OUT/bench_8k256.err; echo 8k256=$?
python bench.py --impl reference --steps 3 > $OUT/ref_hd64.json 2> $OUT/ref_hd64.err; echo ref=$?
for wl in hd64 4k128 8k256; do
  for n in 2 4 8; do
    python bench.py --workload $wl --share-of $n --steps 10 --e2e-steps 0 --no-cpu-baseline > $OUT/share_${wl}_${n}.json 2> $OUT/share_${wl}_${n}.err; echo share_${wl}_${n}=$?
  done
done
python3 - <<PY
import json, glob
for f in sorted(glob.glob("$OUT/*.json")):
    try: d = json.load(open(f))
    except Exception as e: print(f, "ERR", e); continue
    sh = d.get("emulated_share", {})
    print(f.split("/")[-1], round(d["value"], 1), "step", round(d.get("hbm_frac_step", 0) or 0, 3),
          "scan", round(d.get("roofline", {}).get("frac", 0) or 0, 3),
          "per_gpu", round(sh.get("per_gpu_hbm_frac_step", 0), 3) if sh else "",
          "e2e", round((d.get("e2e") or {}).get("value") or 0, 1), "clk", d.get("clocks", {}).get("sm_mhz"))
PY
