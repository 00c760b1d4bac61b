#!/bin/bash
# Steady-state per-GPU shares (--steps 100: the pipelined steps' fill and
# drain amortised) and the driver's own N = 1 command on the final code.
set -u
OUT=gpurun_out/r02p
mkdir -p $OUT
python bench.py --gpus 1 --steps 20 --warmup 5 > $OUT/bench_driver_cmd.json 2> $OUT/bench_driver_cmd.err; echo drv=$?
for wl in hd64 4k128 8k256; do
  for n in 2 4 8; do
    python bench.py --workload $wl --share-of $n --steps 100 --e2e-steps 0 --no-cpu-baseline > $OUT/share_${wl}_${n}.json 2> $OUT/share_${wl}_${n}.err; echo share_${wl}_${n}=$?
  done
done
python bench.py --workload 4k128 --steps 100 --e2e-steps 1 > $OUT/bench_4k128.json 2> $OUT/bench_4k128.err; echo 4k=$?
python3 - <<PY
import json, glob
for f in sorted(glob.glob("$OUT/*.json")):
    try: d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e: print(f, "ERR", e); continue
    sh = d.get("emulated_share", {}); a = d.get("autotune") or {}
    print(f.split("/")[-1], round(d.get("value", 0), 1), "ms", round(d.get("ms_per_step", 0), 4), "step", round(d.get("hbm_frac_step", 0) or 0, 3),
          "scan", round((d.get("roofline") or {}).get("frac", 0) or 0, 3), "refine", a.get("pipelined_refine_ms"), "clk", (d.get("clocks") or {}).get("sm_mhz"))
PY
