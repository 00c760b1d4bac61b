#!/bin/bash
# Skewed segments A/B: parity, graph-timed one-wave / two-wave grids, shares.
set -u
TAG=${1:-skew}
OUT=gpurun_out/$TAG
mkdir -p $OUT
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_fuzz_gpu.py -q -x -k "skew or fuzz" > $OUT/pytest.log 2>&1; echo pytest=$?; tail -1 $OUT/pytest.log
for sk in 0 110 120 130 140 150; do
  IH_SKEW_X100=$sk IH_NSEG=37 timeout 120 python scripts/graph_time.py 4k128/8 > $OUT/g_4k8_$sk.jsonl 2>&1
  IH_SKEW_X100=$sk IH_NSEG=37 timeout 120 python scripts/graph_time.py 4k128/4 > $OUT/g_4k4_$sk.jsonl 2>&1
  IH_SKEW_X100=$sk IH_NSEG=9 timeout 120 python scripts/graph_time.py hd8 > $OUT/g_hd8_$sk.jsonl 2>&1
  IH_SKEW_X100=$sk IH_NSEG=12 timeout 120 python scripts/graph_time.py 8k256/8 > $OUT/g_8k8_$sk.jsonl 2>&1
done
python3 - <<PY
import json
for wl in ("4k8","4k4","hd8","8k8"):
    row=[]
    for sk in (0,110,120,130,140,150):
        d=[json.loads(l) for l in open(f"$OUT/g_{wl}_{sk}.jsonl") if l.startswith("{")][0]
        row.append(f"{sk}:{d['graph_ms_per_call']:.4f}({d['frac']:.3f})")
    print(wl, " ".join(row))
PY
for wl in 4k128 hd64 8k256; do
  python bench.py --workload $wl --share-of 8 --steps 10 --e2e-steps 0 --no-cpu-baseline > $OUT/share_${wl}_8.json 2> $OUT/share_${wl}_8.err
  python3 -c "
import json; d=json.load(open('$OUT/share_${wl}_8.json')); print('$wl/8', round(d['value']), 'per_gpu', round(d['emulated_share']['per_gpu_hbm_frac_step'],3), 'scan', round(d['roofline']['frac'],3), d['autotune']['segments'], d['autotune'].get('skew'), d['autotune']['tail_div'])"
done
