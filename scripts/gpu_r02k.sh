#!/bin/bash
# Bin pairs (KB=2) as the default for >= 24 bins on wide aligned rows:
# full GPU suite, autotuner's kb stage, same-box bench A/B against IH_KB=4
# (N=1 and the 4-/8-GPU shares), k2_scan DRAM bytes per segment count.
set -u
TAG=${1:-r02k}
OUT=gpurun_out/$TAG
mkdir -p $OUT
timeout 1800 python -m pytest tests -q -m gpu > $OUT/pytest_gpu.log 2>&1; echo pytest=$?; tail -1 $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo smoke=$?
timeout 600 python - > $OUT/autotune_kb.jsonl 2>&1 <<'PY'
import json
from paper_1711_01919_b200 import device
for f, h, w, b in ((64, 1080, 1920, 32), (16, 1080, 1920, 32), (8, 1080, 1920, 32), (64, 900, 1600, 64), (64, 512, 512, 32)):
    r = device.autotune(f, h, w, b, objective="scan")
    print(json.dumps({"shape": [f, h, w, b], "default_kb": device.plan(f, h, w, b)["bins_per_cta"], **r}), flush=True)
PY
echo autotune=$?
for rep in 1 2; do
  for kb in 0 4; do
    env $([ $kb != 0 ] && echo IH_KB=$kb) python bench.py > $OUT/bench_kb${kb}_$rep.json 2> $OUT/bench_kb${kb}_$rep.err; echo bench_kb$kb=$?
  done
done
for n in 2 4 8; do
  for kb in 0 4; do
    env $([ $kb != 0 ] && echo IH_KB=$kb) python bench.py --share-of $n --no-cpu-baseline --e2e-steps 0 > $OUT/share${n}_kb$kb.json 2> $OUT/share${n}_kb$kb.err; echo share${n}_kb$kb=$?
  done
done
cap() {  # nseg
  local n=$1 f=$OUT/traffic_hd64_kb2_$1.csv
  IH_KB=2 IH_NSEG=$n timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
    --clock-control none -k regex:k2_scan -s 1 -c 1 --csv --log-file $f python scripts/one.py hd64 > /dev/null 2>&1
  python - "$n" "$f" >> $OUT/traffic.jsonl <<'PY'
import csv, json, sys
n, f = int(sys.argv[1]), sys.argv[2]
rows = [r for r in csv.reader(open(f)) if len(r) > 10]
h = rows[0]; m = {}
for r in rows[1:]:
    m[r[h.index("Metric Name")]] = (float(r[h.index("Metric Value")].replace(",", "")), r[h.index("Metric Unit")])
def b(k):
    v, u = m[k]; return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
print(json.dumps({"wl": "hd64", "kb": 2, "segments": n, "dram_read": b("dram__bytes_read.sum"),
                  "dram_write": b("dram__bytes_write.sum"), "time": m["gpu__time_duration.sum"]}))
PY
}
for n in 3 4 5 6 7 9; do cap $n; done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k2_scan -s 40 -c 1 -o $OUT/k2_scan_hd64 -f python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1; echo ncu_full=$?
python scripts/ncu_summary.py $OUT/k2_scan_hd64.ncu-rep > $OUT/k2_scan_hd64_summary.json 2>/dev/null
rm -f $OUT/k2_scan_hd64.ncu-rep
du -sh $OUT
