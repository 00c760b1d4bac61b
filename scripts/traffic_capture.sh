#!/bin/bash
# ncu DRAM bytes of k2_scan per workload and row-segment count (the autotuner
# picks the count at run time; bench.py reports traffic only for a captured
# plan).  Output: gpurun_out/<tag>/traffic.jsonl (one line per capture).
set -u
TAG=${1:-r02c}
OUT=gpurun_out/$TAG
mkdir -p $OUT
cap() {  # workload nseg
  local wl=$1 n=$2 f=$OUT/traffic_${1//\//_}_$2.csv
  IH_NSEG=$n timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
    --clock-control none -k regex:k2_scan -s 1 -c 1 --csv --log-file $f python scripts/one.py $wl > /dev/null 2>&1
  python - "$wl" "$n" "$f" >> $OUT/traffic.jsonl <<'PY'
import csv, json, sys
wl, n, f = sys.argv[1], int(sys.argv[2]), sys.argv[3]
rows = [r for r in csv.reader(open(f)) if len(r) > 10]
h = rows[0]; m = {}
for r in rows[1:]:
    m[r[h.index("Metric Name")]] = (float(r[h.index("Metric Value")].replace(",", "")), r[h.index("Metric Unit")])
def b(k):
    v, u = m[k]; return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
print(json.dumps({"wl": wl, "segments": n, "dram_read": b("dram__bytes_read.sum"),
                  "dram_write": b("dram__bytes_write.sum"), "time": m["gpu__time_duration.sum"]}))
PY
}
for n in 3 4 5 6 7 9; do cap hd64 $n; done
for n in 12 18 24; do cap 4k128 $n; done
for n in 8 12 16; do cap 8k256 $n; done
for n in 32 64; do cap 512 $n; done
