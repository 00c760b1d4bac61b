#!/bin/bash
# Per-kernel times and DRAM bytes of B = 1 / 2 / 4 HD x 64 calls (the < 4-bin gap).
OUT=gpurun_out/${1:-smallbins}
mkdir -p $OUT
for wl in hd64b1 hd64b2 hd64b4; do
  timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__warps_active.avg.pct_of_peak_sustained_active,launch__grid_size,launch__occupancy_limit_registers,launch__registers_per_thread \
    --clock-control none -s 6 -c 9 --csv --log-file $OUT/$wl.csv python scripts/one.py $wl > /dev/null 2>&1; echo $wl=$?
done
python - $OUT <<'PY'
import csv, sys, glob, os, collections
for f in sorted(glob.glob(sys.argv[1] + "/*.csv")):
    rows = [r for r in csv.reader(open(f)) if len(r) > 10]
    h = rows[0]; agg = collections.OrderedDict()
    for r in rows[1:]:
        k = (r[h.index("ID")], r[h.index("Kernel Name")][:40])
        agg.setdefault(k, {})[r[h.index("Metric Name")]] = r[h.index("Metric Value")] + " " + r[h.index("Metric Unit")]
    print("==", os.path.basename(f))
    for (i, n), m in agg.items():
        print(f"  {i:>3} {n:40s}", {k.split('__')[1][:28]: v for k, v in m.items()})
PY
