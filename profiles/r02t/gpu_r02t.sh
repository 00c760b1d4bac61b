#!/bin/bash
# ncu --set full summaries of the final code's default query kernels
# (K3 region histograms, K4 quads, K5 chain) and their timings.
set -u
OUT=gpurun_out/r02t
mkdir -p $OUT
python scripts/bench_queries.py > $OUT/queries.jsonl 2>&1; echo queries=$?
prof() {  # name kernel-regex args...
  local name=$1 re=$2; shift 2
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"$re" -s 1 -c 1 \
    -o $OUT/$name -f python scripts/kernels_once.py "$@" > $OUT/$name.log 2>&1
  echo "$name=$?"
  python scripts/ncu_summary.py $OUT/$name.ncu-rep > $OUT/${name}_summary.json 2>/dev/null
  rm -f $OUT/$name.ncu-rep
}
prof k3_full256 'k3_region_histograms' k3full
prof k4_quads 'k4_window_counts_quads' k4
prof k5_chain 'k5_likelihood_map_chain' k5
for f in $OUT/*_summary.json; do python3 -c "
import json,sys; d=json.load(open('$f')); d=d[0] if isinstance(d,list) else d
print('$f'.split('/')[-1], d.get('Kernel Name','')[:60], d.get('gpu__time_duration.sum'), d.get('dram__bytes_read.sum'), d.get('dram__bytes_write.sum'), d.get('gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed'))"; done
