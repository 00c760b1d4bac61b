#!/bin/bash
# Per-kernel ncu captures (one --set full report per non-K2 kernel) plus the
# random-gather ceiling probe.  Outputs under gpurun_out/<tag>/.
set -u
TAG=${1:-r02b}
OUT=gpurun_out/$TAG
mkdir -p $OUT
make -s -C scripts/probes > /dev/null 2>&1
timeout 300 scripts/probes/gather_probe > $OUT/gather_probe.jsonl 2>&1; echo gather=$?
python scripts/bench_queries.py > $OUT/queries.jsonl 2>&1; echo queries=$?
python scripts/bench_scan.py > $OUT/scan_kernels.jsonl 2>&1; echo scans=$?
prof() {  # name kernel-regex args...
  local name=$1 re=$2; shift 2
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"$re" -s 1 -c 1 \
    -o $OUT/$name -f python scripts/kernels_once.py "$@" > $OUT/$name.log 2>&1
  echo "$name=$?"
  python scripts/ncu_summary.py $OUT/$name.ncu-rep > $OUT/${name}_summary.json 2>/dev/null
  # reports are large and gpurun copies back <= 64 MiB: keep only the summary
  # (and the raw page as CSV) unless KEEP_REPS names this capture
  ncu -i $OUT/$name.ncu-rep --page raw --csv > $OUT/${name}_raw.csv 2>/dev/null
  case " ${KEEP_REPS:-} " in *" $name "*) ;; *) rm -f $OUT/$name.ncu-rep ;; esac
}
prof k1_rowscan 'k1_rowscan' k1
prof k1b_colscan 'k1b_colscan' k1
prof k3_shard32 'k3_region' k3
prof k3_full256 'k3_region' k3full
prof k4_pairs 'k4_window' k4
prof k5_map 'k5_likelihood' k5
prof k6_block_totals 'k6_block_totals' k6
prof k6_scan_apply 'k6_scan_apply' k6
prof k6_scan_inner 'k6_scan_inner' k6
prof k6_scan_strided 'k6_scan_strided' k6
prof k6_transpose 'k6_transpose' k6
prof k7_wavefront 'k7_wavefront' k7
rm -f $OUT/*.ncu-rep.tmp
