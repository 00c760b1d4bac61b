# K4 timing: modes 3/4, rows-grid density (IH_K4_CTAS_PER_SM)
mkdir -p gpurun_out/k4s
for m in ${K4_MODES:-3 4}; do for c in ${K4_CPS:-64 128 256 512}; do
  IH_K4_MODE=$m IH_K4_CTAS_PER_SM=$c python scripts/bench_queries.py 2>&1 | grep k4_window | sed "s/^/{\"cps\": $c, \"mode\": $m, \"r\": /;s/$/}/"
done; done > gpurun_out/k4s/sweep.jsonl
