mkdir -p gpurun_out
(for v in 46 48 28 86 84; do for ry in 37 148 296; do IH_K4_VARIANT=$v IH_K4_ROWS_GRID=$ry timeout 600 python scripts/bench_queries.py 2>&1 | grep "k4_" | head -1 | sed "s/^/v$v ry$ry /"; done; done) > gpurun_out/queries_k4c.jsonl
echo done
