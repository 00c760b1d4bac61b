mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py -q -x -k "variants or window or likelihood or small_case_queries" > gpurun_out/pytest_q.log 2>&1; echo pytest=$?
(timeout 600 python scripts/bench_queries.py 2>&1 | grep "k4_\|k5_"
for ry in 8 32 128 1017; do IH_K4_ROWS_GRID=$ry IH_K5_ROWS_GRID=$ry timeout 600 python scripts/bench_queries.py 2>&1 | grep "k4_\|k5_" | sed "s/^/ry$ry /"; done) > gpurun_out/queries_k4ry.jsonl
echo done
