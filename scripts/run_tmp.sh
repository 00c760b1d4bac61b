mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py -q -x -k "likelihood or variants or window" > gpurun_out/pytest_k5.log 2>&1; echo pytest=$?
(timeout 600 python scripts/bench_queries.py 2>&1 | grep "k5_"; IH_K5_DIRECT=1 timeout 600 python scripts/bench_queries.py 2>&1 | grep "k5_") > gpurun_out/queries_k5tab.jsonl
echo done
