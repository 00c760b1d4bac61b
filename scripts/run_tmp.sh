mkdir -p gpurun_out
IH_STAGED_STORES=1 timeout 900 python -m pytest tests/test_parity_gpu.py -q -x -k "config_checksums or hd_64 or segments_and or tail or frames_batch or bin_slabs" > gpurun_out/pytest_stg.log 2>&1; echo pytest=$?
(for n in 3 5 9; do IH_NSEG=$n timeout 300 python scripts/graph_time.py hd64 | sed "s/^/base n$n /"; IH_NSEG=$n IH_STAGED_STORES=1 timeout 300 python scripts/graph_time.py hd64 | sed "s/^/stg2 n$n /"; IH_NSEG=$n IH_STAGED_STORES=1 IH_ROWS_PER_BATCH=1 timeout 300 python scripts/graph_time.py hd64 | sed "s/^/stg1 n$n /"; done
timeout 300 python scripts/graph_time.py hd8 hd1 | sed "s/^/base /"; IH_STAGED_STORES=1 timeout 300 python scripts/graph_time.py hd8 hd1 | sed "s/^/stg2 /") > gpurun_out/graph_stg.jsonl 2>&1
echo done
