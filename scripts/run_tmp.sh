mkdir -p gpurun_out
for tc in 16 8 4; do
  IH_TILE_CHUNKS=$tc timeout 600 python scripts/graph_time.py 512 hd1 hd8 hd64 4k128 4k128/8 8k256/8 > gpurun_out/graph_tc$tc.jsonl 2>&1
done
for n in 17 34 68; do IH_MIN_SEG_ROWS=8 IH_NSEG=$n timeout 300 python scripts/graph_time.py hd1 >> gpurun_out/graph_hd1_nseg.jsonl 2>&1; done
IH_TILE_CHUNKS=4 IH_PYTEST_QUICK=1 timeout 600 python -m pytest tests/test_parity_gpu.py -q -x -k "column_tiles or segments_and or config_checksums" > gpurun_out/pytest_tc4.log 2>&1; echo pytest=$?
echo done
