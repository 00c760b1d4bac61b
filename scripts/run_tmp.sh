mkdir -p gpurun_out
(for tc in 16 2 1; do for n in 8 16 32; do IH_TILE_CHUNKS=$tc IH_NSEG=$n IH_MIN_SEG_ROWS=8 timeout 300 python scripts/graph_time.py 512 | sed "s/^/tc$tc n$n /"; done; done
for tc in 16 4 2; do IH_TILE_CHUNKS=$tc timeout 300 python scripts/graph_time.py hd1 | sed "s/^/tc$tc /"; done) > gpurun_out/small_tc.jsonl 2>&1
echo done
