#!/bin/bash
# Column-tile width x segment count sweep on the small per-GPU shares.
OUT=gpurun_out/${1:-tiles}
mkdir -p $OUT
for tc in 16 10 8 5 4; do
  for ns in 0 18 37 55 74; do
    if [ $ns = 0 ]; then unset IH_NSEG; else export IH_NSEG=$ns; fi
    IH_TILE_CHUNKS=$tc timeout 120 python scripts/graph_time.py 4k128/8 hd8 8k256/8 2>/dev/null | python3 -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); p=d['plan']
    print(json.dumps({'tc':$tc,'nseg_env':$ns,'wl':d['wl'],'ms':d['graph_ms_per_call'],'frac':d['frac'],'T':p['column_tiles'],'TW':p['tile_width'],'segs':p['segments'],'warps':p['warps_per_cta'],'slots':p['resident_ctas']}))"
  done
done > $OUT/sweep.jsonl
python3 - <<PY
import json
rows=[json.loads(l) for l in open("$OUT/sweep.jsonl")]
for wl in ("4k128/8","hd8","8k256/8"):
    best=sorted([r for r in rows if r["wl"]==wl], key=lambda r:r["ms"])[:6]
    for r in best: print(wl, r)
PY
