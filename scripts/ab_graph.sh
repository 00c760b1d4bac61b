#!/bin/bash
# Same-box A/B of graph-timed calls: ab/old (a build of an earlier commit) vs
# this tree, alternating, twice.  Usage: scripts/ab_graph.sh TAG wl...
TAG=$1; shift
OUT=gpurun_out/$TAG
mkdir -p $OUT
for rep in 1 2; do
  (cd ab/old && python scripts/graph_time.py "$@") > $OUT/old_$rep.jsonl 2>&1
  python scripts/graph_time.py "$@" > $OUT/new_$rep.jsonl 2>&1
done
python3 - $OUT <<'PY'
import json, sys, collections
r = collections.defaultdict(dict)
for arm in ("old", "new"):
    for rep in (1, 2):
        for l in open(f"{sys.argv[1]}/{arm}_{rep}.jsonl"):
            if l.startswith("{"):
                d = json.loads(l); r[d["wl"]].setdefault(arm, []).append(d["graph_ms_per_call"] * 1000)
for wl, v in r.items():
    print(f"{wl:10s} old {min(v['old']):9.1f} us  new {min(v['new']):9.1f} us  ({min(v['new'])/min(v['old']):.3f})")
PY
