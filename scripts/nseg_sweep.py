"""Segment-count sweep (CUDA-graph timed calls) for the planner's many-units
regime: prints the heuristic's choice and the best count per workload."""
import json, os, subprocess, sys
wls = sys.argv[1:]
here = os.path.dirname(os.path.abspath(__file__))
for wl in wls:
    res = {}
    for n in [0] + list(range(1, 13)) + [14, 16, 18, 20, 24, 28, 32, 37]:
        env = dict(os.environ, IH_NSEG=str(n)) if n else dict(os.environ)
        env.pop("IH_NSEG", None) if not n else None
        out = subprocess.run([sys.executable, os.path.join(here, "graph_time.py"), wl], env=env,
                             capture_output=True, text=True).stdout
        d = json.loads(out.strip().splitlines()[-1])
        res[n] = (d["plan"]["segments"], d["graph_ms_per_call"], d["frac"])
    heur = res[0]
    best = min((v for k, v in res.items() if k), key=lambda v: v[1])
    print(json.dumps({"wl": wl, "heuristic": heur, "best": best,
                      "all": {str(k): [v[0], round(v[2], 3)] for k, v in res.items() if k}}), flush=True)
