"""Which CTAs of a one-wave k2_scan grid form the tail?  Per segment index
(the slowest grid dimension = dispatch order): median CTA end time, and per
SM the order of its two CTAs.  usage: tail_order.py WORKLOAD"""
import json, os, subprocess, sys, tempfile
import numpy as np
wl = sys.argv[1]
f = tempfile.mktemp(suffix=".npy")
env = dict(os.environ, TRACE_OUT=f)
subprocess.run([sys.executable, os.path.join(os.path.dirname(__file__), "cta_timeline.py"), wl],
               env=env, check=True, capture_output=True)
tr = np.load(f).astype(np.float64)  # [cta] = start, ready, end, smid ; cta = linear block index
n = len(tr)
t0 = tr[:, 0].min()
end = (tr[:, 2] - t0) / 1e3
start = (tr[:, 0] - t0) / 1e3
units = int(sys.argv[2]) if len(sys.argv) > 2 else 8
seg = np.arange(n) // units
res = {"wl": wl, "ctas": n, "end_by_segment_median_us": [round(float(np.median(end[seg == s])), 1) for s in range(seg.max() + 1)]}
# per SM: the two CTAs' linear indices and ends
sm = tr[:, 3].astype(int)
pairs = []
for m in np.unique(sm):
    idx = np.where(sm == m)[0]
    if len(idx) == 2:
        a, b = idx[np.argsort(start[idx])]
        pairs.append((int(a), int(b), float(end[a]), float(end[b])))
first_done_older = np.mean([ea < eb for a, b, ea, eb in pairs]) if pairs else None
res["pairs"] = len(pairs)
res["older_finishes_first_frac"] = first_done_older
res["lower_index_is_older_frac"] = float(np.mean([a < b for a, b, ea, eb in pairs])) if pairs else None
res["end_lower_half_idx_median"] = float(np.median(end[: n // 2]))
res["end_upper_half_idx_median"] = float(np.median(end[n // 2:]))
print(json.dumps(res))
