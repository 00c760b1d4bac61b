import csv, sys
from collections import defaultdict
for path in sys.argv[1:]:
    rows = list(csv.reader(open(path)))
    hdr = [i for i, r in enumerate(rows) if 'Kernel Name' in r][0]
    h = rows[hdr]; ki = h.index('Kernel Name'); vi = h.index('Metric Value'); gi = h.index('Grid Size'); bi = h.index('Block Size')
    agg = defaultdict(list); meta = {}
    for r in rows[hdr + 1:]:
        k = r[ki].split('(')[0].replace('void ', '')
        agg[k].append(float(r[vi])); meta[k] = (r[gi], r[bi])
    print(path.split('/')[-1])
    for k, v in agg.items():
        print(f"   {k:40s} n={len(v):3d} avg={sum(v)/len(v)/1e3:9.2f} us  grid={meta[k][0]} block={meta[k][1]}")
