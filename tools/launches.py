import csv, sys
from collections import OrderedDict
f = sys.argv[1] if len(sys.argv) > 1 else 'gpurun_out/launches.csv'
rows = list(csv.reader(open(f)))
hdr = [i for i, r in enumerate(rows) if 'Kernel Name' in r][0]
h = rows[hdr]; ki = h.index('Kernel Name'); vi = h.index('Metric Value')
agg = OrderedDict()
for r in rows[hdr + 1:]:
    try:
        agg.setdefault(r[ki].split('(')[0][:60], []).append(float(r[vi].replace(',', '')))
    except Exception:
        pass
tot = sum(sum(v) for v in agg.values())
for k, v in agg.items():
    print(f"{len(v):3d} x {sum(v)/len(v)/1e6:9.3f} ms  total {sum(v)/1e6:9.3f} ms ({100*sum(v)/tot:5.1f}%)  {k}")
