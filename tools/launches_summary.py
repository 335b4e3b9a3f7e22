import csv, sys
from collections import defaultdict
rows = list(csv.reader(open(sys.argv[1] if len(sys.argv) > 1 else 'gpurun_out/launches.csv')))
hdr = None; agg = defaultdict(list)
for r in rows:
    if r and r[0] == 'ID': hdr = r; continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d.get('Metric Name') == 'gpu__time_duration.sum':
            agg[d['Kernel Name'][:70]].append(float(d['Metric Value']))
tot = 0
for n, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
    print(f"{sum(v)/len(v)/1000:9.1f} us avg x{len(v):4d}  {n}")
