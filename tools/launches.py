"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
hdr, agg = None, defaultdict(list)
for r in rows:
    if 'Kernel Name' in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        agg[d['Kernel Name'].split('(')[0][:48]].append(float(d['Metric Value']))
tot = 0.0
for k, v in agg.items():
    a = sum(v) / len(v) / 1e3
    tot += sum(v) / 1e3 / steps
    print(f"{k:48s} n={len(v):4d} avg={a:9.1f} us  per-step={sum(v)/1e3/steps:9.1f} us")
print(f"sum per step {tot:.1f} us")
