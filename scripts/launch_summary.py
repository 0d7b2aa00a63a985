"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list per kernel name."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = None
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows:
    if 'Kernel Name' in r:
        h = r
        continue
    if h is None or len(r) != len(h):
        continue
    d = dict(zip(h, r))
    if d.get('Metric Name') != 'gpu__time_duration.sum':
        continue
    n = d['Kernel Name'].split('(')[0][:60]
    unit = d.get('Metric Unit', 'ns')
    v = float(d['Metric Value'].replace(',', ''))
    v *= {'ns': 1.0, 'us': 1e3, 'usecond': 1e3, 'ms': 1e6, 'msecond': 1e6, 'nsecond': 1.0}.get(unit, 1.0)
    agg[n][0] += 1
    agg[n][1] += v
tot = sum(t for _, t in agg.values())
for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k:60s} {c:5d} {t / 1e6:9.3f} ms  avg {t / c / 1e3:8.1f} us  {100 * t / tot:5.1f}%")
