"""Summarise an ncu --csv launch list (gpu__time_duration.sum) per kernel name."""
import csv, collections, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = None
agg = collections.OrderedDict()
for r in rows:
    if r and r[0] == 'ID':
        hdr = r
        continue
    if hdr is None or len(r) < len(hdr):
        continue
    d = dict(zip(hdr, r))
    if d.get('Metric Name') != 'gpu__time_duration.sum':
        continue
    name = d['Kernel Name'].split('(')[0][-60:]
    v = float(d['Metric Value'].replace(',', ''))
    unit = d['Metric Unit']
    scale = {'nsecond': 1e-6, 'ns': 1e-6, 'usecond': 1e-3, 'us': 1e-3, 'msecond': 1.0, 'ms': 1.0}.get(unit, 1e-6)
    agg.setdefault(name, [0.0, 0])
    agg[name][0] += v * scale
    agg[name][1] += 1
tot = sum(v for v, _ in agg.values())
for k, (v, n) in agg.items():
    print(f"{v:10.3f} ms  x{n:<4d} {k}")
print(f"{tot:10.3f} ms  total")
