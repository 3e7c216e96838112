"""Aggregate an ncu launch list (gpu__time_duration.sum CSV) per kernel."""
import csv, collections, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = None; agg = collections.OrderedDict()
for r in rows:
    if 'Kernel Name' in r: hdr = r; continue
    if hdr is None or len(r) != len(hdr): continue
    d = dict(zip(hdr, r))
    if d.get('Metric Name') != 'gpu__time_duration.sum': continue
    k = d['Kernel Name'][:90]; v = float(d['Metric Value'])
    a = agg.setdefault(k, [0, 0.0]); a[0] += 1; a[1] += v
tot = sum(v[1] for v in agg.values())
div = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
print(f"{'launches':>8} {'us/step':>10} {'share':>6}  kernel   (steps={div:g})")
for k, (c, v) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{c:8d} {v/1e3/div:10.1f} {100*v/tot:5.1f}%  {k}")
print(f"total {tot/1e3/div:.1f} us/step")
