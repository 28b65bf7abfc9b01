"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list per kernel."""
import collections, csv, sys
rows = list(csv.reader(open(sys.argv[1])))
start = next(i for i, r in enumerate(rows) if r and r[0] == 'ID')
h = rows[start]; ix = {k: i for i, k in enumerate(h)}
agg = collections.OrderedDict(); tot = 0.0
scale = {'nsecond': 1e-6, 'usecond': 1e-3, 'msecond': 1.0, 'ns': 1e-6, 'us': 1e-3, 'ms': 1.0}
for r in rows[start + 1:]:
    name = r[ix['Kernel Name']]
    name = name[:70]
    v = float(r[ix['Metric Value']].replace(',', '')) * scale.get(r[ix['Metric Unit']], 1e-6)
    a = agg.setdefault(name, [0, 0.0]); a[0] += 1; a[1] += v; tot += v
print(f"total {tot:.3f} ms over {sum(a[0] for a in agg.values())} launches")
for k, (c, v) in sorted(agg.items(), key=lambda a: -a[1][1])[:int(sys.argv[2]) if len(sys.argv) > 2 else 20]:
    print(f"{v:9.3f} ms {100*v/tot:5.1f}% {c:5d}x {v/c*1e3:9.1f} us  {k}")
