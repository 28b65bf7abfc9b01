"""Per-kernel breakdown of one LOBPCG iteration from an `ncu --metrics gpu__time_duration.sum --csv`
launch list: the launches from the second-to-last k_sym_spmm up to (not including) the last one.
python tools/iter_breakdown.py launches.csv"""
import collections, csv, re, sys
rows = list(csv.reader(open(sys.argv[1])))
start = next(i for i, r in enumerate(rows) if r and r[0] == 'ID')
ix = {k: i for i, k in enumerate(rows[start])}
scale = {'nsecond': 1e-3, 'usecond': 1.0, 'msecond': 1e3, 'ns': 1e-3, 'us': 1.0, 'ms': 1e3}
ls = []
for r in rows[start + 1:]:
    if r[ix['Metric Name']] != 'gpu__time_duration.sum':
        continue
    name = r[ix['Kernel Name']]
    v = float(r[ix['Metric Value']].replace(',', '')) * scale.get(r[ix['Metric Unit']], 1e-3)
    ls.append((name, v))
sp = [i for i, (n, _) in enumerate(ls) if 'k_sym_spmm' in n]
a, b = sp[-2], sp[-1]
agg = collections.OrderedDict()
for n, v in ls[a:b]:
    short = re.sub(r'\(.*', '', n).replace('void ', '')
    short = re.sub(r'^.*(unnamed>::|dla::|be::)', '', short)
    if not short.startswith('k_'):
        short = 'library: ' + short[:40]
    e = agg.setdefault(short, [0, 0.0]); e[0] += 1; e[1] += v
tot = sum(e[1] for e in agg.values())
print(f"| kernel | launches | µs | share |\n|---|---:|---:|---:|")
for k, (c, v) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"| `{k}` | {c} | {v:.1f} | {100 * v / tot:.1f}% |")
print(f"| **total** | {sum(e[0] for e in agg.values())} | {tot:.1f} | |")
