"""Top SASS lines of an ncu source page export by a chosen metric column (development tool).

    ncu -i x.ncu-rep --page source --csv --print-source sass > /tmp/sass.csv
    python tools/sass_hot.py /tmp/sass.csv "L1 Wavefronts Shared" 40
"""
import csv
import sys

path, col = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
rows = list(csv.reader(open(path)))
h = rows[1]
ci = h.index(col)
si, ie = h.index("Source"), h.index("Instructions Executed")
samp = h.index("Warp Stall Sampling (All Samples)")
data = []
for r in rows[2:]:
    try:
        v = float(r[ci] or 0)
    except ValueError:
        continue
    data.append((v, r[0][-5:], r[si].strip()[:70], r[ie], r[samp]))
tot = sum(d[0] for d in data)
print(f"total {col}: {tot:.4g}")
for v, a, s, ie_, sm in sorted(data, reverse=True)[:top]:
    print(f"{v:12.4g} {100 * v / tot if tot else 0:5.1f}%  {a} inst={ie_:>10} samp={sm:>6}  {s}")
