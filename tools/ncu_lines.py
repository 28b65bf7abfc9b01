"""Summarise an ncu report per CUDA source line (instructions, stall samples, smem wavefronts)."""
import csv, subprocess, sys
rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"] + sys.argv[3:],
                     capture_output=True, text=True).stdout.splitlines()
r = csv.reader(out)
next(r); next(r); h = next(r)
ix = {}
for i, k in enumerate(h):
    ix.setdefault(k, i)
def num(s):
    try: return int(s)
    except Exception: return 0
agg = []
for x in r:
    if len(x) > 10 and x[0] != '' and x[0] != 'Line No':
        agg.append((num(x[ix['Instructions Executed']]), num(x[ix['Warp Stall Sampling (All Samples)']]),
                    num(x[ix['L1 Wavefronts Shared']]), num(x[ix['L1 Wavefronts Shared Ideal']]), x[0], x[1][:90]))
tot = sum(a[0] for a in agg) or 1; ts = sum(a[1] for a in agg) or 1
print(f"total warp instructions {tot}, stall samples {ts}")
for a in sorted(agg, key=lambda a: -a[1])[:n]:
    print(f"{a[0]/tot*100:5.1f}% ins {a[1]/ts*100:5.1f}% smp  wf {a[2]:>11d}/{a[3]:<11d} L{a[4]:>4s} {a[5]}")
