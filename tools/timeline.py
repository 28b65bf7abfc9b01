"""Kernel timeline of a few T1 LOBPCG iterations (torch.profiler / CUPTI sees every kernel the
library launches): per-iteration busy time, idle gaps between kernels, and the largest gaps with
their neighbours. Development tool: python tools/timeline.py [iters]"""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

from paper_2109_00485_b200 import abi  # noqa: E402

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 3
m, diag, toff = abi.generate_clustered(n=2_900_000, target_nnz=1_100_000_000, block_extent=4000, tile=128, fill=0.10,
                                       seed=1)
ctx = abi.Context(0)
op = abi.Operator(ctx, m, diag, values_prec=abi.BE_F32)
tiles = abi.Tiles(ctx, m, diag, toff)
n = m.nrows
del m
s = abi.IncrementalSolve(ctx, op, n=n, tiles=tiles, k=8, nb=16, tol=1e-300, maxiter=100, seed=1)
s.step(3)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    s.step(iters)
    torch.cuda.synchronize()
s.end()
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
ker = sorted([(e.time_range.start, e.time_range.end, e.name) for e in ev], key=lambda x: x[0])
# merge overlapping (side-stream) intervals
busy, gaps = 0.0, []
cur_s, cur_e, last_name = ker[0][0], ker[0][1], ker[0][2]
for st, en, nm in ker[1:]:
    if st > cur_e:
        busy += cur_e - cur_s
        gaps.append((st - cur_e, last_name[:40], nm[:40]))
        cur_s, cur_e = st, en
    else:
        cur_e = max(cur_e, en)
    last_name = nm
busy += cur_e - cur_s
span = ker[-1][1] - ker[0][0]
tot_gap = sum(g for g, _, _ in gaps)
print(json.dumps({"iterations": iters, "kernels": len(ker), "span_ms": span / 1e3, "busy_ms": busy / 1e3,
                  "gap_ms": tot_gap / 1e3, "gaps": len(gaps)}))
for g, a, b in sorted(gaps, reverse=True)[:15]:
    print(f"{g:8.1f} us  after {a}  before {b}")
