"""Quick SpMM throughput probe (development tool; bench.py is the contract)."""
import argparse, json, sys, time
from pathlib import Path
import numpy as np
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2109_00485_b200 import abi

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=2_900_000)
ap.add_argument("--nnz", type=int, default=1_100_000_000)
ap.add_argument("--kind", default="clustered")
ap.add_argument("--nb", type=int, default=16)
ap.add_argument("--panel", default="f32")
ap.add_argument("--reps", type=int, default=10)
a = ap.parse_args()
import torch
t0 = time.time()
if a.kind == "clustered":
    m, diag, toff = abi.generate_clustered(n=a.n, target_nnz=a.nnz, seed=1)
else:
    s = abi.Synthetic("random", n=a.n, density=a.nnz / (a.n * (a.n - 1) / 2), block_extent=4000, seed=1)
    b = abi.uniform_boundaries(a.n, 4000)
    m = abi.build_csb_coo(s.lower, a.n, a.n, b, b); diag = s.diag; del s
t1 = time.time()
ctx = abi.Context(0)
op = abi.Operator(ctx, m, diag)
t2 = time.time()
info = op.info()
print(f"gen {t1-t0:.1f}s upload {t2-t1:.1f}s nnz {info.nnz} tiles {info.ntiles} dev bytes {info.device_bytes/1e9:.2f} GB", flush=True)
nnz = m.nnz
del m
dt = torch.float32 if a.panel == "f32" else torch.float64
x = (torch.rand(a.n, a.nb, dtype=dt, device="cuda") * 2 - 1)
y = torch.empty_like(x)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
prec = abi.BE_F32 if a.panel == "f32" else abi.BE_F64
s = ctx.stream()
op.timing(1)
ks, aps = [], []
for i in range(a.reps + 2):
    flush.zero_(); torch.cuda.synchronize()
    op.apply_dev(x.data_ptr(), y.data_ptr(), a.n, a.nb, prec, abi.BE_APPLY_SYMMETRIC, s)
    k, ap_ = op.timing(-1)
    if i >= 2: ks.append(k); aps.append(ap_)
sp = x.element_size()
B = nnz * 8 + 2 * a.n * a.nb * sp + a.n * 4
km, am = np.median(ks), np.median(aps)
print(json.dumps(dict(n=a.n, nnz=nnz, nb=a.nb, panel=a.panel, kernel_ms=km, apply_ms=am, alg_GB=B/1e9, GBs_apply=B/am/1e6, GBs_kernel=B/km/1e6)), flush=True)
