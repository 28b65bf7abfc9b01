"""Small workload touching every device kernel, for compute-sanitizer (tools/sanitize.sh)."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2109_00485_b200 import abi  # noqa: E402

ctx = abi.Context(0)
n = 3000
s = abi.Synthetic("random", n=n, density=0.01, block_extent=1000, seed=1)
b = abi.uniform_boundaries(n, 1000)
m = abi.build_csb_coo(s.lower, n, n, b, b)
rng = np.random.default_rng(0)
for prec in (abi.BE_F32, abi.BE_F64):
    op = abi.Operator(ctx, m, s.diag, values_prec=prec)
    for nb in (4, 8, 16, 32):
        x = rng.uniform(-1, 1, (n, nb))
        op.apply_host(x)
        op.apply_host(x, np.zeros((n, nb)), mode=abi.BE_APPLY_NOTRANS_ACC)
        op.apply_host(x, np.zeros((n, nb)), mode=abi.BE_APPLY_TRANS_ACC)
    op.close()
det = abi.Operator(ctx, m, s.diag, values_prec=abi.BE_F64, deterministic=True)
det.apply_host(rng.uniform(-1, 1, (n, 16)))
tiles = abi.Tiles(ctx, m, s.diag, s.tile_offsets)
op = abi.Operator(ctx, m, s.diag, values_prec=abi.BE_F32)
for nb in (8, 16):
    r = abi.lobpcg(ctx, op, tiles=tiles, k=4, nb=nb, tol=1e-6, maxiter=40, seed=1)
r = abi.lobpcg(ctx, op, k=8, nb=24, tol=1e-300, maxiter=4, seed=2)  # nb=24: generic dense kernels
print("sanitize workload done", r["iterations"])
