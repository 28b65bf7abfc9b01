import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
from paper_2109_00485_b200 import abi
kw = dict(n=24000, target_nnz=3_000_000, block_extent=2000, seed=3)
whole, diag, toff = abi.generate_clustered(**kw)
ctx = abi.Context(0)
op = abi.Operator(ctx, whole, diag)
op64 = abi.Operator(ctx, whole, diag, values_prec=abi.BE_F64)
tiles = abi.Tiles(ctx, whole, diag, toff)
for name, o, t in [("f32 precond", op, tiles), ("f64 precond", op64, tiles), ("f32 noprec", op, None)]:
    for tol in (1e-6, 1e-5):
        its = []
        for rep in range(4):
            r = abi.lobpcg(ctx, o, tiles=t, k=8, nb=16, tol=tol, maxiter=300, seed=1)
            its.append((r["iterations"], r["converged"], r["fallbacks"]))
        print(name, tol, its, "last resn", np.max(r["residual_norms"][-1][:8] / np.abs(r["theta"][-1][:8])))
