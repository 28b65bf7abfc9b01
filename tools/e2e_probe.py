"""Fixed per-solve overhead of the host-buffer solve call at T1: time abi.lobpcg for a few maxiter values."""
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2109_00485_b200 import abi  # noqa: E402

m, diag, toff = abi.generate_clustered(n=2_900_000, target_nnz=1_100_000_000, block_extent=4000, tile=128, fill=0.10,
                                       seed=1)
ctx = abi.Context(0)
op = abi.Operator(ctx, m, diag, values_prec=abi.BE_F32)
tiles = abi.Tiles(ctx, m, diag, toff)
x0 = np.random.default_rng(5).uniform(-1, 1, (m.nrows, 16))
for it in (1, 1, 5, 10, 10):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = abi.lobpcg(ctx, op, tiles=tiles, x0=x0, k=8, nb=16, tol=1e-300, maxiter=it, seed=3)
    print(f"maxiter {it}: {time.perf_counter() - t0:.3f} s", flush=True)
