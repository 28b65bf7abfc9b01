"""Time the tile kernel per pass at T1 (development tool): symmetric (both passes),
notrans (pass R only), trans (pass C only), on f32 panels; nb from argv."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2109_00485_b200 import abi  # noqa: E402

nbs = [int(a) for a in sys.argv[1:]] or [16]
m, diag, _ = abi.generate_clustered(n=2_900_000, target_nnz=1_100_000_000, block_extent=4000, tile=128, fill=0.10,
                                    seed=1)
ctx = abi.Context(0)
op = abi.Operator(ctx, m, diag, values_prec=abi.BE_F32)
n = m.nrows
del m
op.timing(1)
for nb in nbs:
    x = torch.rand(n, nb, dtype=torch.float32, device="cuda") * 2 - 1
    y = torch.zeros_like(x)
    for name, mode in (("both", abi.BE_APPLY_SYMMETRIC), ("R", abi.BE_APPLY_NOTRANS_ACC), ("C", abi.BE_APPLY_TRANS_ACC)):
        ks = []
        for i in range(8):
            op.apply_dev(x.data_ptr(), y.data_ptr(), n, nb, abi.BE_F32, mode, ctx.stream())
            k, a = op.timing()
            if i >= 2:
                ks.append(k)
        print(f"nb={nb} {name}: {np.median(ks):.3f} ms", flush=True)
