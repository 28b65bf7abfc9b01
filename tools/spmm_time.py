"""Time the device SpMM (k_sym_spmm path of be_op_apply) at T1 for the library in $BE_LIB
(kernel-variant experiments): python tools/spmm_time.py [reps]"""
import os
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2109_00485_b200 import abi  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
m, diag, _ = abi.generate_clustered(n=2_900_000, target_nnz=1_100_000_000, block_extent=4000, tile=128, fill=0.10,
                                    seed=1)
ctx = abi.Context(0)
op = abi.Operator(ctx, m, diag, values_prec=abi.BE_F32)
n, nb = m.nrows, int(os.environ.get("NB", "16"))
x = torch.rand(n, nb, dtype=torch.float64, device="cuda") * 2 - 1
y = torch.empty_like(x)
op.timing(1)
ks = []
for i in range(reps + 2):
    op.apply_dev(x.data_ptr(), y.data_ptr(), n, nb, stream=ctx.stream())
    k, a = op.timing()
    if i >= 2:
        ks.append(k)
ref = abi.Operator(ctx, m, diag, values_prec=abi.BE_F32)
print(f"{os.environ.get('BE_LIB', 'default')}: sym_spmm kernel {np.median(ks):.3f} ms (min {np.min(ks):.3f})")
