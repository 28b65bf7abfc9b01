import sys; sys.path.insert(0,'.'); sys.path.insert(0,'tests')
import numpy as np
import oracle_lib as ol
from paper_2109_00485_b200 import abi
ctx = abi.Context(0)
n = 1000
for s in range(4):
    g = abi.Synthetic("random", n=n, density=0.005, block_extent=1000, seed=6000 + s)
    m = abi.build_csb_coo(g.lower, n, n, [0, n], [0, n])
    kw = dict(k=5, nb=8, tol=1e-6, maxiter=500, seed=6100 + s)
    o = ol.Impl("orc").lobpcg(m, g.diag, g.tile_offsets, **kw)
    refs = [ol.Impl("ref", threads=t, variant=v).lobpcg(m, g.diag, g.tile_offsets, **kw)["iterations"] for t, v in ((1,0),(4,0),(4,1),(8,0),(8,1))]
    gp = abi.lobpcg(ctx, abi.Operator(ctx, m, g.diag, values_prec=abi.BE_F64), tiles=abi.Tiles(ctx, m, g.diag, g.tile_offsets), **kw)
    g2 = abi.lobpcg(ctx, abi.Operator(ctx, m, g.diag, values_prec=abi.BE_F64), tiles=abi.Tiles(ctx, m, g.diag, g.tile_offsets), **kw)
    print(s, "orc", o["iterations"], "ref", refs, "gpu", gp["iterations"], g2["iterations"], "restarts", gp["restarts"], "fb", gp["fallbacks"])
    if gp["iterations"] >= 500:
        print("  lam", gp["lambda_"], o["lambda_"])
        for it in (10, 50, 100, 200, 499):
            print("  ", it, gp["residual_norms"][it][:5], gp["n_converged"][it])
        print("  orc last", o["residual_norms"][-1][:5])
