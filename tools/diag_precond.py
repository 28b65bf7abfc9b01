import sys; sys.path.insert(0,'.'); sys.path.insert(0,'tests')
import numpy as np
import oracle_lib as ol
from paper_2109_00485_b200 import abi
from test_lobpcg_gpu import make_test_matrix
ctx = abi.Context(0)
m, d = make_test_matrix(500, 2495, 77)
toff = np.array([0] + list(range(25, 500, 25)) + [500])
want = ol.Impl("orc").lobpcg(m, d, toff, k=4, nb=8, tol=1e-9, maxiter=800, seed=77)
got = abi.lobpcg(ctx, abi.Operator(ctx, m, d, values_prec=abi.BE_F64), tiles=abi.Tiles(ctx, m, d, toff), k=4, nb=8, tol=1e-9, maxiter=800, seed=77)
for i in range(min(want['iterations'], got['iterations'])):
    print(i+1, want['n_converged'][i], got['n_converged'][i], np.max(np.abs(want['theta'][i]-got['theta'][i])/np.abs(want['theta'][i])), want['residual_norms'][i][:4], got['residual_norms'][i][:4])
# single precond application parity
r = np.random.default_rng(1).uniform(-1,1,(500,8)); sh = np.linspace(1,3,8)
w1,_ = abi.Tiles(ctx, m, d, toff).apply_host(sh, r); w2,_ = ol.Impl("orc").precond(m, d, toff, sh, r)
print("precond relerr", np.linalg.norm(w1-w2)/np.linalg.norm(w2))
for thr,var in ((1,0),(4,0),(4,1),(8,0)):
    x = ol.Impl("ref", threads=thr, variant=var).lobpcg(m, d, toff, k=4, nb=8, tol=1e-9, maxiter=800, seed=77)
    print("ref", thr, var, x['iterations'])
