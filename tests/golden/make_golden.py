"""Generate the golden fixtures in tests/golden/ from the REFERENCE itself.

Runs in the build container only (needs oracle/_ref/libref.so, compiled from
the unmodified reference headers by oracle/Makefile). The fixtures are small
.npz files committed to the repo; tests/test_golden_cpu.py checks the oracle
restatement and the library's host code against them, and the GPU parity
tests can use them on the GPU box where /root/reference does not exist.

    python tests/golden/make_golden.py
"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent))
sys.path.insert(0, str(HERE.parents[1]))
import oracle_lib as ol  # noqa: E402

REF = ol.Impl("ref", threads=1, variant=0)


def csb_arrays(bn, bo, lr, lc, v):
    return dict(block_nnz=bn, block_nnz_offsets=bo, local_rows=lr, local_cols=lc, values=v)


def case(name, kind, n, density, extent, seed, nb, k, shifts, bandwidth=8):
    rows, cols, vals, diag, toff = ol.ref_generate_synthetic(kind, n, density=density, bandwidth=bandwidth,
                                                             block_extent=extent, seed=seed)
    rb = np.array(list(range(0, n, extent)) + [n], np.int64)
    bn, bo, lr, lc, v = ol.ref_build_csb(rows, cols, vals, n, n, rb, rb)
    from paper_2109_00485_b200 import abi  # host-only CSB container for the ref calls
    m = abi.Csb(n, n, rb, rb, bn, bo, lr, lc, v)
    rng = np.random.default_rng(seed + 100)
    x = rng.uniform(-1, 1, (n, nb))
    y = REF.spmm(m, diag, x)                       # SymmetricOperator::apply (serial baseline)
    yn = REF.spmm(m, None, x, y=np.ones((n, nb)), mode=1)  # U += L W
    yt = REF.spmm(m, None, x, y=np.ones((n, nb)), mode=2)  # U += L^T W
    r = rng.uniform(-1, 1, (n, nb))
    w, fb = REF.precond(m, diag, toff, shifts, r, m=4)
    out = dict(kind=kind, n=n, density=density, extent=extent, seed=seed, bandwidth=bandwidth,
               rows=rows, cols=cols, vals=vals, diag=diag, tile_offsets=toff, row_bounds=rb,
               x=x, y_sym=y, y_notrans=yn, y_trans=yt, r=r, shifts=np.asarray(shifts, float), w_precond=w,
               precond_fallbacks=fb, **csb_arrays(bn, bo, lr, lc, v))
    for tag, t in (("pon", toff), ("poff", None)):
        res = REF.lobpcg(m, diag, t, k=k, nb=nb, tol=1e-6, maxiter=150, fom_m=4, seed=seed)
        out[f"lobpcg_{tag}_lambda"] = res["lambda_"]
        out[f"lobpcg_{tag}_iterations"] = res["iterations"]
        out[f"lobpcg_{tag}_converged"] = res["converged"]
        out[f"lobpcg_{tag}_theta"] = res["theta"]
        out[f"lobpcg_{tag}_nconv"] = res["n_converged"]
        out[f"lobpcg_{tag}_operator_calls"] = res["operator_calls"]
    np.savez_compressed(HERE / f"{name}.npz", **out)
    print(name, "nnz", len(vals), "iters on/off", out["lobpcg_pon_iterations"], out["lobpcg_poff_iterations"])


def dense_cases():
    rng = np.random.default_rng(5)
    out = {}
    for i, (n, k) in enumerate([(6, 2), (12, 4), (48, 16)]):
        a = rng.standard_normal((n, n))
        a = a + a.T
        q = rng.standard_normal((n, n))
        b = q @ q.T + n * np.eye(n)
        c, d = REF.sygv_lowest(a, b, k, 1e-10)
        out[f"sygv{i}_a"], out[f"sygv{i}_b"], out[f"sygv{i}_k"] = a, b, k
        out[f"sygv{i}_c"], out[f"sygv{i}_d"] = c, d
    np.savez_compressed(HERE / "dense.npz", **out)
    print("dense", len(out))


if __name__ == "__main__":
    # kinds: 0 Banded, 1 BlockTile, 2 Random (synth.hpp:14)
    case("random_n600", 2, 600, 0.03, 150, 3, nb=6, k=3, shifts=[0.0, 0.5, -1.0, 2.0, 0.0, 1.5])
    case("banded_n500", 0, 500, 0.02, 128, 4, nb=5, k=2, shifts=[0.1, 0.2, 0.3, 0.4, 0.5], bandwidth=6)
    case("blocktile_n700", 1, 700, 0.02, 200, 5, nb=8, k=4, shifts=[0.0] * 8)
    dense_cases()
