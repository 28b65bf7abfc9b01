"""Golden results of the REFERENCE on BASELINE.json configs[0] (C1) and a
T1-shaped fixed-iteration Ritz trace, for the slow GPU parity tests.

C1 = SynthParams{kind=Random, n=1e5, density=5e7/(n(n-1)/2), block_extent=4000,
tile 4..512, seed=1} (synth.hpp:33-43), SolverConfig{k=8, nb=16,
tol=1e-6, maxiter=500, fom m=4, seed=1} (lobpcg.hpp:24-48), precond on and
off, each under the summation orders the reference itself offers (serial,
8-thread baseline, 8-thread fused-atomic: SURVEY 8c "envelope").

The matrix is regenerated on the GPU box by the library's bit-exact
generate_synthetic restatement; the fixture stores a SHA-256 of the reference's
CSB arrays so the test proves it solved the same bytes.

Runs in the build container only (needs oracle/_ref/libref.so):
    python tests/golden/make_golden_c1.py        (~10 min on 8 cores)
"""
from __future__ import annotations

import hashlib
import json
import sys
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent))
sys.path.insert(0, str(HERE.parents[1]))
import oracle_lib as ol  # noqa: E402

N = 100_000
NNZ = 50_000_000
EXTENT = 4000


def csb_digest(bn, bo, lr, lc, v, diag):
    h = hashlib.sha256()
    for a in (bn, bo, lr, lc, v, diag):
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def main():
    from paper_2109_00485_b200 import abi  # host-only CSB container for the ref calls
    dens = NNZ / (N * (N - 1) / 2)
    t0 = time.time()
    rows, cols, vals, diag, toff = ol.ref_generate_synthetic(2, N, density=dens, block_extent=EXTENT, seed=1)
    rb = np.array(list(range(0, N, EXTENT)) + [N], np.int64)
    bn, bo, lr, lc, v = ol.ref_build_csb(rows, cols, vals, N, N, rb, rb)
    m = abi.Csb(N, N, rb, rb, bn, bo, lr, lc, v)
    print(f"C1 generated+built in {time.time() - t0:.1f}s, nnz {len(v)}", flush=True)
    out = dict(n=N, nnz=int(len(v)), density=dens, extent=EXTENT, seed=1, k=8, nb=16, tol=1e-6, maxiter=500,
               fom_m=4, csb_sha256=csb_digest(bn, bo, lr, lc, v, diag), ntiles=int(len(toff) - 1), runs={})
    for tag, t in (("off", None), ("on", toff)):
        for name, threads, variant in (("serial", 1, 0), ("baseline8", 8, 0), ("fused8", 8, 1)):
            t0 = time.time()
            r = ol.Impl("ref", threads=threads, variant=variant).lobpcg(m, diag, t, k=8, nb=16, tol=1e-6,
                                                                        maxiter=500, fom_m=4, seed=1)
            out["runs"][f"{tag}_{name}"] = dict(iterations=r["iterations"], converged=r["converged"],
                                                operator_calls=r["operator_calls"], lambda_=r["lambda_"].tolist(),
                                                theta_first10=r["theta"][:10].tolist(),
                                                theta=r["theta"][:, :8].tolist(),
                                                residual_norms=r["residual_norms"][:, :8].tolist(),
                                                n_converged=r["n_converged"].tolist(), fallbacks=r["fallbacks"],
                                                seconds=round(time.time() - t0, 1))
            print(tag, name, r["iterations"], r["lambda_"][:3], f"{time.time() - t0:.1f}s", flush=True)
    (HERE / "c1_reference.json").write_text(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
