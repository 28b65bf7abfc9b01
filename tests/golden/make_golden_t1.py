"""Golden Ritz-value trace of the REFERENCE on the Test-1-shaped problem
(BASELINE.json configs[1]: n = 2.9e6, 1.1e9 stored lower nonzeros, nev = 8,
block k = 16), 10 fixed iterations (tol = 1e-300, the pattern of
test_lobpcg.cpp:341), for the slow GPU parity test: with the preconditioner
on under ThreadPool(8) ("theta") and ThreadPool(4) ("theta_t4": the
reference's own summation-order spread), and with it off ("theta_off",
ThreadPool(8)), where the trajectory is not chaotic.

The matrix is the clustered generator's (counter-based, so the GPU
box regenerates the same bytes -- the fixture stores a SHA-256 of the CSB
arrays to prove it). The reference runs through oracle/_ref/libref.so
(unmodified reference headers, lobpcg.hpp:291-449) on 8 host threads.

    python tests/golden/make_golden_t1.py      (~3 min, ~25 GB RAM)
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

T1 = dict(n=2_900_000, target_nnz=1_100_000_000, block_extent=4000, tile=128, fill=0.10, block_occupancy=1.0, seed=1)
ITERS = 10


def digest(m, diag):
    h = hashlib.sha256()
    for a in (m.block_nnz, m.block_nnz_offsets, m.local_rows, m.local_cols, m.values, diag):
        h.update(memoryview(np.ascontiguousarray(a)).cast("B"))
    return h.hexdigest()


def main():
    from paper_2109_00485_b200 import abi
    t0 = time.time()
    m, diag, toff = abi.generate_clustered(**T1)
    print(f"T1 generated in {time.time() - t0:.1f}s: nnz {m.nnz}", flush=True)
    t0 = time.time()
    dg = digest(m, diag)
    print(f"digest {dg} in {time.time() - t0:.1f}s", flush=True)
    t0 = time.time()
    r = ol.Impl("ref", threads=8, variant=0).lobpcg(m, diag, toff, k=8, nb=16, tol=1e-300, maxiter=ITERS, fom_m=4,
                                                   seed=1)
    print(f"reference {ITERS} iterations in {time.time() - t0:.1f}s", flush=True)
    out = dict(params=T1, nnz=int(m.nnz), csb_sha256=dg, k=8, nb=16, fom_m=4, seed=1, iterations=r["iterations"],
               theta=r["theta"].tolist(), residual_norms=r["residual_norms"].tolist(),
               operator_calls=r["operator_calls"], fallbacks=r["fallbacks"])
    t0 = time.time()
    r4 = ol.Impl("ref", threads=4, variant=0).lobpcg(m, diag, toff, k=8, nb=16, tol=1e-300, maxiter=ITERS, fom_m=4,
                                                    seed=1)
    out["theta_t4"] = r4["theta"].tolist()
    print(f"reference (4 threads) {ITERS} iterations in {time.time() - t0:.1f}s", flush=True)
    t0 = time.time()
    ro = ol.Impl("ref", threads=8, variant=0).lobpcg(m, diag, None, k=8, nb=16, tol=1e-300, maxiter=ITERS, fom_m=4,
                                                    seed=1)
    out["theta_off"] = ro["theta"].tolist()
    out["residual_norms_off"] = ro["residual_norms"].tolist()
    print(f"reference (precond off) {ITERS} iterations in {time.time() - t0:.1f}s", flush=True)
    (HERE / "t1_reference.json").write_text(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
