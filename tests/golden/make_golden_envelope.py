"""Summation-order envelopes of the REFERENCE for the precondition-on runs
(SURVEY 8c): the reference's lobpcg_solve through oracle/_ref/libref.so with
ThreadPool(T) for several T (the Gram / SpMM partial sums, densela.hpp:74-89,
change with T). Adds to c1_reference.json: {"envelope_on": {T: iterations}}
plus the full Ritz trajectory of T = 4; adds to t1_reference.json the 10-
iteration Ritz trace of T = 4 ("theta_t4"). The GPU tests compare our
trajectories against the reference's own spread, not against one order.

    python tests/golden/make_golden_envelope.py      (~20 min)
"""
from __future__ import annotations

import json
import sys
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent))
sys.path.insert(0, str(HERE.parents[1]))
import oracle_lib as ol  # noqa: E402


def c1():
    from paper_2109_00485_b200 import abi
    path = HERE / "c1_reference.json"
    g = json.loads(path.read_text())
    n = g["n"]
    s = abi.Synthetic("random", n=n, density=g["density"], block_extent=g["extent"], seed=g["seed"])
    b = abi.uniform_boundaries(n, g["extent"])
    m = abi.build_csb_coo(s.lower, n, n, b, b)
    env = {}
    for t in (2, 3, 4, 5, 6, 7):
        t0 = time.time()
        r = ol.Impl("ref", threads=t, variant=0).lobpcg(m, s.diag, s.tile_offsets, k=8, nb=16, tol=1e-6,
                                                        maxiter=500, fom_m=4, seed=1)
        env[str(t)] = r["iterations"]
        if t == 4:
            g["runs"]["on_t4"] = dict(iterations=r["iterations"], lambda_=r["lambda_"].tolist(),
                                      theta=r["theta"][:, :8].tolist())
        print("C1 on threads", t, r["iterations"], f"{time.time() - t0:.0f}s", flush=True)
    env["1"] = g["runs"]["on_serial"]["iterations"]
    env["8"] = g["runs"]["on_baseline8"]["iterations"]
    g["envelope_on"] = env
    path.write_text(json.dumps(g, indent=1))


def t1():
    from paper_2109_00485_b200 import abi
    path = HERE / "t1_reference.json"
    g = json.loads(path.read_text())
    m, diag, toff = abi.generate_clustered(**g["params"])
    t0 = time.time()
    r = ol.Impl("ref", threads=4, variant=0).lobpcg(m, diag, toff, k=8, nb=16, tol=1e-300, maxiter=g["iterations"],
                                                   fom_m=4, seed=1)
    g["theta_t4"] = r["theta"].tolist()
    print("T1 threads 4", f"{time.time() - t0:.0f}s", flush=True)
    path.write_text(json.dumps(g, indent=1))


if __name__ == "__main__":
    c1()
    t1()
