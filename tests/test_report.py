"""The JSON run report ("blockeig/run-report/v1", driver.hpp:236-281,
docs/report-schema.md) of a device solve, next to the reference driver's own
report for the same generated problem (oracle/_ref: cmd_solve of the
unmodified reference headers)."""
from __future__ import annotations

import ctypes as C
import json

import numpy as np
import pytest

import oracle_lib as ol
from paper_2109_00485_b200 import report


def test_size_histogram_buckets():  # driver.hpp:80-100
    h = report.size_histogram([4, 5, 7, 8, 16, 511, 512, 1])
    assert h[0] == {"min_size": 1, "max_size": 1, "count": 1}
    assert h[1]["count"] == 0 and h[2] == {"min_size": 4, "max_size": 7, "count": 3}
    assert h[3]["count"] == 1 and h[4]["count"] == 1 and h[8] == {"min_size": 256, "max_size": 511, "count": 1}
    assert h[9] == {"min_size": 512, "max_size": 1023, "count": 1} and len(h) == 10


def _fake(iters=3, nb=4):
    return dict(lambda_=np.arange(1.0, 3.0), converged=True, iterations=iters, operator_calls=iters + 1, fallbacks=0,
                restarts=0, theta=np.ones((iters, nb)), residual_norms=np.full((iters, nb), 1e-3),
                n_converged=np.arange(iters), times=np.full((iters, 4), 0.5))


def test_report_fields_and_finiteness():
    cfg = report.config_echo(k=2, nb=4, tol=1e-6, maxiter=10, fom_iters=4, seed=1, no_precond=False,
                             input_echo={"gen": "random", "n": 10})
    j = report.solve_report(_fake(), n=10, nnz_lower=20, config=cfg, tile_sizes=[4, 6])
    assert j["schema"] == "blockeig/run-report/v1" and j["command"] == "solve"
    assert j["iterations"] == 3 and len(j["history"]) == 3 and j["history"][0]["iter"] == 1
    assert j["residual_norms"] == [1e-3, 1e-3] and j["timings"]["total"] == 1.5
    assert j["precond_stats"]["tiles"] == 2
    json.loads(report.dumps(j))
    bad = _fake()
    bad["lambda_"] = np.array([np.nan, 1.0])
    with pytest.raises(ValueError):
        report.solve_report(bad, n=10, nnz_lower=20, config=cfg)


def _keys(x):
    if isinstance(x, dict):
        return {k: _keys(v) for k, v in x.items()}
    if isinstance(x, list) and x and isinstance(x[0], dict):
        return [_keys(x[0])]
    return None


@pytest.mark.gpu
@pytest.mark.parametrize("no_precond", [True, False])
def test_device_report_matches_the_reference_report(ctx, no_precond):
    lib = ol.ref()
    if lib is None:
        pytest.skip("oracle/_ref/libref.so not built")
    from paper_2109_00485_b200 import abi
    n, dens, ext, k, nb, tol, maxiter, seed = 3000, 0.01, 1000, 4, 8, 1e-6, 200, 1
    f = lib.ref_cmd_solve
    f.argtypes = [C.c_char_p, C.c_int64, C.c_double, C.c_int64, C.c_int, C.c_int, C.c_double, C.c_int, C.c_uint64,
                  C.c_int, C.POINTER(C.c_int64)]
    ln = C.c_int64()
    assert f(b"random", n, dens, ext, k, nb, tol, maxiter, seed, int(no_precond), C.byref(ln)) == 0
    buf = C.create_string_buffer(ln.value)
    assert lib.ref_last_report(buf, C.c_int64(ln.value)) == 0
    ref = json.loads(buf.raw[:ln.value].decode())
    # the same problem: generate_synthetic is bit-exact (tests/test_golden_cpu.py)
    s = abi.Synthetic("random", n=n, density=dens, block_extent=ext, seed=seed)
    b = abi.uniform_boundaries(n, ext)
    m = abi.build_csb_coo(s.lower, n, n, b, b)
    op = abi.Operator(ctx, m, s.diag, values_prec=abi.BE_F64, deterministic=True)
    tiles = None if no_precond else abi.Tiles(ctx, m, s.diag, s.tile_offsets)
    res = abi.lobpcg(ctx, op, tiles=tiles, k=k, nb=nb, tol=tol, maxiter=maxiter, seed=seed)
    echo = dict(ref["config"]["input"])  # the driver's input echo (gen, n, density, bandwidth, block_extent, cache)
    cfg = report.config_echo(k=k, nb=nb, tol=tol, maxiter=maxiter, fom_iters=4, seed=seed, no_precond=no_precond,
                             input_echo=echo, variant="baseline")
    ours = report.solve_report(res, n=n, nnz_lower=m.nnz, config=cfg,
                               tile_sizes=None if no_precond else list(np.diff(s.tile_offsets)))
    assert _keys(ours) == _keys(ref)
    assert ours["config"] == ref["config"] and ours["n"] == ref["n"] and ours["nnz_lower"] == ref["nnz_lower"]
    rel = np.max(np.abs(np.array(ours["eigenvalues"]) - ref["eigenvalues"]) / np.abs(ref["eigenvalues"]))
    assert rel <= 1e-6, rel
    assert ours["converged"] and ref["converged"]
    if no_precond:  # not chaotic: the same iteration count (north star: +-1)
        assert abs(ours["iterations"] - ref["iterations"]) <= 1
    else:
        assert ours["precond_stats"] == ref["precond_stats"]
    assert ours["operator_calls"] == ours["iterations"] + 1
