"""The reference driver's JSON run report ("blockeig/run-report/v1", solve command)
for a device solve: driver.hpp:236-281 and docs/report-schema.md:6-50.

`solve_report(result, ...)` turns the dict returned by `abi.lobpcg` into the
same document the reference CLI emits for `solve`: the config echo, n,
nnz_lower, eigenvalues, converged, iterations, operator_calls, the per-
iteration history (theta, residual_norms, n_converged, t_spmm, t_precond,
t_dense, t_total in seconds), final residual_norms of the first k columns,
accumulated timings, precond_stats (tiles, fallbacks, power-of-two
size_histogram) unless the preconditioner is off, comm (nd > 1) and restarts.
Like the reference emitter (driver.hpp:191-195) it rejects NaN / infinity.
"""
from __future__ import annotations

import json
import math

SCHEMA = "blockeig/run-report/v1"


def size_histogram(sizes):
    """Power-of-two buckets [1,2), [2,4), ... (driver.hpp:80-100)."""
    counts = []
    for s in sizes:
        b, hi = 0, 2
        while s >= hi:
            hi *= 2
            b += 1
        if b >= len(counts):
            counts.extend([0] * (b + 1 - len(counts)))
        counts[b] += 1
    out, lo = [], 1
    for c in counts:
        out.append({"min_size": lo, "max_size": 2 * lo - 1, "count": c})
        lo *= 2
    return out


def config_echo(*, k, nb, tol, maxiter, fom_iters, seed, no_precond, input_echo, variant="sm100a", nd=1,
                threads=1, cache_size=256, vector_width=256):
    """driver.hpp:168-182 (variant: the device kernel's name; threads: host worker threads)."""
    return {"k": k, "nb": nb if nb > 0 else k + 3, "tol": tol, "maxiter": maxiter, "fom_iters": fom_iters,
            "variant": variant, "cache_size": cache_size, "vector_width": vector_width, "nd": nd,
            "threads": threads, "seed": seed, "no_precond": no_precond, "input": input_echo}


def _check_finite(x, path="report"):
    if isinstance(x, float) and not math.isfinite(x):
        raise ValueError(f"{path}: non-finite value in run report")
    if isinstance(x, dict):
        for k, v in x.items():
            _check_finite(v, f"{path}.{k}")
    elif isinstance(x, (list, tuple)):
        for i, v in enumerate(x):
            _check_finite(v, f"{path}[{i}]")


def solve_report(res, *, n, nnz_lower, config, tile_sizes=None, comm=None):
    """The `solve` run report of one abi.lobpcg result (driver.hpp:242-281)."""
    k = config["k"]
    times = res.get("times")
    hist = []
    tot = {"spmm": 0.0, "precond": 0.0, "densela": 0.0, "total": 0.0}
    for i in range(res["iterations"]):
        t = [float(v) for v in times[i]] if times is not None else [0.0, 0.0, 0.0, 0.0]
        hist.append({"iter": i + 1, "theta": [float(v) for v in res["theta"][i]],
                     "residual_norms": [float(v) for v in res["residual_norms"][i]],
                     "n_converged": int(res["n_converged"][i]), "t_spmm": t[0], "t_precond": t[1],
                     "t_dense": t[2], "t_total": t[3]})
        tot["spmm"] += t[0]
        tot["precond"] += t[1]
        tot["densela"] += t[2]
        tot["total"] += t[3]
    j = {"schema": SCHEMA, "command": "solve", "config": config, "n": int(n), "nnz_lower": int(nnz_lower),
         "eigenvalues": [float(v) for v in res["lambda_"]], "converged": bool(res["converged"]),
         "iterations": int(res["iterations"]), "operator_calls": int(res["operator_calls"]), "history": hist}
    if hist:
        j["residual_norms"] = hist[-1]["residual_norms"][:k]
    j["timings"] = tot
    if config.get("nd", 1) > 1 and comm is not None:
        j["comm"] = {"volume_doubles": int(comm["volume_doubles"]), "collective_calls": int(comm["collective_calls"])}
    if not config.get("no_precond") and tile_sizes is not None:
        j["precond_stats"] = {"tiles": len(tile_sizes), "fallbacks": int(res["fallbacks"]),
                              "size_histogram": size_histogram(tile_sizes)}
    j["restarts"] = int(res["restarts"])
    _check_finite(j)
    return j


def dumps(report) -> str:
    """driver.hpp:191-195: two-space indented JSON, one document."""
    _check_finite(report)
    return json.dumps(report, indent=2) + "\n"
