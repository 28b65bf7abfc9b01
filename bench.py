#!/usr/bin/env python
"""LOBPCG hot path benchmark (BASELINE.json metric, Test-1 shape by default).

A step is one LOBPCG iteration (preconditioner, W hygiene, the symmetric
SpMM, Rayleigh-Ritz, updates, residuals) of the device-resident solver on the
Test-1-shaped synthetic Hamiltonian (n = 2.9e6, 1.1e9 stored lower nonzeros,
nev = 8, block k = nb = 16). `value` is throughput in algorithmic GB/s of
that iteration ("Measurement"): B_iter = B_spmm + 40 n nb 8 +
16 * (preconditioner tile entries), B_spmm = 8 nnz + 16 n nb + 8 n, divided
by the device time of the timed iterations (CUDA events on the solver's
stream), summed over ranks. ms_per_step is the LOBPCG iteration time. The
`roofline` object is the SpMM (the dominant kernel) against the measured HBM
copy bandwidth of MEASURED_PEAKS.json.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--config t1|c1|t1random] [--nb 16] [--nev 8] [--precond on|off]
                  [--values f32|f64] [--no-cpu-baseline] [--no-tts]

Input (one node, N = 1): the problem is generated ONCE, in a separate process,
into a CSB1 cache file plus its diagonal section (csb.hpp:204-262,
driver.hpp:136-161) and a tile-offset sidecar, and SHA-256 hashed. The
reference arm reads that file with the reference's own load_csb (through
oracle/_ref/libref.so: libblockeig_b200.so is never loaded in that process);
our arm loads the same file with be_csb_load; both lines carry the hash.
The correctness gate (one device SpMM against the reference's own
SymmetricOperator::apply) runs BEFORE the timed region; a failing gate prints
no value and exits non-zero (driver.hpp:299-373).

Under torchrun (N > 1) the distributed solver runs (weak scaling):
the Test-1-shaped problem is scaled to n = 2.9e6 N rows and 1.1e9 N stored
nonzeros; every rank generates only its nnz-balanced slab of block rows (and
the diagonal blocks of its panel rows for the preconditioner), the X panel is
allgathered and partial Y panels reduce-scattered with NCCL, and the Gram /
norm partials are allreduced. `value` is the whole-job algorithmic bytes per
second; timing is the max over ranks of CUDA-event time.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

CONFIGS = {
    # BASELINE.json configs[1]: Test-1 shape on 1 B200 (clustered generator)
    "t1": dict(kind="clustered", n=2_900_000, nnz=1_100_000_000, extent=4000, tile=128, fill=0.10,
               block_occupancy=1.0),
    # configs[0]: the reference's own CPU-runnable case (generate_synthetic Random)
    "c1": dict(kind="random", n=100_000, nnz=50_000_000, extent=4000),
    # SURVEY 8d stress point: uniform random at the Test-1 size and density (every 128-tile of the
    # lower triangle occupied at fill 2.6e-4, ~4 entries each: the distribution of the reference's
    # Random kind, synth.hpp:109-124, generated block row by block row -- its single mt19937_64
    # stream over 1.1e9 entries would not fit the host)
    "t1random": dict(kind="clustered", n=2_900_000, nnz=1_100_000_000, extent=4000, tile=128, fill=2.616e-4,
                     block_occupancy=1.0),
}
CACHE_DIR = Path(os.environ.get("BE_BENCH_CACHE", "/tmp/blockeig_bench"))


def args_parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", choices=sorted(CONFIGS), default="t1")
    ap.add_argument("--nb", type=int, default=16)
    ap.add_argument("--nev", type=int, default=8)
    ap.add_argument("--precond", choices=["on", "off"], default="on")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-gate", action="store_true", help="skip the correctness gate against the reference SpMM")
    ap.add_argument("--dist", action="store_true", help="run the distributed (NCCL) path even on one rank")
    ap.add_argument("--partition", choices=["2d", "slabs"], default="2d",
                    help="multi-GPU SpMM partition: nnz-balanced 2-D tiles (default) or block-row slabs")
    ap.add_argument("--cpu-iters", type=int, default=2)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--values", choices=["f32", "f64"], default="f32",
                    help="stored matrix values on the device: f32 (8 B/nnz budget) or f64 (12 B/nnz, the reference's precision)")
    ap.add_argument("--no-tts", action="store_true", help="skip the time-to-solution solve (tol 1e-6)")
    ap.add_argument("--report", help="write the time-to-solution solve's run report (blockeig/run-report/v1) here")
    ap.add_argument("--write-cache", help=argparse.SUPPRESS)  # internal: generate the input file in a child process
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def build_problem(cfg, seed):
    from paper_2109_00485_b200 import abi
    if cfg["kind"] == "clustered":
        m, diag, toff = abi.generate_clustered(n=cfg["n"], target_nnz=cfg["nnz"], block_extent=cfg["extent"],
                                               tile=cfg["tile"], fill=cfg["fill"],
                                               block_occupancy=cfg["block_occupancy"], seed=seed)
        return m, diag, toff
    n = cfg["n"]
    s = abi.Synthetic("random", n=n, density=cfg["nnz"] / (n * (n - 1) / 2), block_extent=cfg["extent"], seed=seed)
    b = abi.uniform_boundaries(n, cfg["extent"])
    m = abi.build_csb_coo(s.lower, n, n, b, b)
    return m, s.diag, s.tile_offsets


def cache_paths(config, seed):
    base = CACHE_DIR / f"{config}_seed{seed}"
    return base.with_suffix(".csb1"), base.with_suffix(".tiles"), base.with_suffix(".sha256")


def write_cache(config, seed):
    """(child process) generate the problem with the library's generator and write CSB1 +
    diagonal section (be_csb_save, byte-identical to save_csb + the driver's section), the tile
    offsets sidecar (i64 count, offsets) and the file's SHA-256."""
    import hashlib
    csb, tiles, sha = cache_paths(config, seed)
    CACHE_DIR.mkdir(parents=True, exist_ok=True)
    m, diag, toff = build_problem(CONFIGS[config], seed)
    tmp = csb.with_suffix(".csb1.tmp")
    m.save(tmp, diag)
    toff = np.ascontiguousarray(toff, np.int64)
    with open(tiles, "wb") as f:
        f.write(np.int64(len(toff)).tobytes())
        f.write(toff.tobytes())
    h = hashlib.sha256()
    with open(tmp, "rb") as f:
        while True:
            b = f.read(1 << 26)
            if not b:
                break
            h.update(b)
    os.replace(tmp, csb)
    sha.write_text(json.dumps({"sha256": h.hexdigest(), "bytes": csb.stat().st_size, "nrows": m.nrows,
                               "nnz": m.nnz}))


def ensure_cache(config, seed):
    """The shared input file (generated once, in a separate process); returns its description."""
    csb, tiles, sha = cache_paths(config, seed)
    if not (csb.exists() and tiles.exists() and sha.exists()):
        t0 = time.time()
        subprocess.run([sys.executable, str(ROOT / "bench.py"), "--write-cache", config, "--seed", str(seed)],
                       check=True)
        gen = time.time() - t0
    else:
        gen = 0.0
    d = json.loads(sha.read_text())
    d.update(file=str(csb), tiles=str(tiles), generate_and_write_s=round(gen, 1), format="CSB1 + diagonal section")
    return d


def host_info():
    """lscpu model, physical cores, logical CPUs of the box running the CPU arm."""
    info = {"logical_cpus": os.cpu_count()}
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        kv = dict(line.split(":", 1) for line in out.splitlines() if ":" in line)
        kv = {k.strip(): v.strip() for k, v in kv.items()}
        info["model"] = kv.get("Model name")
        info["physical_cores"] = int(kv.get("Core(s) per socket", "0")) * int(kv.get("Socket(s)", "1"))
        info["threads_per_core"] = int(kv.get("Thread(s) per core", "1"))
    except Exception:
        pass
    return info


def alg_bytes(n, nnz, nb, tile_ent, precond, sv=4):
    """B_spmm = nnz (sv + 4) + 2 n nb 8 + 8 n (matrix once, X and Y panels, diagonal);
    B_iter = B_spmm + 40 n nb 8 + 16 (preconditioner tile entries)."""
    b_spmm = (sv + 4) * nnz + 2 * n * nb * 8 + 8 * n
    b_iter = b_spmm + 40 * n * nb * 8 + (16 * tile_ent if precond else 0)
    return b_spmm, b_iter


class ClockSampler:
    """nvidia-smi clocks and throttle reasons during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.rows = []
        self._stop = threading.Event()
        self._t = None

    def start(self):
        def run():
            while not self._stop.is_set():
                try:
                    out = subprocess.run(["nvidia-smi", "-i", str(self.device), "--query-gpu=" + self.Q,
                                          "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                         timeout=5).stdout.strip()
                    if out:
                        self.rows.append([x.strip() for x in out.split(",")])
                except Exception:
                    pass
                self._stop.wait(0.2)
        self._t = threading.Thread(target=run, daemon=True)
        self._t.start()

    def stop(self):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            for name, v in zip(names, r[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": float(self.rows[0][1]) if self.rows[0][1].replace(".", "").isdigit() else None,
                "reasons": sorted(reasons), "samples": len(self.rows)}


def measured_peak():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        return float(json.loads(p.read_text())["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


def ncu_traffic(config, nb):
    p = ROOT / "profiles" / "spmm_traffic.json"
    if p.exists():
        d = json.loads(p.read_text())
        return d.get(f"{config}_nb{nb}")
    return None


def ref_lib():
    sys.path.insert(0, str(ROOT / "tests"))
    import ctypes as C

    import oracle_lib as ol
    lib = ol.ref()
    if lib is None:
        return None
    lib.ref_prepare_file.restype = C.c_void_p
    lib.ref_prepare_file.argtypes = [C.c_char_p, C.c_char_p, C.c_int]
    lib.ref_prepared_nrows.restype = C.c_int64
    lib.ref_prepared_nrows.argtypes = [C.c_void_p]
    lib.ref_prepared_nnz.restype = C.c_int64
    lib.ref_prepared_nnz.argtypes = [C.c_void_p]
    return lib


def cpu_reference(inp, nev, nb, iters, seed, precond):
    """The reference's own lobpcg_solve (oracle/_ref/libref.so) on all host threads, on the
    problem read from the shared CSB1 file with the reference's load_csb; per-iteration
    IterationRecord::t_total. Returns (times, threads, tile entries, nrows, nnz, load seconds)."""
    lib = ref_lib()
    if lib is None:
        return None
    threads = os.cpu_count() or 1
    t0 = time.time()
    h = lib.ref_prepare_file(inp["file"].encode(), inp["tiles"].encode() if precond else None, threads)
    if not h:
        raise RuntimeError(lib.ref_last_error().decode())
    t_load = time.time() - t0
    try:
        ent = int(lib.ref_tile_entries(h))
        n, nnz = int(lib.ref_prepared_nrows(h)), int(lib.ref_prepared_nnz(h))
        times = np.zeros(iters)
        got = lib.ref_lobpcg_iter_times(h, nev, nb, iters, seed, 1 if precond else 0, times.ctypes.data)
        per = times[:got]
    finally:
        lib.ref_release(h)
    return per, threads, ent, n, nnz, t_load


def correctness_gate(op, m, diag, nb, seed, tol=1e-5):
    """The reference driver's gate (driver.hpp:299-373: no timing for a failing
    output), precision-aware: one device SpMM against the reference's own
    SymmetricOperator::apply (oracle/_ref, f64, all host threads) on the same
    X; pass when the relative Frobenius error is <= 1e-5 (f32 values)."""
    sys.path.insert(0, str(ROOT / "tests"))
    import oracle_lib as ol
    if ol.ref() is None:
        return {"ok": None, "why": "oracle/_ref/libref.so not built"}
    x = np.random.default_rng(seed + 3).uniform(-1, 1, (m.nrows, nb))
    t0 = time.time()
    y = op.apply_host(x)
    want = ol.Impl("ref", threads=os.cpu_count() or 1).spmm(m, diag, x)
    rel = float(np.linalg.norm(y - want) / np.linalg.norm(want))
    return {"ok": rel <= tol, "rel_frobenius": rel, "tol": tol, "seconds": time.time() - t0,
            "vs": "reference SymmetricOperator::apply (f64, oracle/_ref), X = U(-1,1) seed+3"}


def run_reference(a, rank):
    """--impl reference: the reference's CPU LOBPCG iteration on the box's host cores, on the
    shared CSB1 input read by the reference's own loader (this process never loads our library)."""
    if rank != 0:
        return
    cfg = CONFIGS[a.config]
    precond = a.precond == "on"
    inp = ensure_cache(a.config, a.seed)
    res = cpu_reference(inp, a.nev, a.nb, a.warmup + a.steps, a.seed, precond)
    if res is None:
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libref.so not built"}))
        return
    per, threads, ent, n, nnz, t_load = res
    _, b_iter = alg_bytes(n, nnz, a.nb, ent, precond, sv=8)
    timed = per[a.warmup:]
    t = float(np.sum(timed))
    value = b_iter * len(timed) / t / 1e9
    host = host_info()
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": 0, "steps": len(timed),
        "warmup": a.warmup, "ms_per_step": 1e3 * t / len(timed), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic", "config": workload(a, cfg, n, nnz, "f64"),
        "cpu_baseline": {"value": value, "unit": "GB/s", "cores": threads, "kind": "reference", "host": host,
                         "sample": f"{len(timed)} timed reference lobpcg_solve iterations (tol=1e-300, baseline "
                                   f"SpMM variant, ThreadPool({threads}) on {host.get('physical_cores')} physical "
                                   f"cores) after {a.warmup} warm-up iterations"},
        "e2e": {"value": value, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "input": dict(inp, reference_load_s=round(t_load, 1),
                      loaded_with="blockeig::load_csb + driver.hpp:136-161 diagonal section"),
    }
    print(json.dumps(line), flush=True)


METRIC = "LOBPCG iteration time and SpMM achieved HBM GB/s (% of peak) at 1/2/4/8 B200"


def workload(a, cfg, n, nnz, values):
    return {"workload": f"{a.config}: n={n}, half-nnz={nnz}, nev={a.nev}, block k={a.nb}, "
                        f"precond {a.precond}", "n": n, "nnz": nnz, "nb": a.nb, "nev": a.nev,
            "precond": a.precond == "on", "generator": cfg,
            "l2": "inputs larger than L2 (matrix stream >= 8 B/nnz >> 126 MB)", "values": values,
            "panels": "f64"}


def run_dist(a, rank, world, local):
    """Weak-scaled distributed LOBPCG (one rank per GPU, NCCL)."""
    import torch
    import torch.distributed as dist

    from paper_2109_00485_b200 import abi
    torch.cuda.set_device(local)
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29517")
    os.environ.setdefault("RANK", str(rank))
    os.environ.setdefault("WORLD_SIZE", str(world))
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    cfg = dict(CONFIGS[a.config])
    if cfg["kind"] != "clustered":
        raise SystemExit("--gpus > 1 runs the clustered weak-scaling problem (--config t1)")
    n, nnz = cfg["n"] * world, cfg["nnz"] * world
    precond = a.precond == "on"
    p = abi.clustered_params(n=n, target_nnz=nnz, block_extent=cfg["extent"], tile=cfg["tile"], fill=cfg["fill"],
                             block_occupancy=cfg["block_occupancy"], seed=a.seed)
    from paper_2109_00485_b200 import weak
    ctx = abi.Context(local)
    uid = [abi.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(uid, src=0)
    comm = abi.Comm(ctx, nccl_id=uid[0], rank=rank, world=world)

    def allreduce_sum(x):
        t = torch.from_numpy(np.ascontiguousarray(x)).cuda()
        dist.all_reduce(t)
        return t.cpu().numpy()

    t0 = time.time()
    rp = weak.rank_problem(ctx, comm, p, rank, world, precond, allreduce_sum, partition=a.partition)
    t_setup = time.time() - t0
    op, tiles, cuts, lo, hi = rp["op"], rp["tiles"], rp["cuts"], rp["lo"], rp["hi"]
    # this rank's share of the matrix: its 2-D tile (r0, r1, c0, c1) or its block-row slab
    share = rp["rect"] if rp["rect"] is not None else rp["slabs"]
    shares = allreduce_sum(np.eye(world)[rank][:, None] * np.asarray(share, np.float64)[None, :len(share)]) \
        if rp["rect"] is not None else np.asarray(rp["slabs"])
    nnz_local = rp["nnz_local"]
    stats = allreduce_sum(np.array([float(nnz_local), float(rp["tile_entries"])]))
    nnz_tot, ent_tot = int(stats[0]), int(stats[1])
    b_spmm, b_iter = alg_bytes(n, nnz_tot, a.nb, ent_tot, precond)
    stream = torch.cuda.ExternalStream(ctx.stream())
    # correctness gate before timing: the distributed apply must be the symmetric operator --
    # x^T (A y) = y^T (A x) for random x, y (global dots over ranks), and A 1 = D 1 + (L + L^T) 1
    # against the row sums of the rank's own slab and diagonal (computed on the host, summed over
    # ranks), both to the f32 SpMM bar
    gate = None
    if not a.no_gate:
        rng = np.random.default_rng(a.seed + 11 + rank)
        xl, yl = rng.uniform(-1, 1, (hi - lo, 4)), rng.uniform(-1, 1, (hi - lo, 4))
        ax, ay = op.apply_host(xl), op.apply_host(yl)
        dots = allreduce_sum(np.array([np.sum(xl * ay), np.sum(yl * ax), np.sum(ax * ax)]))
        sym = abs(dots[0] - dots[1]) / max(abs(dots[0]), 1e-300)
        ones = op.apply_host(np.ones((hi - lo, 1)))[:, 0]
        sys.path.insert(0, str(ROOT / "tests"))
        import oracle_lib as ol
        rel1 = None
        if ol.ref() is not None:  # (L + L^T) 1 of this rank's slab by the reference's spmm_notrans / spmm_trans
            refi = ol.Impl("ref", threads=max(1, (os.cpu_count() or 1) // world))
            slab = rp["slab_csb"]
            rows1 = refi.spmm(slab, None, np.ones((n, 1)), y=np.zeros((n, 1)), mode=1)
            rows1 = refi.spmm(slab, None, np.ones((n, 1)), y=rows1, mode=2)[:, 0]
            want = allreduce_sum(rows1)[lo:hi] + rp["diag"]
            err = allreduce_sum(np.array([np.sum((ones - want) ** 2), np.sum(want ** 2)]))
            rel1 = float(np.sqrt(err[0] / max(err[1], 1e-300)))
        ok = bool(sym <= 1e-5 and (rel1 is None or rel1 <= 1e-5))
        gate = {"ok": ok, "symmetry_rel": float(sym), "ones_rel_frobenius": rel1, "tol": 1e-5,
                "vs": "x^T A y = y^T A x; A 1 against the reference's spmm_notrans + spmm_trans of every slab + D"}
        if not ok:
            if rank == 0:
                print(json.dumps({"metric": METRIC, "error": "correctness gate failed: no timing reported",
                                  "gate": gate, "n_gpus": world}), flush=True)
            sys.exit(2)
    solver = abi.IncrementalSolve(ctx, op, tiles=tiles, k=a.nev, nb=a.nb, tol=1e-300,
                                  maxiter=a.warmup + a.steps + 1, seed=a.seed)
    solver.step(a.warmup)
    torch.cuda.synchronize()
    dist.barrier()
    clocks = ClockSampler(local)
    clocks.start()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    l0 = ctx.launches()
    ev0.record(stream)
    done = solver.step(a.steps)
    ev1.record(stream)
    torch.cuda.synchronize()
    launches = ctx.launches() - l0
    clk = clocks.stop()
    tt = torch.tensor([ev0.elapsed_time(ev1)], device="cuda")
    dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    t_ms = float(tt.item())
    res = solver.end()
    rec = res["times"][a.warmup:a.warmup + done]
    spmm_ms = 1e3 * float(np.mean(rec[:, 0])) if len(rec) else float("nan")
    peak, peak_kind = measured_peak()
    # roofline of this rank's share of the SpMM (its slab + its panel rows), whole distributed apply
    b_spmm_local = 8 * nnz_local + 2 * (hi - lo) * a.nb * 8 + 8 * (hi - lo)
    ach = b_spmm_local / (spmm_ms * 1e-3) / 1e9
    # end to end through the solve call with host buffers (x0 in, eigenvectors out)
    x0 = np.random.default_rng(a.seed + rank).uniform(-1, 1, (hi - lo, a.nb))
    torch.cuda.synchronize()
    dist.barrier()
    e0 = time.perf_counter()
    r2 = abi.lobpcg(ctx, op, tiles=tiles, x0=x0, k=a.nev, nb=a.nb, tol=1e-300, maxiter=a.steps, seed=a.seed)
    e_s = torch.tensor([time.perf_counter() - e0], device="cuda", dtype=torch.float64)
    dist.all_reduce(e_s, op=dist.ReduceOp.MAX)
    e_s = float(e_s.item())
    info = comm.info()
    line = {
        "metric": METRIC, "value": b_iter * done / (t_ms * 1e-3) / 1e9, "unit": "GB/s", "n_gpus": world,
        "steps": done, "warmup": a.warmup, "ms_per_step": t_ms / max(done, 1), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32 SpMM / f64 dense", "data": "synthetic",
        "config": {"workload": f"t1 weak-scaled x{world}: n={n}, half-nnz={nnz_tot}, nev={a.nev}, block k={a.nb}, "
                               f"precond {a.precond}", "n": n, "nnz": nnz_tot, "nb": a.nb, "nev": a.nev,
                   "precond": precond, "generator": cfg, "parallelism": f"dist{world} (row panels + nnz-balanced "
                   f"SpMM {'2-D tiles' if a.partition == '2d' else 'slabs'}, segment-wise NCCL send/recv exchange, "
                   "allreduce)",
                   "l2": "inputs larger than L2 (matrix stream 8 B/nnz >> 126 MB)", "values": "f32", "panels": "f64"},
        "roofline": {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak,
                     "traffic": None, "kernel": "distributed sym_spmm apply on rank 0 (slab SpMM + exchange)",
                     "bytes_per_launch": b_spmm_local, "ms_per_launch": spmm_ms, "peak_kind": peak_kind},
        "cpu_baseline": None,
        "e2e": {"value": b_iter * r2["iterations"] / e_s / 1e9, "unit": "GB/s",
                "h2d_bytes_per_step": int(x0.nbytes * world / max(r2["iterations"], 1)),
                "d2h_bytes_per_step": int((n * a.nev * 8 + a.nev * 8 * world) / max(r2["iterations"], 1)),
                "iterations": r2["iterations"], "seconds": e_s},
        "gpu_launches": launches,
        "clocks": clk,
        "gate": gate,
        "lobpcg": {"iter_ms": t_ms / max(done, 1), "spmm_ms": spmm_ms,
                   "precond_ms": 1e3 * float(np.mean(rec[:, 1])) if len(rec) else None,
                   "setup_s": {"generate_and_upload": t_setup}, "parallelism": f"dist{world}",
                   "comm": {"backend": info["backend"], "calls": info["calls"], "bytes_rank0": info["bytes"]},
                   "cuts": [int(c) for c in cuts], "partition": a.partition,
                   "shares": np.asarray(shares).astype(np.int64).tolist()},
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    op.close()
    comm.close()
    dist.destroy_process_group()


def main():
    a = args_parse()
    if a.write_cache:
        return write_cache(a.write_cache, a.seed)
    rank, world, local = dist_env()
    if a.impl == "reference":
        return run_reference(a, rank)
    if world > 1 or a.dist:
        return run_dist(a, rank, world, local)
    import torch

    from paper_2109_00485_b200 import abi
    torch.cuda.set_device(local)
    cfg = CONFIGS[a.config]
    precond = a.precond == "on"
    vprec, sv = (abi.BE_F32, 4) if a.values == "f32" else (abi.BE_F64, 8)
    inp = ensure_cache(a.config, a.seed)  # the same bytes the reference arm reads
    ctx = abi.Context(local)
    # the tile-format configuration (T1) is streamed from the file (be_op_create_csb1); the sparse
    # ones (c1, t1random) get the row-list format, which the in-memory build chooses
    stream_build = a.config == "t1"
    t_stream = None
    if stream_build:
        t0 = time.time()
        op, _ = abi.Operator.from_csb1(ctx, inp["file"], values_prec=vprec)
        t_stream = time.time() - t0
    t0 = time.time()
    m, diag = abi.Csb.load(inp["file"])  # the preconditioner tiles and the correctness gate
    toff = np.fromfile(inp["tiles"], dtype=np.int64)[1:]
    t_load = time.time() - t0
    t0 = time.time()
    if not stream_build:
        op = abi.Operator(ctx, m, diag, values_prec=vprec)
    tiles = abi.Tiles(ctx, m, diag, toff) if precond else None
    t_up = time.time() - t0
    n, nnz = m.nrows, m.nnz
    ent = tiles.count()[2] if tiles else 0
    b_spmm, b_iter = alg_bytes(n, nnz, a.nb, ent, precond, sv=sv)
    stream = torch.cuda.ExternalStream(ctx.stream())

    # correctness gate first (driver.hpp:299-373: no timing for a failing output)
    gate = None if a.no_gate else correctness_gate(op, m, diag, a.nb, a.seed, 1e-5 if a.values == "f32" else 1e-12)
    if gate is not None and gate["ok"] is False:
        print(json.dumps({"metric": METRIC, "error": "correctness gate failed: no timing reported", "gate": gate,
                          "n_gpus": world, "config": workload(a, cfg, n, nnz, a.values)}), flush=True)
        sys.exit(2)

    # warm-up + timed iterations of one solve (tol 1e-300 keeps it iterating)
    solver = abi.IncrementalSolve(ctx, op, tiles=tiles, k=a.nev, nb=a.nb, tol=1e-300,
                                  maxiter=a.warmup + a.steps + 1, seed=a.seed)
    solver.step(a.warmup)
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    clocks.start()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    l0 = ctx.launches()
    ev0.record(stream)
    done = solver.step(a.steps)
    ev1.record(stream)
    torch.cuda.synchronize()
    launches = ctx.launches() - l0
    clk = clocks.stop()
    t_ms = ev0.elapsed_time(ev1)
    res = solver.end()
    rec = res["times"][a.warmup:a.warmup + done]
    spmm_ms = 1e3 * float(np.mean(rec[:, 0])) if len(rec) else float("nan")
    ms_step = t_ms / max(done, 1)
    value = world * b_iter * done / (t_ms * 1e-3) / 1e9
    peak, peak_kind = measured_peak()
    ach = b_spmm / (spmm_ms * 1e-3) / 1e9

    # end to end: the reference-facing solve call with host buffers (x0 in, X out)
    x0 = np.random.default_rng(a.seed).uniform(-1, 1, (n, a.nb))
    torch.cuda.synchronize()
    e0 = time.perf_counter()
    r2 = abi.lobpcg(ctx, op, tiles=tiles, x0=x0, k=a.nev, nb=a.nb, tol=1e-300, maxiter=a.steps, seed=a.seed)
    e_s = time.perf_counter() - e0
    e2e_val = world * b_iter * r2["iterations"] / e_s / 1e9

    cpu = None
    if rank == 0 and not a.no_cpu_baseline:
        got = cpu_reference(inp, a.nev, a.nb, a.cpu_iters, a.seed, precond)
        if got is not None:
            per, threads, _, _, _, t_rl = got
            host = host_info()
            cpu = {"value": b_iter / float(np.median(per)) / 1e9, "unit": "GB/s", "cores": threads, "kind": "reference",
                   "host": host, "ms_per_step": 1e3 * float(np.median(per)),
                   "sample": f"{len(per)} reference lobpcg_solve iterations of the same problem read from the same "
                             f"CSB1 file (tol=1e-300, baseline SpMM variant, ThreadPool({threads}) on "
                             f"{host.get('physical_cores')} physical cores of a {host.get('model')}); median "
                             f"iteration {1e3 * float(np.median(per)):.0f} ms"}
    tts = None
    if not a.no_tts:  # time to solution (lobpcg.hpp defaults: tol 1e-6), host buffers in and out
        t0 = time.perf_counter()
        r3 = abi.lobpcg(ctx, op, tiles=tiles, k=a.nev, nb=a.nb, tol=1e-6, maxiter=500, seed=a.seed)
        tts = {"tol": 1e-6, "maxiter": 500, "converged": r3["converged"], "iterations": r3["iterations"],
               "seconds": time.perf_counter() - t0, "lambda_min": float(r3["lambda_"][0]),
               "precond": precond}
        if cpu is not None:
            tts["reference_estimated_s"] = r3["iterations"] * cpu["ms_per_step"] * 1e-3
            tts["reference_estimate"] = "our iteration count x the reference's measured median iteration time"
        if a.report and rank == 0:  # the reference driver's solve report (driver.hpp:242-281)
            from paper_2109_00485_b200 import report
            rcfg = report.config_echo(k=a.nev, nb=a.nb, tol=1e-6, maxiter=500, fom_iters=4, seed=a.seed,
                                      no_precond=not precond, nd=world, variant="sm100a",
                                      input_echo={"gen": cfg["kind"], "n": cfg["n"], "nnz": cfg["nnz"],
                                                  "block_extent": cfg["extent"], "cache": inp.get("file"),
                                                  "cache_hit": True})
            sizes = None
            if tiles is not None:
                sizes = list(np.diff(np.fromfile(inp["tiles"], dtype=np.int64)[1:]))
            Path(a.report).write_text(report.dumps(report.solve_report(r3, n=n, nnz_lower=nnz, config=rcfg,
                                                                       tile_sizes=sizes)))
            tts["run_report"] = a.report
    traffic = ncu_traffic(a.config, a.nb) if a.values == "f32" else None
    line = {
        "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world, "steps": done, "warmup": a.warmup,
        "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": f"{a.values} SpMM / f64 dense", "data": "synthetic", "config": workload(a, cfg, n, nnz, a.values),
        "roofline": {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak,
                     "traffic": traffic, "kernel": "sym_spmm (k_f64_to_f32 + tile or row-list SpMM kernel + k_finish_f64)",
                     "bytes_per_launch": b_spmm, "ms_per_launch": spmm_ms, "peak_kind": peak_kind},
        "cpu_baseline": cpu,
        "e2e": {"value": e2e_val, "unit": "GB/s", "h2d_bytes_per_step": int(x0.nbytes / max(r2["iterations"], 1)),
                "d2h_bytes_per_step": int((n * a.nev * 8 + a.nev * 8) / max(r2["iterations"], 1) + 4 * a.nb * 8),
                "iterations": r2["iterations"], "seconds": e_s},
        "gpu_launches": launches,
        "clocks": clk,
        "gate": gate,
        "time_to_solution": tts,
        "input": dict(inp, our_load_s=round(t_load, 1), loaded_with="be_csb_load"),
        "lobpcg": {"iter_ms": ms_step, "spmm_ms": spmm_ms, "precond_ms": 1e3 * float(np.mean(rec[:, 1])),
                   "setup_s": {"operator_streamed_from_file": t_stream, "load": t_load, "upload": t_up},
                   "parallelism": "1 GPU"},
    }
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
