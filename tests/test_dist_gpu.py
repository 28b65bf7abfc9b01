"""Multi-GPU path on one B200: the ranks are host threads sharing
an in-process communicator group (the same distributed operator / solver code
as under NCCL, only the three collectives differ), plus NCCL at world 1.

Bars: distributed SpMM = single-GPU SpMM = oracle within 1e-5 relative
(fp32 values); distributed LOBPCG eigenvalues within 1e-6 of the oracle and
of the single-GPU solve, iterations within +-1 (preconditioner off; on, within
+-1 of the single-GPU count); the device tile format of every rank decodes
back to exactly its slab's entries."""
import threading

import numpy as np
import pytest

import oracle_lib as ol
from paper_2109_00485_b200 import abi

pytestmark = pytest.mark.gpu


def run_ranks(world, fn):
    group = abi.CommGroup(world)
    out = [None] * world
    errs = []

    def worker(r):
        try:
            ctx = abi.Context(0)
            comm = abi.Comm(ctx, group=group, rank=r)
            out[r] = fn(r, ctx, comm)
            comm.close()
            ctx.close()
        except BaseException as e:  # noqa: BLE001
            errs.append((r, e))
            group.abort()  # peers blocked in a collective fail with ProtocolDeadlock instead of hanging

    ts = [threading.Thread(target=worker, args=(r,), daemon=True) for r in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout=600)
    if errs:
        first = [e for _, e in errs if not isinstance(e, abi.ProtocolDeadlock)] or [errs[0][1]]
        raise first[0]
    assert not any(t.is_alive() for t in ts), "a rank did not finish"
    group.close()
    return out


def problem(n=6000, density=0.004, extent=1000, seed=3):
    s = abi.Synthetic("random", n=n, density=density, block_extent=extent, seed=seed)
    b = abi.uniform_boundaries(n, extent)
    m = abi.build_csb_coo(s.lower, n, n, b, b)
    return m, s.diag, s.tile_offsets


def partition(m, world):
    cuts = abi.dist_rows(m.row_offsets, world)
    slabs = abi.dist_balance(m.block_row_nnz(), world)
    return cuts, slabs


@pytest.mark.parametrize("world", [2, 3, 4, 8])
def test_dist_spmm_matches_single_and_oracle(ctx, world):
    """Segment-wise exchange: X segments travel only to the ranks whose slab touches
    them, partial Y segments only to their owners; the result equals the single-GPU SpMM and the
    oracle, the exchange plan is the C++ rule (be_dist_touched) on every rank, and the bytes moved
    stay below the full-panel allgather + reduce-scatter it replaced."""
    m, diag, _ = problem(extent=500 if world > 4 else 1000)
    n, nb = m.nrows, 16
    x = np.random.default_rng(5).uniform(-1, 1, (n, nb))
    cuts, slabs = partition(m, world)

    def rank(r, c, comm):
        slab = m.slab(int(slabs[r]), int(slabs[r + 1]))
        op = abi.DistOperator(c, comm, slab, cuts, diag[cuts[r]:cuts[r + 1]])
        y = op.apply_host(x[cuts[r]:cuts[r + 1]])
        y2 = op.apply_host(x[cuts[r]:cuts[r + 1]])  # the exchange buffers are reused
        info = comm.info()
        need = op.need()
        op.close()
        return y, y2, info, need, abi.dist_touched(slab, cuts, world)

    res = run_ranks(world, rank)
    y = np.vstack([a[0] for a in res])
    assert all(np.array_equal(a, b) or np.linalg.norm(a - b) <= 1e-6 * np.linalg.norm(a) for a, b, *_ in res)
    want = ol.Impl("orc").spmm(m, diag, x)
    single = abi.Operator(ctx, m, diag).apply_host(x)
    assert np.linalg.norm(y - want) / np.linalg.norm(want) <= 1e-5
    assert np.linalg.norm(y - single) / np.linalg.norm(single) <= 1e-6
    need = np.array([t for *_, t in res])  # the host rule, rank by rank
    assert all(np.array_equal(r[3], need) for r in res)  # every rank built the same plan from its tiles
    # slab p (rows [s_p, s_p+1), columns below s_p+1) touches exactly the segments starting before its end
    for p in range(world):
        if slabs[p + 1] > slabs[p]:
            end = m.row_offsets[int(slabs[p + 1])]
            assert np.array_equal(need[p], cuts[:-1] < end) or need[p].sum() <= (cuts[:-1] < end).sum()
    lmax = int(np.max(np.diff(cuts)))
    full = 2 * 2 * (world - 1) * lmax * nb * 4  # two applies of AG + RS, bytes each rank received
    assert all(i["backend"] == "local" and i["calls"] == 1 + 2 * (1 + world) for _, _, i, *_ in res)  # setup + 2 x (X + one Y call per segment)
    if world > 2:
        assert sum(i["bytes"] for _, _, i, *_ in res) < world * full


@pytest.mark.parametrize("world", [2, 4, 8])
def test_dist_spmm_2d_tiles_match_single_and_oracle(ctx, world):
    """North_star's partition: every rank holds an nnz-balanced 2-D tile of blocks
    (be_dist_tiles2d) instead of a block-row slab; the panels stay equal-row segments. The
    distributed SpMM equals the single-GPU SpMM and the oracle, each rank's exchange plan is the
    host rule on its tile, and no rank exchanges more segments than with slabs."""
    m, diag, _ = problem(extent=500 if world > 4 else 1000)
    n, nb = m.nrows, 16
    x = np.random.default_rng(6).uniform(-1, 1, (n, nb))
    cuts, slabs = partition(m, world)
    rects = abi.dist_tiles2d(m.block_weights(), m.row_offsets, world)

    def rank(r, c, comm):
        tile = m.rect(*(int(v) for v in rects[r]))
        op = abi.DistOperator(c, comm, tile, cuts, diag[cuts[r]:cuts[r + 1]])
        y = op.apply_host(x[cuts[r]:cuts[r + 1]])
        need = op.need()
        op.close()
        return y, need, abi.dist_touched(tile, cuts, world), tile.nnz

    res = run_ranks(world, rank)
    y = np.vstack([a[0] for a in res])
    assert sum(a[3] for a in res) == m.nnz
    want = ol.Impl("orc").spmm(m, diag, x)
    single = abi.Operator(ctx, m, diag).apply_host(x)
    assert np.linalg.norm(y - want) / np.linalg.norm(want) <= 1e-5
    assert np.linalg.norm(y - single) / np.linalg.norm(single) <= 1e-6
    need = np.array([a[2] for a in res])
    assert all(np.array_equal(a[1], need) for a in res)
    need1d = np.array([abi.dist_touched(m.slab(int(slabs[p]), int(slabs[p + 1])), cuts, world) for p in range(world)])
    assert need.sum() <= need1d.sum()


def test_dist_decode_is_the_slab(ctx):
    m, diag, _ = problem(n=3000, extent=500)
    world = 3
    cuts, slabs = partition(m, world)
    trip = m.to_triples()

    def rank(r, c, comm):
        sl = m.slab(int(slabs[r]), int(slabs[r + 1]))
        op = abi.DistOperator(c, comm, sl, cuts, diag[cuts[r]:cuts[r + 1]], values_prec=abi.BE_F32)
        rows, cols, vals, idx = op.decode()
        st = sl.to_triples()
        op.close()
        return rows, cols, vals, idx, st

    res = run_ranks(world, rank)
    total = 0
    for rows, cols, vals, idx, st in res:
        # device entry -> slab CSB index -> the same (row, col, f32(value))
        assert np.array_equal(rows, st["row"][idx]) and np.array_equal(cols, st["col"][idx])
        assert np.array_equal(vals, st["value"][idx].astype(np.float32).astype(np.float64))
        assert np.array_equal(np.sort(idx), np.arange(len(st)))
        total += len(st)
    assert total == len(trip)


def test_dist_rejects_misaligned_cuts(ctx):
    m, diag, _ = problem(n=3000, extent=500)

    def rank(r, c, comm):
        cuts = np.array([0, 1234, 3000])  # 1234 is not a block boundary
        with pytest.raises(abi.MisalignedTiles):
            abi.DistOperator(c, comm, m.slab(0, 6) if r == 0 else m.slab(6, 6), cuts, diag[:1234] if r == 0 else diag[1234:])
        return True

    assert all(run_ranks(2, rank))


@pytest.mark.parametrize("precond", [False, True])
@pytest.mark.parametrize("world", [2, 3])
def test_dist_lobpcg_matches_single(ctx, world, precond):
    m, diag, toff = problem(n=6000, density=0.003, extent=1000, seed=11)
    n, k, nb = m.nrows, 8, 16
    cuts, slabs = partition(m, world)
    tiles = abi.Tiles(ctx, m, diag, toff) if precond else None
    single = abi.lobpcg(ctx, abi.Operator(ctx, m, diag), tiles=tiles, k=k, nb=nb, tol=1e-6, maxiter=300, seed=1)
    want = ol.Impl("orc").lobpcg(m, diag, k=k, nb=nb, tol=1e-6, maxiter=300, seed=1,
                                 toff=toff if precond else None)

    def rank(r, c, comm):
        op = abi.DistOperator(c, comm, m.slab(int(slabs[r]), int(slabs[r + 1])), cuts, diag[cuts[r]:cuts[r + 1]])
        t = abi.Tiles(c, m, diag[cuts[r]:cuts[r + 1]], toff, row_range=(int(cuts[r]), int(cuts[r + 1]))) \
            if precond else None
        res = abi.lobpcg(c, op, tiles=t, k=k, nb=nb, tol=1e-6, maxiter=300, seed=1)
        op.close()
        return res

    res = run_ranks(world, rank)
    lam = res[0]["lambda_"]
    assert all(np.array_equal(r["lambda_"], lam) for r in res)  # identical decisions on every rank
    assert all(r["iterations"] == res[0]["iterations"] for r in res)
    assert res[0]["converged"]
    assert np.max(np.abs(lam - want["lambda_"]) / np.abs(want["lambda_"])) <= 1e-6
    assert np.max(np.abs(lam - single["lambda_"]) / np.abs(single["lambda_"])) <= 1e-6
    its = res[0]["iterations"]
    if not precond:
        assert abs(its - single["iterations"]) <= 1
        assert abs(its - want["iterations"]) <= 1
    else:  # the count follows the summation order: the reference's envelope + the single-GPU solve, +-1
        from test_lobpcg_gpu import envelope
        lo, hi = envelope(m, diag, toff, k=k, nb=nb, tol=1e-6, maxiter=300, seed=1)
        lo, hi = min(lo, single["iterations"]), max(hi, single["iterations"])
        # (the envelope samples the reference over ThreadPool(1..8) x {baseline, fused-atomic})
        assert lo - 1 <= its <= hi + 1, (its, lo, hi)
    # the distributed eigenvectors are the single-GPU ones, row-partitioned
    x = np.vstack([r["x"] for r in res])
    for v in range(k):
        a, b = x[:, v], single["x"][:, v]
        cos = abs(a @ b) / (np.linalg.norm(a) * np.linalg.norm(b))
        assert cos > 1 - 1e-6


def test_dist_x0_slices_match_global_random_block(ctx):
    """X0 of rank r is rows [cuts[r], cuts[r+1]) of random_block(n, nb, seed)
    (block_vector.hpp:47-53): one solve step from the same start agrees."""
    m, diag, _ = problem(n=3000, density=0.004, extent=500, seed=2)
    world, k, nb = 2, 4, 8
    cuts, slabs = partition(m, world)
    single = abi.lobpcg(ctx, abi.Operator(ctx, m, diag), k=k, nb=nb, tol=1e-300, maxiter=1, seed=9)

    def rank(r, c, comm):
        op = abi.DistOperator(c, comm, m.slab(int(slabs[r]), int(slabs[r + 1])), cuts, diag[cuts[r]:cuts[r + 1]])
        res = abi.lobpcg(c, op, k=k, nb=nb, tol=1e-300, maxiter=1, seed=9)
        op.close()
        return res

    res = run_ranks(world, rank)
    other = abi.lobpcg(ctx, abi.Operator(ctx, m, diag), k=k, nb=nb, tol=1e-300, maxiter=1, seed=10)
    # same start: Ritz values agree to f32-SpMM rounding; another seed's start is far off
    assert np.allclose(res[0]["theta"][0], single["theta"][0], rtol=1e-7, atol=0)
    assert not np.allclose(other["theta"][0], single["theta"][0], rtol=1e-4, atol=0)


def test_failing_rank_releases_peers(ctx):
    """A rank that fails before a collective must not hang the others: they
    get ProtocolDeadlock (dist.hpp:256-263), the failure itself surfaces."""
    m, diag, _ = problem(n=3000, extent=500)
    cuts, slabs = partition(m, 2)

    def rank(r, c, comm):
        if r == 1:
            raise abi.BadParams("rank 1 gives up")
        op = abi.DistOperator(c, comm, m.slab(int(slabs[r]), int(slabs[r + 1])), cuts, diag[cuts[r]:cuts[r + 1]])
        op.apply_host(np.zeros((int(cuts[1] - cuts[0]), 4)))

    with pytest.raises(abi.BadParams):
        run_ranks(2, rank)


def test_nccl_world1(ctx):
    m, diag, _ = problem(n=3000, extent=500)
    uid = abi.nccl_unique_id()
    comm = abi.Comm(ctx, nccl_id=uid, rank=0, world=1)
    cuts = np.array([0, m.nrows])
    op = abi.DistOperator(ctx, comm, m, cuts, diag)
    x = np.random.default_rng(1).uniform(-1, 1, (m.nrows, 16))
    y = op.apply_host(x)
    want = abi.Operator(ctx, m, diag).apply_host(x)
    assert np.linalg.norm(y - want) / np.linalg.norm(want) <= 1e-6
    assert comm.info()["backend"] == "nccl"
    res = abi.lobpcg(ctx, op, k=4, nb=8, tol=1e-6, maxiter=200, seed=1)
    ref = abi.lobpcg(ctx, abi.Operator(ctx, m, diag), k=4, nb=8, tol=1e-6, maxiter=200, seed=1)
    assert np.allclose(res["lambda_"], ref["lambda_"], rtol=1e-9)
    op.close()
    comm.close()


@pytest.mark.parametrize("partition", ["2d", "slabs"])
@pytest.mark.parametrize("world", [2, 3])
def test_weak_scaling_glue_matches_whole_matrix(ctx, world, partition):
    """The bench's per-rank problem construction (weak.rank_problem: slab and
    diagonal-block generation, the summed |row| diagonal, rank-range tiles)
    solves the same problem as the whole matrix on one GPU."""
    from paper_2109_00485_b200 import weak
    kw = dict(n=24000, target_nnz=3_000_000, block_extent=2000, seed=3)
    p = abi.clustered_params(**kw)
    whole, diag, toff = abi.generate_clustered(**kw)
    # tol 3e-5: with the FOM preconditioner this clustered problem has a residual floor near 3e-6
    # relative -- the reference's own preconditioned solve (oracle/_ref, f64) stalls at maxiter
    # for tol 1e-6 too (no preconditioner: converges) -- so the tolerance sits well above it
    single = abi.lobpcg(ctx, abi.Operator(ctx, whole, diag), tiles=abi.Tiles(ctx, whole, diag, toff), k=8, nb=16,
                        tol=3e-5, maxiter=300, seed=1)
    slots = [None] * world
    bar = threading.Barrier(world)

    def rank(r, c, comm):
        def allreduce_sum(x):  # host-side sum over the rank threads, in rank order
            slots[r] = x
            bar.wait()
            out = slots[0].copy()
            for q in range(1, world):
                out += slots[q]
            bar.wait()
            return out

        rp = weak.rank_problem(c, comm, p, r, world, True, allreduce_sum, partition=partition)
        assert np.allclose(rp["diag"], diag[rp["lo"]:rp["hi"]], rtol=1e-13, atol=0)
        res = abi.lobpcg(c, rp["op"], tiles=rp["tiles"], k=8, nb=16, tol=3e-5, maxiter=300, seed=1)
        rp["op"].close()
        return res

    res = run_ranks(world, rank)
    assert single["converged"] and res[0]["converged"]
    assert np.max(np.abs(res[0]["lambda_"] - single["lambda_"]) / single["lambda_"]) <= 1e-6
    # preconditioned iteration counts follow the summation order: both counts inside the
    # reference's own ThreadPool(1..8) x variant envelope of this problem, +-1
    from test_lobpcg_gpu import envelope
    lo, hi = envelope(whole, diag, toff, k=8, nb=16, tol=3e-5, maxiter=300, seed=1)
    assert lo - 1 <= res[0]["iterations"] <= hi + 1, (res[0]["iterations"], lo, hi)
    assert lo - 1 <= single["iterations"] <= hi + 1, (single["iterations"], lo, hi)


@pytest.mark.parametrize("nd", [1, 3])
def test_triangular_layout_parity_variant(ctx, nd):
    """The reference's own layout (dist.hpp, nd(nd+1)/2 ranks: 1 and 6) on the
    device path: each rank holds partition_matrix's stored block and owns its
    segment_of_rank; the SpMM matches the oracle and the distributed LOBPCG
    the single-GPU solve."""
    m, diag, _ = problem(n=6000, density=0.003, extent=1000, seed=21)
    n, nb = m.nrows, 16
    world = nd * (nd + 1) // 2
    sub = [n * g // nd for g in range(nd + 1)]
    beg, end = abi.tri_segments(nd, sub)
    x = np.random.default_rng(2).uniform(-1, 1, (n, nb))
    single = abi.lobpcg(ctx, abi.Operator(ctx, m, diag), k=8, nb=nb, tol=1e-6, maxiter=300, seed=1)

    def rank(r, c, comm):
        slab, seg_bounds, owner, d = abi.tri_rank_problem(m, diag, nd, sub, r, extent=1000)
        op = abi.DistOperator(c, comm, slab, seg_bounds, d, owner=owner)
        y = op.apply_host(x[beg[r]:end[r]])
        res = abi.lobpcg(c, op, k=8, nb=nb, tol=1e-6, maxiter=300, seed=1)
        op.close()
        return y, res

    out = run_ranks(world, rank)
    y = np.zeros((n, nb))
    for r, (yr, _) in enumerate(out):
        y[beg[r]:end[r]] = yr
    want = ol.Impl("orc").spmm(m, diag, x)
    assert np.linalg.norm(y - want) / np.linalg.norm(want) <= 1e-5
    res = out[0][1]
    assert np.max(np.abs(res["lambda_"] - single["lambda_"]) / single["lambda_"]) <= 1e-6
    assert abs(res["iterations"] - single["iterations"]) <= 1
