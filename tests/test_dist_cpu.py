"""CPU checks of the multi-GPU path's host logic (no device calls):

* the C++ partition rules (be_dist_rows / be_dist_balance) agree bit-exactly
  with the plain-Python restatement in dist_model.py on many shapes;
* CSB slabs of the balanced cut reassemble exactly to the input matrix (the
  reassembly oracle of test_dist.cpp:146-153);
* world-size-2 `gloo` run of the exchange scheme: every rank builds its slab's
  partial Y over the padded layout from the allgathered X segments, the
  reduce-scatter hands each rank its rows, and the concatenation equals the
  full symmetric SpMM of the oracle restatement.
"""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest

import dist_model as dm
from paper_2109_00485_b200 import abi


def test_partition_rules_match_restatement():
    rng = np.random.default_rng(0)
    for _ in range(200):
        nblk = int(rng.integers(1, 40))
        ext = rng.integers(1, 5000, nblk)
        bounds = np.concatenate([[0], np.cumsum(ext)])
        for world in range(1, min(nblk, 9) + 1):
            assert np.array_equal(abi.dist_rows(bounds, world), dm.dist_rows(bounds, world))
        w = rng.integers(0, 10 ** int(rng.integers(1, 11)), nblk)
        if rng.random() < 0.2:
            w[rng.integers(0, nblk, max(1, nblk // 3))] = 0
        for world in range(1, 10):
            c = abi.dist_balance(w, world)
            assert np.array_equal(c, dm.dist_balance(w, world))
            assert c[0] == 0 and c[-1] == nblk and np.all(np.diff(c) >= 0)


def test_partition_edge_cases():
    with pytest.raises(abi.BadParams):
        abi.dist_rows([0, 10, 20], 3)  # fewer block rows than ranks
    assert list(abi.dist_rows([0, 10], 1)) == [0, 10]
    assert list(abi.dist_balance([], 3)) == [0, 0, 0, 0]
    assert list(abi.dist_balance([0, 0, 0], 2)) == [0, 0, 3]
    # T1-like weights: the nnz balance of a lower triangle puts more block rows on rank 0
    w = np.arange(1, 726) * 1000
    c = abi.dist_balance(w, 8)
    assert np.all(np.diff(c)[:-1] >= np.diff(c)[1:] - 1)


def test_slabs_reassemble_exactly():
    n = 2000
    s = abi.Synthetic("random", n=n, density=0.01, block_extent=300, seed=4)
    b = abi.uniform_boundaries(n, 300)
    m = abi.build_csb_coo(s.lower, n, n, b, b)
    full = m.to_triples()
    for world in (1, 2, 3, 5):
        cuts = abi.dist_balance(m.block_row_nnz(), world)
        parts = [m.slab(int(cuts[r]), int(cuts[r + 1])).to_triples() for r in range(world)]
        assert sum(len(p) for p in parts) == len(full)
        assert np.array_equal(np.concatenate(parts), full)  # block row-major order is preserved


def _free_port():
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def _gloo_rank(rank, world, port, n, nb, partition="slabs"):
    """One rank of the segment-wise exchange of the distributed operator on CPU
    with gloo: the C++ rule (be_dist_touched) decides which X segments travel where and which
    partial Y segments go to which owner; the partial SpMM of the slab is the restated model
    (tests/dist_model.py); the owner sums the partials in ascending rank order."""
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    s = abi.Synthetic("random", n=n, density=0.01, block_extent=250, seed=7)
    b = abi.uniform_boundaries(n, 250)
    m = abi.build_csb_coo(s.lower, n, n, b, b)
    cuts = abi.dist_rows(m.row_offsets, world)
    slabs = abi.dist_balance(m.block_row_nnz(), world)
    lmax = int(np.max(np.diff(cuts)))
    x = np.random.default_rng(1).uniform(-1, 1, (n, nb))
    if partition == "2d":  # this rank's nnz-balanced 2-D tile (be_dist_tiles2d)
        slab = m.rect(*(int(v) for v in abi.dist_tiles2d(m.block_weights(), m.row_offsets, world)[rank]))
    else:
        slab = m.slab(int(slabs[rank]), int(slabs[rank + 1]))
    mine = abi.dist_touched(slab, cuts, world)
    allt = [None] * world
    dist.all_gather_object(allt, mine.tolist())
    need = np.array(allt, dtype=bool)  # need[p, r]: rank p's slab touches segment r
    # X: my segment to the ranks that touch it, the touched segments from their owners
    xpad = np.zeros((world * lmax, nb))
    xpad[rank * lmax: rank * lmax + cuts[rank + 1] - cuts[rank]] = x[cuts[rank]:cuts[rank + 1]]
    reqs, bufs = [], {}
    mine_t = torch.from_numpy(np.ascontiguousarray(xpad[rank * lmax:(rank + 1) * lmax]).ravel())
    for p in range(world):
        if p == rank:
            continue
        if need[p, rank]:
            reqs.append(dist.isend(mine_t, p))
        if need[rank, p]:
            bufs[p] = torch.zeros(lmax * nb, dtype=torch.float64)
            reqs.append(dist.irecv(bufs[p], p))
    for q in reqs:
        q.wait()
    for p, buf in bufs.items():
        xpad[p * lmax:(p + 1) * lmax] = buf.numpy().reshape(lmax, nb)
    t = slab.to_triples()
    ypart = dm.slab_partial_spmm(t["row"], t["col"], t["value"], xpad.ravel(), cuts, nb).reshape(world * lmax, nb)
    # the slab only writes the segments it touches (the rule is exact, not conservative)
    for r in range(world):
        if not need[rank, r]:
            assert not np.any(ypart[r * lmax:(r + 1) * lmax])
    # Y: partial segments to their owners; mine summed in ascending rank order
    reqs, parts = [], {}
    for p in range(world):
        if p == rank:
            continue
        if need[rank, p]:
            reqs.append(dist.isend(torch.from_numpy(np.ascontiguousarray(ypart[p * lmax:(p + 1) * lmax]).ravel()), p))
        if need[p, rank]:
            parts[p] = torch.zeros(lmax * nb, dtype=torch.float64)
            reqs.append(dist.irecv(parts[p], p))
    for q in reqs:
        q.wait()
    acc = None
    for p in range(world):
        v = ypart[rank * lmax:(rank + 1) * lmax] if p == rank else (parts[p].numpy().reshape(lmax, nb) if p in parts else None)
        if v is not None:
            acc = v.copy() if acc is None else acc + v
    nl = cuts[rank + 1] - cuts[rank]
    y = acc[:nl] + s.diag[cuts[rank]:cuts[rank + 1], None] * x[cuts[rank]:cuts[rank + 1]]
    got = [None] * world
    dist.all_gather_object(got, y)
    dist.destroy_process_group()
    if rank == 0:
        import oracle_lib as ol
        want = ol.Impl("orc").spmm(m, s.diag, x)
        yy = np.vstack(got)
        err = np.linalg.norm(yy - want) / np.linalg.norm(want)
        assert err < 1e-13, err


@pytest.mark.parametrize("partition", ["slabs", "2d"])
@pytest.mark.parametrize("world", [2, 3])
def test_gloo_exchange_matches_oracle(world, partition):
    import torch.multiprocessing as mp
    mp.spawn(_gloo_rank, args=(world, _free_port(), 1500, 8, partition), nprocs=world, join=True)


def test_clustered_parts_reassemble_the_matrix():
    """Each rank generates only its block rows (weak-scaling bench): the parts
    are exactly the whole-matrix generator's entries, the summed |row| parts
    give its diagonal, and the expected weights track the real counts."""
    p = abi.clustered_params(n=9000, target_nnz=2_000_000, block_extent=1000, seed=5)
    whole, diag, toff = abi.generate_clustered(n=9000, target_nnz=2_000_000, block_extent=1000, seed=5)
    w = abi.clustered_weights(p)
    cuts = abi.dist_balance(w, 3)
    parts, absum = [], np.zeros(9000)
    for r in range(3):
        m, rowabs, t = abi.generate_clustered_part(p, int(cuts[r]), int(cuts[r + 1]))
        assert np.array_equal(t, toff)
        parts.append(m.to_triples())
        absum += rowabs
    assert np.array_equal(np.concatenate(parts), whole.to_triples())
    d = abi.clustered_diag(p, absum, 0, 9000)
    assert np.allclose(d, diag, rtol=1e-13, atol=0)
    one, rowabs, _ = abi.generate_clustered_part(p, 0, len(w))
    assert np.array_equal(abi.clustered_diag(p, rowabs, 0, 9000), diag)  # one part: bit-exact
    real = whole.block_row_nnz()
    assert abs(real.sum() - w.sum()) / w.sum() < 0.02
    dg, _, _ = abi.generate_clustered_part(p, 2, 5, diag_blocks_only=True)
    t = dg.to_triples()
    b = whole.row_offsets
    blk = lambda x: np.searchsorted(b, x, side="right") - 1
    assert np.all(blk(t["row"]) == blk(t["col"])) and np.all((blk(t["row"]) >= 2) & (blk(t["row"]) < 5))


# ---- the reference's triangular layout (dist.hpp), restated bit-exactly
def test_tri_layout_known_answers():  # test_dist.cpp:86-117
    blocks, dr = abi.tri_layout(1)
    assert blocks.tolist() == [[0, 0, 0]] and dr.tolist() == [0]
    blocks, dr = abi.tri_layout(5)
    assert len(blocks) == 15
    assert {(i, j) for i, j, t in blocks if t} == {(0, 3), (0, 4), (1, 4)}
    rank_of = {(int(i), int(j)): r for r, (i, j, _) in enumerate(blocks)}
    assert [rank_of[(0, 0)], rank_of[(1, 0)], rank_of[(2, 0)], rank_of[(1, 1)], rank_of[(0, 3)], rank_of[(4, 4)]] == \
        [0, 1, 2, 3, 9, 14]
    for nd in (0, 2, -3):
        with pytest.raises(abi.EvenNd):
            abi.tri_layout(nd)


def test_tri_layout_matches_reference():
    import oracle_lib as ol
    if ol.ref() is None:
        pytest.skip("reference build absent")
    for nd in (1, 3, 5, 7, 9):
        b, d = abi.tri_layout(nd)
        rb, rd = ol.ref_build_layout(nd)
        assert np.array_equal(b, rb) and np.array_equal(d, rd)


@pytest.mark.parametrize("nd", [1, 3, 5])
def test_tri_partition_matches_reference(nd):
    """Every rank's stored entries and segment equal partition_matrix's
    (dist.hpp:113-198), entries compared as multisets in global coordinates
    (test_dist.cpp:146-153's reassembly rule); together they are the input."""
    import oracle_lib as ol
    if ol.ref() is None:
        pytest.skip("reference build absent")
    n = 900
    s = abi.Synthetic("random", n=n, density=0.01, block_extent=300, seed=8)
    b = abi.uniform_boundaries(n, 300)
    m = abi.build_csb_coo(s.lower, n, n, b, b)
    sub = [n * g // nd for g in range(nd + 1)]
    beg, end = abi.tri_segments(nd, sub)
    key = lambda r, c, v: sorted(zip(r.tolist(), c.tolist(), v.tolist()))
    total = 0
    for rank in range(nd * (nd + 1) // 2):
        t = abi.tri_rank_triples(m, nd, sub, rank)
        rr, rc, rv, seg = ol.ref_partition_rank(m, s.diag, nd, sub, 64, rank)
        assert key(t["row"], t["col"], t["value"]) == key(rr, rc, rv)
        assert (int(beg[rank]), int(end[rank])) == seg
        total += len(t)
    assert total == m.nnz


def test_csb1_slab_loader(tmp_path):
    """A rank reads only its block rows of a CSB1 cache (csb.hpp:204-302 format,
    driver.hpp:136-161 diagonal section): same arrays as slicing the whole matrix."""
    n = 2500
    s = abi.Synthetic("random", n=n, density=0.01, block_extent=400, seed=12)
    b = abi.uniform_boundaries(n, 400)
    m = abi.build_csb_coo(s.lower, n, n, b, b)
    path = tmp_path / "h.csb"
    m.save(path, s.diag)
    for b0, b1 in [(0, 7), (0, 3), (2, 5), (6, 7), (4, 4)]:
        got, d = abi.Csb.load_rows(path, b0, b1)
        want = m.slab(b0, b1)
        for f in ("row_offsets", "col_offsets", "block_nnz", "block_nnz_offsets", "local_rows", "local_cols", "values"):
            assert np.array_equal(getattr(got, f), getattr(want, f)), f
        lo, hi = int(b[b0]), int(b[b1])
        if hi > lo:
            assert np.array_equal(d, s.diag[lo:hi])


# ---- nnz-balanced 2-D tiles (be_dist_tiles2d) -----------------------------------------------
def _lower_weights(rng, nblk, kind):
    if kind == "uniform":
        w = np.full((nblk, nblk), 100, np.int64)
    elif kind == "random":
        w = rng.integers(0, 1000, (nblk, nblk))
    else:  # sparse: most blocks empty
        w = rng.integers(0, 1000, (nblk, nblk)) * (rng.random((nblk, nblk)) < 0.15)
    return np.tril(w).astype(np.int64)


def test_tiles2d_matches_restatement_and_covers():
    rng = np.random.default_rng(3)
    for trial in range(120):
        nblk = int(rng.integers(1, 24))
        w = _lower_weights(rng, nblk, ("uniform", "random", "sparse")[trial % 3])
        bounds = np.concatenate([[0], np.cumsum(rng.integers(1, 3000, nblk))])
        for world in (1, 2, 3, 4, 5, 8, 16):
            got = abi.dist_tiles2d(w, bounds, world)
            assert np.array_equal(got, dm.dist_tiles2d(w, bounds, world)), (trial, world)
            owner = -np.ones((nblk, nblk), np.int64)
            for r, (r0, r1, c0, c1) in enumerate(got):
                blk = owner[r0:r1, c0:c1]
                assert np.all((blk == -1) | (np.tril(w)[r0:r1, c0:c1] == 0)), "rectangles overlap"
                blk[np.tril(w)[r0:r1, c0:c1] > 0] = r
            assert np.all(owner[w > 0] >= 0), "a non-empty block has no rank"


def test_tiles2d_balance_and_exchange_volume():
    """On the clustered generator's T1-shaped block weights (scaled down): every rank's tile is
    within 2 % of the ideal nnz share, and the panel segments a rank's SpMM exchanges (rows or
    columns it touches) are fewer than with block-row slabs for the heaviest rank."""
    p = abi.clustered_params(n=290_000, target_nnz=110_000_000, block_extent=1000, seed=1)
    w = abi.clustered_block_weights(p)
    bounds = abi.uniform_boundaries(p.n, p.block_extent)
    assert abs(np.tril(w).sum() - abi.clustered_weights(p).sum()) / w.sum() < 1e-3
    for world in (2, 4, 8):
        rects = abi.dist_tiles2d(w, bounds, world)
        share = np.array([np.tril(w)[r0:r1, c0:c1].sum() for r0, r1, c0, c1 in rects])
        assert share.sum() == np.tril(w).sum()
        assert share.max() <= 1.02 * share.sum() / world, (world, share)
        cuts = abi.dist_rows(bounds, world)
        t2d = [len(dm.touched_segments(w, bounds, cuts, r)) for r in rects]
        slabs = abi.dist_balance(w.sum(axis=1), world)
        t1d = [len(dm.touched_segments(w, bounds, cuts, (slabs[r], slabs[r + 1], 0, len(w)))) for r in range(world)]
        assert sum(t2d) <= sum(t1d) and max(t2d) <= max(t1d), (world, t2d, t1d)


def test_clustered_tiles_reassemble_the_matrix():
    """Each rank generates only its 2-D tile: the tiles are exactly the whole-matrix generator's
    entries and the summed |row| parts give its diagonal."""
    kw = dict(n=9000, target_nnz=2_000_000, block_extent=1000, seed=5)
    p = abi.clustered_params(**kw)
    whole, diag, toff = abi.generate_clustered(**kw)
    bounds = abi.uniform_boundaries(9000, 1000)
    rects = abi.dist_tiles2d(abi.clustered_block_weights(p), bounds, 4)
    trip, absum = [], np.zeros(9000)
    for r0, r1, c0, c1 in rects:
        m, rowabs, t = abi.generate_clustered_tile(p, (int(r0), int(r1)), (int(c0), int(c1)))
        assert np.array_equal(t, toff)
        assert np.array_equal(m.to_triples(), whole.rect(int(r0), int(r1), int(c0), int(c1)).to_triples())
        trip.append(m.to_triples())
        absum += rowabs
    t = np.concatenate(trip)
    want = whole.to_triples()
    assert len(t) == len(want)
    assert np.array_equal(np.sort(t, order=["row", "col"]), np.sort(want, order=["row", "col"]))
    assert np.allclose(abi.clustered_diag(p, absum, 0, 9000), diag, rtol=1e-13, atol=0)
