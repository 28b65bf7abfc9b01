"""One rank's share of the weak-scaled clustered problem (bench.py --gpus N,
and the threaded multi-rank tests): the SpMM share -- an nnz-balanced 2-D tile of
blocks (default) or a slab of nnz-balanced block rows --
the panel rows it owns (equal rows), their diagonal (the synth.hpp:147-157
rule over sum|row| summed across the ranks' slabs) and the diagonal blocks
its preconditioner tiles need. Every rank generates only its own part.
"""
from __future__ import annotations

import numpy as np

from . import abi


def rank_problem(ctx, comm, params, rank: int, world: int, precond: bool, allreduce_sum, values_prec=abi.BE_F32,
                 partition: str = "2d"):
    """allreduce_sum(np.ndarray) -> np.ndarray summed over ranks (host-side
    glue: torch.distributed in the bench, a thread barrier in the tests).
    partition "2d": this rank's nnz-balanced 2-D tile of blocks (be_dist_tiles2d, the default);
    "slabs": nnz-balanced block-row slabs (be_dist_balance).
    Returns dict(op, tiles, cuts, slabs | rect, lo, hi, nnz_local, tile_entries)."""
    n = params.n
    bounds = abi.uniform_boundaries(n, params.block_extent)
    cuts = abi.dist_rows(bounds, world)
    slabs = rect = None
    if partition == "2d":
        rect = abi.dist_tiles2d(abi.clustered_block_weights(params), bounds, world)[rank]
        slab, rowabs, toff = abi.generate_clustered_tile(params, (int(rect[0]), int(rect[1])),
                                                         (int(rect[2]), int(rect[3])))
    elif partition == "slabs":
        slabs = abi.dist_balance(abi.clustered_weights(params), world)
        slab, rowabs, toff = abi.generate_clustered_part(params, int(slabs[rank]), int(slabs[rank + 1]))
    else:
        raise ValueError(f"partition must be '2d' or 'slabs', not {partition!r}")
    tot = allreduce_sum(rowabs)
    lo, hi = int(cuts[rank]), int(cuts[rank + 1])
    diag = abi.clustered_diag(params, tot[lo:hi], lo, hi)
    del tot, rowabs
    op = abi.DistOperator(ctx, comm, slab, cuts, diag, values_prec=values_prec)
    tiles = None
    if precond:
        b_lo, b_hi = int(np.searchsorted(bounds, lo)), int(np.searchsorted(bounds, hi))
        dblk = abi.generate_clustered_part(params, b_lo, b_hi, diag_blocks_only=True)[0]
        tiles = abi.Tiles(ctx, dblk, diag, toff, row_range=(lo, hi))
        del dblk
    return dict(op=op, tiles=tiles, cuts=cuts, slabs=slabs, rect=rect, lo=lo, hi=hi, nnz_local=slab.nnz,
                tile_entries=tiles.count()[2] if tiles else 0, diag=diag, toff=toff, slab_csb=slab)
