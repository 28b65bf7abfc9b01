"""Test infrastructure: a plain-Python restatement of the multi-GPU partition
and data flow of the distributed operator (paper_2109_00485_b200/csrc/spmm.cu,
op_create_dist / op_apply_dist), used by the CPU tests to check the C++ rules
bit-exactly and to replay the exchange with torch.distributed (gloo).

The reference's own multi-rank semantics (dist.hpp) are a fixed triangular
layout over nd(nd+1)/2 ranks; the B200 build partitions for any rank count:
  * panel rows: equal rows on CSB block boundaries (dist_rows);
  * SpMM slabs: contiguous CSB block rows of near-equal stored nonzeros
    (dist_balance);
  * exchange: X segments padded to lmax rows are allgathered, the partial Y
    panels (world * lmax rows) reduce-scattered back to the row owners.
"""
from __future__ import annotations

import numpy as np


def dist_rows(bounds, world):
    """cut p = the block boundary closest to n p / world (lower on ties),
    then forced strictly increasing with room for the ranks after p."""
    b = [int(x) for x in bounds]
    nblk = len(b) - 1
    if world < 1 or nblk < world:
        raise ValueError("bad world")
    n = b[-1]
    k = [0] * (world + 1)
    k[world] = nblk
    for p in range(1, world):
        best, bestd = 0, None
        for j in range(nblk + 1):
            dd = abs(b[j] * world - n * p)
            if bestd is None or dd < bestd:
                best, bestd = j, dd
        k[p] = best
    for p in range(1, world):
        k[p] = min(max(k[p], k[p - 1] + 1), nblk - (world - p))
    return np.array([b[x] for x in k], np.int64)


def dist_balance(weights, world):
    """cut p = first item index whose prefix weight reaches total p / world."""
    w = [int(x) for x in weights]
    total = sum(w)
    cuts = [0] + [len(w)] * world
    pre, i = 0, 0
    for p in range(1, world):
        while i < len(w) and pre * world < total * p:
            pre += w[i]
            i += 1
        cuts[p] = i
    return np.array(cuts, np.int64)


def padded(rows, cuts):
    """global row -> padded exchange index q * lmax + (row - cuts[q])."""
    cuts = np.asarray(cuts)
    lmax = int(np.max(np.diff(cuts)))
    q = np.searchsorted(cuts, rows, side="right") - 1
    return q * lmax + (rows - cuts[q]), lmax


def slab_partial_spmm(rows, cols, vals, x_full_padded, cuts, nb):
    """One rank's contribution to the padded partial Y: both applications of
    each stored entry of its slab (A_ij X_j -> Y_i, A_ij X_i -> Y_j)."""
    pr, lmax = padded(rows, cuts)
    pc, _ = padded(cols, cuts)
    y = np.zeros((len(cuts) - 1) * lmax * nb).reshape(-1, nb)
    x = x_full_padded.reshape(-1, nb)
    np.add.at(y, pr, vals[:, None] * x[pc])
    np.add.at(y, pc, vals[:, None] * x[pr])
    return y
