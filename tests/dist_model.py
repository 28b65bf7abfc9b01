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


def dist_tiles2d(w, bounds, world):
    """Recursive coordinate bisection of the lower block grid (be_dist_tiles2d), restated:
    shrink to the bounding box of the non-empty blocks; p > 1 ranks: cut the longer side
    (matrix rows, rows on ties, a one-block side never) at the line k in [1, L-1] minimising
    |W(first k lines) p - W(rect) (p // 2)| (smaller k on ties), first part p // 2 ranks."""
    w = np.tril(np.asarray(w, dtype=np.int64))
    b = [int(x) for x in bounds]
    out = np.zeros((world, 4), np.int64)

    def rec(r0, r1, c0, c1, p, rank0):
        sub = w[r0:r1, c0:c1]
        nzr, nzc = np.nonzero(sub.sum(axis=1))[0], np.nonzero(sub.sum(axis=0))[0]
        nz = np.nonzero(sub)
        if len(nz[0]) == 0:
            return
        r0, r1 = r0 + int(nz[0].min()), r0 + int(nz[0].max()) + 1
        c0, c1 = c0 + int(nz[1].min()), c0 + int(nz[1].max()) + 1
        del nzr, nzc
        if p == 1 or (r1 - r0 < 2 and c1 - c0 < 2):
            out[rank0] = (r0, r1, c0, c1)
            return
        by_rows = c1 - c0 < 2 or (r1 - r0 >= 2 and b[r1] - b[r0] >= b[c1] - b[c0])
        sub = w[r0:r1, c0:c1]
        line = [int(x) for x in (sub.sum(axis=1) if by_rows else sub.sum(axis=0))]
        tot, pl = sum(line), p // 2
        pre, best, bestd = 0, 1, None
        for k in range(1, len(line)):
            pre += line[k - 1]
            d = abs(pre * p - tot * pl)
            if bestd is None or d < bestd:
                best, bestd = k, d
        if by_rows:
            rec(r0, r0 + best, c0, c1, pl, rank0)
            rec(r0 + best, r1, c0, c1, p - pl, rank0 + pl)
        else:
            rec(r0, r1, c0, c0 + best, pl, rank0)
            rec(r0, r1, c0 + best, c1, p - pl, rank0 + pl)

    rec(0, w.shape[0], 0, w.shape[0], world, 0)
    return out


def touched_segments(w, bounds, cuts, rect):
    """Panel segments (cuts) whose rows a rectangle's non-empty blocks read or write."""
    r0, r1, c0, c1 = (int(x) for x in rect)
    q = set()
    for bi in range(r0, r1):
        for bj in range(c0, min(c1, bi + 1)):
            if w[bi][bj] > 0:
                q.add(int(np.searchsorted(cuts, bounds[bi], side="right") - 1))
                q.add(int(np.searchsorted(cuts, bounds[bj], side="right") - 1))
    return q
