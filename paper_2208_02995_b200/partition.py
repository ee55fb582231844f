"""Host-side row partitioning for the multi-GPU path (one process per GPU).

``partition_rows`` picks the contiguous global row range each rank owns
(passed to emin_setup as opts.row_begin/row_end).  ``halo_plan`` states, in
numpy, what dist.cu builds on the device from those ranges: the halo rows of
a rank (global F ids of F rows it does not own but its A_FF rows reference,
sorted, hence grouped by owner) and the rows each owner sends.  The gloo
tests check both against the single-process result (tests/test_partition_gloo.py).
"""
from __future__ import annotations

import numpy as np


def partition_rows(P_rowptr, is_coarse, nranks, plane=None):
    """Contiguous ranges [b_r, e_r) covering all rows, balancing nnz(W) (the
    F-row pattern entries, the unit of work) and cut at multiples of
    ``plane`` rows (one z-plane of a lexicographic grid) when given."""
    n = len(is_coarse)
    if nranks <= 1:
        return [(0, n)]
    w = np.where(np.asarray(is_coarse) == 0, np.diff(np.asarray(P_rowptr)), 0).astype(np.float64)
    cum = np.cumsum(w)
    tot = cum[-1]
    cuts = [0]
    for k in range(1, nranks):
        c = int(np.searchsorted(cum, tot * k / nranks))
        if plane:
            c = int(round(c / plane)) * plane
        c = min(max(c, cuts[-1] + 1), n - (nranks - k))
        cuts.append(c)
    cuts.append(n)
    return [(cuts[r], cuts[r + 1]) for r in range(nranks)]


def f_ids(is_coarse):
    """Global F id of every row (-1 for C rows), ascending with the row."""
    isc = np.asarray(is_coarse) != 0
    fid = np.cumsum(~isc) - 1
    fid[isc] = -1
    return fid


def halo_plan(A_rowptr, A_col, is_coarse, ranges, rank):
    """Halo rows of ``rank`` (sorted global F ids) and their owners."""
    isc = np.asarray(is_coarse) != 0
    fid = f_ids(is_coarse)
    b, e = ranges[rank]
    rows = np.arange(b, e)
    rows = rows[~isc[rows]]
    fb = fid[rows[0]] if rows.size else 0
    fe = fid[rows[-1]] + 1 if rows.size else 0
    lo, hi = A_rowptr[b], A_rowptr[e]
    owner_row = np.repeat(np.arange(b, e), np.diff(A_rowptr[b:e + 1]))
    cols = np.asarray(A_col[lo:hi])
    keep = (~isc[owner_row]) & (~isc[cols])
    g = fid[cols[keep]]
    halo = np.unique(g[(g < fb) | (g >= fe)])
    # owner of each halo row: the rank whose F range contains it
    franges = []
    for (bb, ee) in ranges:
        ff = fid[bb:ee]
        ff = ff[ff >= 0]
        franges.append((int(ff[0]), int(ff[-1]) + 1) if ff.size else (0, 0))
    owners = np.array([next(p for p, (x, y) in enumerate(franges) if x <= h < y) for h in halo], dtype=np.int64)
    return halo, owners, (int(fb), int(fe)), franges


def rank_slice(prob, rb, re_):
    """The inputs a rank passes to emin_setup for its rows [rb, re_): its
    rows of A, P and B only (row pointers rebased to 0, global column ids),
    plus the global is_coarse and B_c (include/emin.h).  Host numpy arrays."""
    a0, a1 = int(prob.A_rowptr[rb]), int(prob.A_rowptr[re_])
    p0, p1 = int(prob.P_rowptr[rb]), int(prob.P_rowptr[re_])
    return dict(
        A_rowptr=np.ascontiguousarray(prob.A_rowptr[rb:re_ + 1] - a0),
        A_col=np.ascontiguousarray(prob.A_col[a0:a1]),
        A_val=np.ascontiguousarray(prob.A_val[a0:a1]),
        is_coarse=prob.is_coarse,
        P_rowptr=np.ascontiguousarray(prob.P_rowptr[rb:re_ + 1] - p0),
        P_col=np.ascontiguousarray(prob.P_col[p0:p1]),
        P_val=None if prob.P_val is None else np.ascontiguousarray(prob.P_val[p0:p1]),
        B=np.ascontiguousarray(prob.B[rb:re_]),
        Bc=prob.Bc,
    )


def plane_rows(prob):
    """Rows of one z-plane of the problem's lexicographic grid (the cut unit
    of partition_rows; whole nodes for the 3-dof elasticity rows)."""
    dims = prob.meta["dims"]
    per = 3 if prob.block_size == 3 else 1
    if len(dims) > 2 and dims[2] > 1:
        return int(dims[0] * dims[1] * per)
    return int(dims[0] * per)          # 2D: one grid line
