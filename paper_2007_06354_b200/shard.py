"""Multi-GPU row sharding (host logic).

Owner rows are partitioned into contiguous ranges balanced by edge count --
the GPU analogue of the reference's edge-balanced thread ranges
(block_plan.cpp:83-99).  Each rank uploads the CSR slice of its rows (global
neighbour ids and edge ids, indptr rebased), so the forward needs no
reduction: every output row has exactly one owner.  Source features are
replicated (configs 1-4) or all-gathered (config 5) by the caller.
"""
from __future__ import annotations

import numpy as np


def balanced_row_ranges(indptr, parts):
    """Split rows [0, R) into `parts` contiguous ranges with ~equal edges.

    Boundary k is the first row whose prefix edge count reaches k*E/parts;
    returns an int64 array of parts+1 boundaries (0 ... R)."""
    indptr = np.asarray(indptr, dtype=np.int64)
    rows = len(indptr) - 1
    m = int(indptr[-1])
    if parts < 1:
        raise ValueError("parts must be >= 1")
    targets = (np.arange(1, parts, dtype=np.float64) * m / parts)
    cut = np.searchsorted(indptr, targets, side="left").astype(np.int64)
    cut = np.clip(cut, 0, rows)
    bounds = np.concatenate([[0], cut, [rows]]).astype(np.int64)
    return np.maximum.accumulate(bounds)


def slice_csr(indptr, indices, eids, lo, hi):
    """CSR of rows [lo, hi): indptr rebased to 0, global column/edge ids."""
    indptr = np.asarray(indptr)
    b, e = int(indptr[lo]), int(indptr[hi])
    local = (indptr[lo:hi + 1].astype(np.int64) - b).astype(np.uint32)
    return local, np.ascontiguousarray(indices[b:e]), np.ascontiguousarray(eids[b:e])


def shard_edges(indptr, parts):
    """Edges owned by each part under balanced_row_ranges (for reporting)."""
    bounds = balanced_row_ranges(indptr, parts)
    ip = np.asarray(indptr, dtype=np.int64)
    return ip[bounds[1:]] - ip[bounds[:-1]]
