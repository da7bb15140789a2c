"""Multi-GPU neighbourhood aggregation with sharded source features
(BASELINE config 5: GraphSAGE-mean over 8 GPUs).

Every rank owns a contiguous, edge-balanced range of nodes (shard.py): the
destination rows it aggregates AND the rows of the source-feature matrix it
holds.  The forward needs every source row, so the feature matrix is
all-gathered -- by COLUMN CHUNK, on a communication stream, so that the
aggregation of chunk c (columns are independent: every output element is a
fold over one column) overlaps the all-gather of chunk c + 1.  The gathered
chunk is laid out rank-major with every rank's block padded to the largest
shard (`cap` rows), which is what NCCL's all-gather produces; the local CSR's
neighbour ids are remapped once, at plan time, to those padded positions, so
the kernels gather straight from the collective's output.

Backward (mean): grad_x[u] = sum over out-edges (u -> v) of grad_out[v] / deg(v).
grad_out is dst-sharded exactly like x, so it is all-gathered the same way
and each rank folds its own source rows over its slice of the transposed
CSR, scaling each gathered row by 1/deg(v) inside the kernel (other_scale):
deterministic, no atomics, no reduce-scatter ("preferred").

The host logic here is exercised on CPU by tests/test_dist.py (gloo,
world_size 2) with the aggregation injected; on GPUs the aggregation is the
library's kernels (api.binary_reduce) and the collective is NCCL.
"""
from __future__ import annotations

import numpy as np

from .shard import balanced_row_ranges, slice_csr

__all__ = ["ShardPlan", "ShardedMean", "column_chunks"]


def column_chunks(feat, chunk=256):
    """[(c0, width, padded width)] covering `feat` columns; padded widths are
    multiples of 4 (16-byte rows for the vector kernels)."""
    out = []
    c0 = 0
    while c0 < feat:
        w = min(chunk, feat - c0)
        out.append((c0, w, (w + 3) & ~3))
        c0 += w
    return out


class ShardPlan:
    """One rank's share of a square graph (nodes = rows = columns).

    ``bounds``: node ranges of all ranks (edge-balanced on the dst-major CSR);
    ``fwd``: (indptr, indices, eids) of this rank's dst rows with neighbour
    ids remapped to padded gathered positions; ``bwd``: the same for this
    rank's rows of the transposed (src-major) CSR; ``deg``: in-degree of
    every node (the mean's divisor)."""

    def __init__(self, indptr, indices, eids, num_nodes, rank, world, t_indptr=None,
                 t_indices=None, t_eids=None):
        indptr = np.asarray(indptr)
        self.world, self.rank = int(world), int(rank)
        self.num_nodes = int(num_nodes)
        self.bounds = balanced_row_ranges(indptr, world)
        sizes = np.diff(self.bounds)
        self.cap = int(max(int(sizes.max()) if len(sizes) else 0, 1))
        self.lo, self.hi = int(self.bounds[rank]), int(self.bounds[rank + 1])
        self.rows = self.hi - self.lo
        self.deg = np.diff(indptr.astype(np.int64))
        ip, ix, ei = slice_csr(indptr, indices, eids, self.lo, self.hi)
        self.fwd = (ip, self.padded(ix), ei)
        self.bwd = None
        if t_indptr is not None:
            tip, tix, tei = slice_csr(t_indptr, t_indices, t_eids, self.lo, self.hi)
            self.bwd = (tip, self.padded(tix), tei)

    @property
    def gathered_rows(self):
        return self.world * self.cap

    def padded(self, ids):
        """Global node ids -> positions in the rank-major padded gather."""
        ids = np.asarray(ids, dtype=np.int64)
        owner = np.searchsorted(self.bounds, ids, side="right") - 1
        return (owner * self.cap + (ids - self.bounds[owner])).astype(np.uint32)

    def pad_rows(self, local):
        """This rank's rows padded to `cap` (the all-gather's input block)."""
        out = np.zeros((self.cap,) + local.shape[1:], dtype=local.dtype)
        out[: len(local)] = local
        return out

    def scale_padded(self):
        """1.0f / (float)deg(v) at every padded position (0 for empty rows
        and padding): the mean backward's per-neighbour scale."""
        s = np.zeros(self.gathered_rows, np.float32)
        for k in range(self.world):
            lo, hi = int(self.bounds[k]), int(self.bounds[k + 1])
            d = self.deg[lo:hi].astype(np.float32)
            with np.errstate(divide="ignore"):
                s[k * self.cap: k * self.cap + hi - lo] = np.where(d > 0, np.float32(1.0) / d, 0)
        return s


class ShardedMean:
    """copy_u + mean over a dst-row shard with column-chunked all-gather of
    the source features (and its backward).

    ``allgather(full, local)`` gathers every rank's `local` block into `full`
    (rank-major); ``aggregate(kind, chunk, src, out, scale)`` runs the
    aggregation of one column chunk: kind "fwd" folds `src` rows over the
    forward CSR into `out` (mean), kind "bwd" folds them over the transposed
    CSR scaled by `scale` (sum).  Both default to the GPU implementations
    (NCCL through torch.distributed, the library's kernels)."""

    def __init__(self, plan, feat, *, chunk=256, device=None, allgather=None, aggregate=None):
        import torch
        self.plan, self.feat = plan, int(feat)
        self.chunks = column_chunks(self.feat, chunk)
        self.device = torch.device(device) if device is not None else torch.device("cpu")
        self.cuda = self.device.type == "cuda"
        self.allgather = allgather or _nccl_allgather
        if aggregate is None:
            aggregate = _GpuAggregate(plan, self.device)
        self.aggregate = aggregate
        mk = lambda r, w: torch.zeros((r, w), dtype=torch.float32, device=self.device)  # noqa: E731
        self.local = [mk(plan.cap, wp) for (_, _, wp) in self.chunks]
        self.full = [mk(plan.gathered_rows, wp) for (_, _, wp) in self.chunks]
        self.scale = torch.from_numpy(plan.scale_padded()).to(self.device)
        if self.cuda:
            self.comm = torch.cuda.Stream(device=self.device)
            self.events = [torch.cuda.Event() for _ in self.chunks]

    def load(self, rows):
        """Stage this rank's feature rows (or gradient rows) [rows, feat]
        into the chunked all-gather inputs (a layout copy, not compute)."""
        for (c0, w, _), buf in zip(self.chunks, self.local):
            buf[: rows.shape[0], :w].copy_(rows[:, c0:c0 + w])

    def _run(self, kind, out):
        import torch
        if self.cuda:
            main = torch.cuda.current_stream(self.device)
            self.comm.wait_stream(main)  # the staged inputs are ready
            with torch.cuda.stream(self.comm):
                for k, (full, local) in enumerate(zip(self.full, self.local)):
                    self.allgather(full, local)
                    self.events[k].record(self.comm)
        for k, (c0, w, _) in enumerate(self.chunks):
            if self.cuda:
                torch.cuda.current_stream(self.device).wait_event(self.events[k])
            else:
                self.allgather(self.full[k], self.local[k])
            self.aggregate(kind, k, self.full[k][:, :w], out[:, c0:c0 + w], self.scale)
        return out

    def forward(self, out):
        """out[rows, feat] = mean over in-edges of the gathered source rows."""
        return self._run("fwd", out)

    def backward(self, grad_src):
        """grad_src[rows, feat] from the staged (``load``) output gradient."""
        return self._run("bwd", grad_src)


def _nccl_allgather(full, local):
    import torch.distributed as dist
    dist.all_gather_into_tensor(full, local)


class _GpuAggregate:
    """The library's kernels on the plan's forward / transposed CSR slices."""

    def __init__(self, plan, device):
        from . import api as P
        self.P = P
        idx = device.index if device.index is not None else 0
        ip, ix, ei = plan.fwd
        self.g_fwd = P.Graph(ip, ix, np.arange(len(ix), dtype=np.uint32), num_rows=plan.rows,
                             num_cols=plan.gathered_rows, orientation=P.DST_MAJOR, device=idx)
        self.g_bwd = None
        if plan.bwd is not None:
            tip, tix, _ = plan.bwd
            self.g_bwd = P.Graph(tip, tix, np.arange(len(tix), dtype=np.uint32),
                                 num_rows=plan.rows, num_cols=plan.gathered_rows,
                                 orientation=P.SRC_MAJOR, device=idx)

    def __call__(self, kind, k, src, out, scale):
        P = self.P
        if kind == "fwd":
            P.binary_reduce(self.g_fwd, (P.U, P.NONE, P.COPY, P.MEAN, P.V), u=src, out=out)
        else:
            # out = U on the src-major slice: the gathered operand is the V side
            P.binary_reduce(self.g_bwd, (P.V, P.NONE, P.COPY, P.SUM, P.U), v=src, out=out,
                            other_scale=scale)
