"""Multi-GPU sharding host logic on CPU: edge-balanced owner-row
ranges, CSR slicing, and a world_size-2 gloo run in which each rank
aggregates its dst-row shard (the oracle stands in for the kernel, which
needs a GPU) and an all_gather reassembles exactly the single-process
result."""
import os

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from gspmm_testutil import ROOT
from oracle import oracle as O
from paper_2007_06354_b200.shard import balanced_row_ranges, shard_edges, slice_csr


@pytest.mark.parametrize("parts", [1, 2, 3, 4, 8])
def test_balanced_ranges_cover_and_balance(parts):
    src, dst = O.gen_rmat(5000, 80000, seed=1)
    ip, ix, ei = O.build_csr(5000, src, dst)
    b = balanced_row_ranges(ip, parts)
    assert b[0] == 0 and b[-1] == 5000 and (np.diff(b) >= 0).all() and len(b) == parts + 1
    per = shard_edges(ip, parts)
    assert per.sum() == 80000
    max_row = int(np.diff(ip.astype(np.int64)).max())
    assert per.max() <= 80000 / parts + max_row  # balanced up to one row
    pieces = [slice_csr(ip, ix, ei, int(b[k]), int(b[k + 1])) for k in range(parts)]
    assert np.concatenate([p[1] for p in pieces]).tolist() == ix.tolist()
    assert np.concatenate([p[2] for p in pieces]).tolist() == ei.tolist()
    for k, p in enumerate(pieces):
        assert p[0][0] == 0 and p[0][-1] == len(p[1])


def test_degenerate_ranges():
    ip = np.array([0, 0, 0, 5], np.uint32)  # all edges on the last row
    b = balanced_row_ranges(ip, 4)
    assert b[0] == 0 and b[-1] == 3 and (np.diff(b) >= 0).all()
    ip = np.zeros(1, np.uint32)  # no rows
    assert balanced_row_ranges(ip, 2).tolist() == [0, 0, 0]


def _worker(rank, world, port, q):
    try:
        _work(rank, world, port, q)
    except Exception as ex:  # report instead of hanging the parent
        q.put((rank, repr(ex)))


def _work(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import torch
        n = 3000
        src, dst = O.gen_rmat(n, 40000, seed=7)
        g = O.Graph(n, src, dst)
        x = O.normal_features(n, 32, 1)
        w = O.gcn_weights(n, src, dst)
        ip, ix, ei = g.dst_major
        b = balanced_row_ranges(ip, world)
        lo, hi = int(b[rank]), int(b[rank + 1])
        lip, lix, lei = slice_csr(ip, ix, ei, lo, hi)
        # edge operand in this shard's CSR position order (what the GPU path
        # does with permute_edges + EDGE_BY_POS); local edge ids = positions
        w_pos = np.ascontiguousarray(w[lei])
        lei = np.arange(len(lei), dtype=np.uint32)
        fx, fw = O._feat(x), O._feat(w_pos)
        out = np.empty((hi - lo, 32), np.float32)
        st = O.LIB.or_binary_reduce(O.DST_MAJOR, hi - lo, n, lip.ctypes.data, lix.ctypes.data,
                                    lei.ctypes.data, O.U, O.E, O.MUL, O.SUM, O.V, fx, None, fw,
                                    out.ctypes.data)
        assert st == 0
        # ragged all_gather: pad to the largest shard
        rows = torch.tensor([hi - lo])
        sizes = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(sizes, rows)
        cap = int(max(s.item() for s in sizes))
        buf = torch.zeros((cap, 32))
        buf[: hi - lo] = torch.from_numpy(out)
        parts = [torch.zeros((cap, 32)) for _ in range(world)]
        dist.all_gather(parts, buf)
        full = np.concatenate([p[: int(s.item())].numpy() for p, s in zip(parts, sizes)])
        want = O.binary_reduce(g, (O.U, O.E, O.MUL, O.SUM, O.V), u=x, e=w)
        q.put((rank, bool(O.bit_equal(full, want))))
    finally:
        dist.destroy_process_group()


def test_two_rank_gloo_sharded_aggregation():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + os.getpid() % 1000
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert sorted(res) == [(0, True), (1, True)]
