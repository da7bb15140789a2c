"""Config-5 multi-GPU path on CPU: dst-row / source-feature
shards, column-chunked all-gather of the source features (gloo stands in for
NCCL) and of the output gradient, remapped neighbour ids, and the mean
forward / backward on each rank's CSR slices.  The aggregation of a chunk is
injected (the oracle's restated RowParallelSpmm; the kernels need a GPU);
the rank results, concatenated, must equal the single-process oracle bit for
bit."""
import os

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from gspmm_testutil import ROOT  # noqa: F401  (sys.path)
from oracle import oracle as O
from paper_2007_06354_b200.dist import ShardPlan, ShardedMean, column_chunks


def test_column_chunks():
    assert column_chunks(602, 256) == [(0, 256, 256), (256, 256, 256), (512, 90, 92)]
    assert column_chunks(100, 256) == [(0, 100, 100)]
    assert column_chunks(5, 4) == [(0, 4, 4), (4, 1, 4)]


@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_plan_remap_is_a_bijection_onto_gathered_rows(world):
    n = 2000
    src, dst = O.gen_powerlaw(n, 3, 300, seed=2)
    g = O.Graph(n, src, dst)
    ip, ix, ei = g.dst_major
    seen = []
    for r in range(world):
        p = ShardPlan(ip, ix, ei, n, r, world)
        pos = p.padded(np.arange(n))
        # every node lands in its owner's block, in order, and nowhere else
        assert len(set(pos.tolist())) == n and pos.max() < p.gathered_rows
        owner = pos // p.cap
        assert (np.diff(pos[owner == r].astype(np.int64)) == 1).all()
        seen.append((p.lo, p.hi))
        assert p.rows == p.hi - p.lo and p.fwd[0][-1] == len(p.fwd[1])
    assert seen[0][0] == 0 and seen[-1][1] == n
    assert all(seen[k][1] == seen[k + 1][0] for k in range(world - 1))


def _oracle_aggregate(plan):
    """Chunk aggregation on CPU by the oracle (test stand-in for the kernels)."""
    def agg(kind, k, src, out, scale):
        src = np.ascontiguousarray(src.numpy())
        if kind == "fwd":
            ip, ix, ei = plan.fwd
            res = np.empty((plan.rows, src.shape[1]), np.float32)
            O._check(O.LIB.or_mean(O.DST_MAJOR, plan.rows, plan.gathered_rows, ip.ctypes.data,
                                   ix.ctypes.data, ei.ctypes.data, O.U, O._feat(src),
                                   res.ctypes.data), "mean")
        else:
            ip, ix, _ = plan.bwd
            pos = np.arange(len(ix), dtype=np.uint32)
            e = np.ascontiguousarray(scale.numpy()[ix.astype(np.int64)]).reshape(-1, 1)
            res = np.empty((plan.rows, src.shape[1]), np.float32)
            O._check(O.LIB.or_binary_reduce(O.SRC_MAJOR, plan.rows, plan.gathered_rows,
                                            ip.ctypes.data, ix.ctypes.data, pos.ctypes.data,
                                            O.V, O.E, O.MUL, O.SUM, O.U, None, O._feat(src),
                                            O._feat(e), res.ctypes.data), "bwd")
        import torch
        out.copy_(torch.from_numpy(res))
    return agg


def _gloo_allgather(world):
    def ag(full, local):
        dist.all_gather(list(full.chunk(world)), local.contiguous())
    return ag


def _worker(rank, world, port, q):
    try:
        _work(rank, world, port, q)
    except Exception as ex:  # report instead of hanging the parent
        import traceback
        q.put((rank, repr(ex) + traceback.format_exc()))


def _work(rank, world, port, q):
    import torch
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n, feat = 3000, 70
        src, dst = O.gen_powerlaw(n, 4, 400, seed=5)
        g = O.Graph(n, src, dst)
        ip, ix, ei = g.dst_major
        tip, tix, tei = g.src_major
        plan = ShardPlan(ip, ix, ei, n, rank, world, tip, tix, tei)
        x = O.normal_features(n, feat, 1)
        gy = O.normal_features(n, feat, 3)
        sm = ShardedMean(plan, feat, chunk=32, allgather=_gloo_allgather(world),
                         aggregate=_oracle_aggregate(plan))
        sm.load(torch.from_numpy(x[plan.lo:plan.hi]))
        out = torch.zeros((plan.rows, feat + 2))[:, :feat]  # padded leading dimension
        sm.forward(out)
        sm.load(torch.from_numpy(gy[plan.lo:plan.hi]))
        gx = torch.zeros((plan.rows, feat))
        sm.backward(gx)
        # reassemble every rank's rows (ragged: pad to cap)
        parts = [torch.zeros((plan.cap, 2 * feat)) for _ in range(world)]
        mine = torch.zeros((plan.cap, 2 * feat))
        mine[: plan.rows, :feat] = out
        mine[: plan.rows, feat:] = gx
        dist.all_gather(parts, mine)
        full = np.concatenate([parts[k][: int(plan.bounds[k + 1] - plan.bounds[k])].numpy()
                               for k in range(world)])
        want_f = O.mean(g, x)
        want_b = O.mean_backward(g, gy)
        q.put((rank, bool(O.bit_equal(full[:, :feat], want_f)) and
               bool(O.bit_equal(full[:, feat:], want_b))))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_gloo_sharded_mean_fwd_bwd_matches_single_process(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29700 + os.getpid() % 1000
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=180) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert sorted(res) == [(r, True) for r in range(world)], res
