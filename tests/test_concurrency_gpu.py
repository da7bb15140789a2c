"""One graph handle shared by several streams and host threads (the
reference's CsrGraph is safe to share, csr.hpp:35): every call
gets its own per-stream device state, so concurrent calls stay bitwise.
Also the boundary's input checks (out-of-range ids in the device CSR build,
expanded operands, bad output views) and the fault-injection self-test of the
parity harness (a corrupted element must fail the checks, as the reference's
--inject-fault does, tools/main.cpp:201-204)."""
import threading

import numpy as np
import pytest

from gspmm_testutil import HAS_GPU
from oracle import oracle as O

pytestmark = pytest.mark.gpu

if HAS_GPU:
    import torch

    import paper_2007_06354_b200 as P


def power_graph(n=4000, m=120000, seed=3):
    src, dst = O.gen_rmat(n, m, seed=seed)
    src, dst = O.add_self_loops(n, src, dst)
    return O.Graph(n, src, dst)


def test_two_streams_one_handle_bitwise():
    g = power_graph()
    h = P.Graph(*g.dst_major, orientation=P.DST_MAJOR)
    h.set_plan(long_threshold=300)  # long-row units and segments in every call
    assert h.num_long_rows > 0
    xs = [O.normal_features(g.n, d, d) for d in (64, 100, 256)]
    w = O.gcn_weights(g.n, g.src, g.dst)
    want = [O.binary_reduce(g, O.named_config("u_mul_e_add_v"), u=x, e=w) for x in xs]
    xd = [torch.from_numpy(x).cuda() for x in xs]
    wd = torch.from_numpy(w).cuda()
    streams = [torch.cuda.Stream() for _ in range(2)]
    outs = [[torch.empty((g.n, x.shape[1]), device="cuda") for x in xs] for _ in range(2)]
    torch.cuda.synchronize()
    for it in range(30):  # interleaved enqueues on both streams, no host sync
        for k, s in enumerate(streams):
            i = (it + k) % len(xs)
            P.binary_reduce(h, "u_mul_e_add_v", u=xd[i], e=wd, out=outs[k][i], stream=s)
    torch.cuda.synchronize()
    for k in range(2):
        for i in range(len(xs)):
            assert O.bit_equal(outs[k][i].cpu().numpy(), want[i]), (k, i)


def test_host_threads_one_handle_bitwise():
    g = power_graph(seed=5)
    hd = P.Graph(*g.dst_major, orientation=P.DST_MAJOR)
    hs = P.Graph(*g.src_major, orientation=P.SRC_MAJOR)
    for h in (hd, hs):
        h.set_plan(long_threshold=200)
    x = O.normal_features(g.n, 128, 1)
    gy = O.normal_features(g.n, 128, 2)
    w = O.gcn_weights(g.n, g.src, g.dst)
    deg = O.in_degree(g)
    inv = np.zeros(g.n, np.float32)
    inv[deg > 0] = np.float32(1) / deg[deg > 0].astype(np.float32)
    want = {
        "fwd": O.binary_reduce(g, O.named_config("u_mul_e_add_v"), u=x, e=w),
        "max": O.copy_max_argmax(g, x),
        "bwd": O.mean_backward(g, gy),
    }
    xd, gyd, wd = (torch.from_numpy(a).cuda() for a in (x, gy, w))
    invd = torch.from_numpy(inv).cuda()
    errors = []

    def worker(t):
        try:
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                for it in range(15):
                    kind = ("fwd", "max", "bwd")[(t + it) % 3]
                    if kind == "fwd":
                        got = P.binary_reduce(hd, "u_mul_e_add_v", u=xd, e=wd, stream=s)
                        s.synchronize()
                        ok = O.bit_equal(got.cpu().numpy(), want["fwd"])
                    elif kind == "max":
                        v, a, _ = P.binary_reduce(hd, "u_copy_max_v", u=xd, want_arg_other=True,
                                                  stream=s)
                        s.synchronize()
                        ok = O.bit_equal(v.cpu().numpy(), want["max"][0]) and \
                            np.array_equal(a.cpu().numpy(), want["max"][1])
                    else:
                        got = P.binary_reduce(hs, (P.V, P.NONE, P.COPY, P.SUM, P.U), v=gyd,
                                              other_scale=invd, stream=s)
                        s.synchronize()
                        ok = O.bit_equal(got.cpu().numpy(), want["bwd"])
                    if not ok:
                        errors.append((t, it, kind))
        except Exception as e:  # pragma: no cover - surfaced below
            errors.append((t, repr(e)))

    ts = [threading.Thread(target=worker, args=(t,)) for t in range(4)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errors, errors[:5]


def test_host_async_calls_on_two_streams_one_handle():
    # the enqueue-only host entry on one handle from two streams at once
    # (each call stages through its own stream-ordered buffer)
    g = power_graph(seed=9)
    h = P.Graph(*g.dst_major, orientation=P.DST_MAJOR)
    xs = [torch.from_numpy(O.normal_features(g.n, 96, k)).pin_memory().numpy() for k in range(4)]
    outs = [torch.empty((g.n, 96), pin_memory=True).numpy() for _ in range(4)]
    args = [torch.empty((g.n, 96), dtype=torch.int32, pin_memory=True).numpy() for _ in range(4)]
    s = [torch.cuda.Stream(), torch.cuda.Stream()]
    for k in range(4):
        P.binary_reduce_host_async(h, "u_copy_max_v", u=xs[k], out=outs[k], arg_other=args[k],
                                   stream=s[k % 2])
    torch.cuda.synchronize()
    for k in range(4):
        v, a, _ = O.copy_max_argmax(g, xs[k])
        assert O.bit_equal(outs[k], v) and np.array_equal(args[k], a), k


def test_host_entry_other_scale_and_argmax_backward_host():
    g = power_graph(seed=11)
    hs = P.Graph(*g.src_major, orientation=P.SRC_MAJOR)
    gy = O.normal_features(g.n, 40, 4)
    deg = O.in_degree(g)
    inv = np.zeros(g.n, np.float32)
    inv[deg > 0] = np.float32(1) / deg[deg > 0].astype(np.float32)
    out = np.empty((g.n, 40), np.float32)
    s = torch.cuda.Stream()
    P.binary_reduce_host_async(hs, (P.V, P.NONE, P.COPY, P.SUM, P.U), v=gy, out=out,
                               other_scale=inv, stream=s)
    s.synchronize()
    assert O.bit_equal(out, O.mean_backward(g, gy))
    _, au, _ = O.copy_max_argmax(g, O.normal_features(g.n, 40, 5))
    got = P.argmax_backward_host(au, gy, g.n)
    want = O.argmax_backward(au, gy, g.n)
    assert O.max_rel_error(got, want) <= 1e-6


def test_argmax_backward_range_owner_computes():
    # the multi-GPU owner-computes form: every source-row range receives
    # exactly its rows of the whole scatter
    g = power_graph(seed=13)
    x = O.normal_features(g.n, 32, 1)
    gy = O.normal_features(g.n, 32, 2)
    _, au, _ = O.copy_max_argmax(g, x)
    want = O.argmax_backward(au, gy, g.n)
    aud, gyd = torch.from_numpy(au).cuda(), torch.from_numpy(gy).cuda()
    bounds = [0, 1000, 1001, 2500, g.n]
    parts = [P.argmax_backward(aud, gyd, hi - lo, src_lo=lo).cpu().numpy()
             for lo, hi in zip(bounds[:-1], bounds[1:])]
    got = np.concatenate(parts)
    assert O.max_rel_error(got, want) <= 1e-6


def test_device_csr_build_rejects_out_of_range_ids():
    n = 100
    src = torch.tensor([1, 2, 3, 150, 4], dtype=torch.int32, device="cuda")
    dst = torch.tensor([0, 5, 7, 8, 120], dtype=torch.int32, device="cuda")
    with pytest.raises(P.StructureError, match="edge 3 references node id 150 >= num_nodes 100"):
        P.build_csr_device(n, src, dst, P.DST_MAJOR)


def test_expanded_operand_and_bad_out_views_rejected():
    g = power_graph(n=300, m=3000)
    h = P.Graph(*g.dst_major, orientation=P.DST_MAJOR)
    bias = torch.randn(1, 16, device="cuda")
    with pytest.raises(P.ShapeError):
        P.binary_reduce(h, "u_copy_add_v", u=bias.expand(g.n, 16))
    x = torch.randn(g.n, 16, device="cuda")
    with pytest.raises(P.ShapeError):
        P.binary_reduce(h, "u_copy_add_v", u=x, out=torch.empty(g.n, 16, dtype=torch.float64,
                                                                device="cuda"))
    with pytest.raises(P.ShapeError):  # transposed (column-major) output
        P.binary_reduce(h, "u_copy_add_v", u=x, out=torch.empty(16, g.n, device="cuda").t())
    with pytest.raises(P.ShapeError):
        P.binary_reduce(h, "u_copy_add_v", u=x, out=torch.empty(g.n, 15, device="cuda"))


def test_fault_injection_is_detected():
    # the parity harness must fail on one corrupted element (the reference's
    # --inject-fault hook, tools/main.cpp:201-204): sum (tolerance check),
    # max (bitwise) and argmax (integer) outputs
    g = power_graph(seed=17)
    x = O.normal_features(g.n, 64, 1)
    xd = torch.from_numpy(x).cuda()
    h = P.Graph(*g.dst_major, orientation=P.DST_MAJOR)
    s = P.binary_reduce(h, "u_copy_add_v", u=xd).cpu().numpy()
    want = O.binary_reduce(g, O.named_config("u_copy_add_v"), u=x)
    assert O.bit_equal(s, want)
    bad = s.copy()
    bad[123, 7] += np.float32(1e-3) * max(1.0, abs(float(bad[123, 7])))
    assert not O.bit_equal(bad, want)
    assert O.max_rel_error(bad, want) > 1e-5
    v, a, _ = P.binary_reduce(h, "u_copy_max_v", u=xd, want_arg_other=True)
    v, a = v.cpu().numpy(), a.cpu().numpy()
    wv, wa, _ = O.copy_max_argmax(g, x)
    assert O.bit_equal(v, wv) and np.array_equal(a, wa)
    v[5, 5] = np.nextafter(v[5, 5], np.float32(np.inf))
    a[7, 3] += 1
    assert not O.bit_equal(v, wv)
    assert not np.array_equal(a, wa)
