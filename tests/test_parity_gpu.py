"""GPU parity: the sm_100a kernels (through the C-ABI) against the pinned
oracle on identical seeded inputs.

The bar is BIT-EXACTNESS for every op, sums included: the kernels fold each
output element sequentially in canonical edge order with separately rounded
products and sums, exactly like the reference's RowParallelSpmm
(kernels.cpp:162-195), which the oracle restates and the golden fixtures pin.
The reference's own looser criterion (max_rel_error <= 1e-5 against the f64
oracle_aggregate, compare.hpp:30-45) is checked as well.
"""
import numpy as np
import pytest


from gspmm_testutil import HAS_GPU, ROOT
from oracle import oracle as O

pytestmark = pytest.mark.gpu

if HAS_GPU:
    import torch

    import paper_2007_06354_b200 as P

SUM_TOL = 1e-5  # reference acceptance tolerance for sum-like reduces


def dev_graph(g, orientation):
    """Device handle for one orientation of an oracle Graph (cached); a plan
    set on the oracle Graph (g.plan = dict(...)) is applied to new handles."""
    cache = g.__dict__.setdefault("_dev", {})
    if orientation not in cache:
        ip, ix, ei = g.csr(orientation)
        h = P.Graph(ip, ix, ei, g.n, g.n, orientation, validate=True)
        if getattr(g, "plan", None):
            h.set_plan(**g.plan)
        cache[orientation] = h
    return cache[orientation]


def cuda(a):
    if a is None:
        return None
    a = np.ascontiguousarray(a, np.float32)
    if a.ndim == 1:
        a = a.reshape(-1, 1)
    return torch.from_numpy(a).cuda()


def gpu_reduce(g, cfg, u=None, v=None, e=None, **kw):
    orientation = O.SRC_MAJOR if cfg[4] == O.U else O.DST_MAJOR
    h = dev_graph(g, orientation)
    res = P.binary_reduce(h, cfg, cuda(u), cuda(v), cuda(e), **kw)
    torch.cuda.synchronize()
    if isinstance(res, tuple):
        return tuple(None if r is None else r.cpu().numpy() for r in res)
    return res.cpu().numpy()


def g_of(n, edges):
    return O.Graph(n, np.array([e[0] for e in edges], np.uint32),
                   np.array([e[1] for e in edges], np.uint32))


# ------------------------------- goldens of proj/tests/test_kernels.cpp
def test_goldens_from_reference_tests():
    g = g_of(3, [(0, 2), (1, 2)])
    assert gpu_reduce(g, O.named_config("u_copy_add_v"), u=[[1, 2], [3, 4], [0, 0]]).tolist() == \
        [[0, 0], [0, 0], [4, 6]]                                           # :49-66
    g = g_of(2, [(0, 1)])
    assert gpu_reduce(g, O.named_config("u_copy_add_v"), u=[[5, -3], [9, 9]]).tolist() == \
        [[0, 0], [5, -3]]                                                  # :68-78
    g3 = g_of(3, [(0, 1), (2, 1)])
    assert gpu_reduce(g3, O.named_config("u_copy_max_v"), u=[[5], [-7], [2]])[:, 0].tolist() == \
        [0, 5, 0]                                                          # :80-90
    assert gpu_reduce(g, O.named_config("u_mul_e_add_v"), u=[[2, 3], [0, 0]],
                      e=[[10, 10]])[1].tolist() == [20, 30]                # :92-103
    out = gpu_reduce(g, O.named_config("u_dot_v_add_e"), u=[[1, 2], [0, 0]], v=[[0, 0], [3, 4]])
    assert out.shape == (1, 1) and out[0, 0] == 11                         # :105-116
    assert gpu_reduce(g, O.named_config("u_add_v_copy_e"), u=[[1], [0]],
                      v=[[0], [5]])[0, 0] == 6                             # :118-127
    gd = g_of(2, [(0, 1), (0, 1)])
    assert gpu_reduce(gd, O.named_config("e_copy_max_v"), e=[[3], [7]])[1, 0] == 7  # :129-137
    gc = g_of(3, [(2, 1), (0, 1)])                                         # test_oracle.cpp:64-73
    assert gpu_reduce(gc, O.named_config("u_copy_copy_v"), u=[[10], [0], [99]])[1, 0] == 99


def test_empty_graph_all_zero():  # test_kernels.cpp:190-200
    g = O.Graph(4, np.array([], np.uint32), np.array([], np.uint32))
    for name in ("u_copy_add_v", "u_copy_max_v"):
        assert (gpu_reduce(g, O.named_config(name), u=np.ones((4, 3))) == 0).all()


def test_copy_reduce_infers_entity():  # test_kernels.cpp:176-188
    g = g_of(3, [(0, 2), (1, 2)])
    h = dev_graph(g, O.DST_MAJOR)
    out = P.copy_reduce(h, cuda([[1], [10]]), P.SUM)
    assert out.cpu().numpy()[2, 0] == 11
    with pytest.raises(P.ShapeError):
        P.copy_reduce(h, cuda(np.zeros((5, 1))), P.SUM)


def test_validation_errors():  # test_kernels.cpp:139-174
    g = g_of(2, [(0, 1)])
    cfg = O.named_config("u_copy_add_v")
    with pytest.raises(P.ShapeError):  # wrong orientation for the output
        P.binary_reduce(dev_graph(g, O.SRC_MAJOR), cfg, cuda(np.zeros((2, 4))))
    h = dev_graph(g, O.DST_MAJOR)
    with pytest.raises(P.ShapeError):  # missing operand
        P.binary_reduce(h, cfg)
    with pytest.raises(P.ShapeError):  # row mismatch
        P.binary_reduce(h, cfg, cuda(np.zeros((3, 4))))
    with pytest.raises(P.ShapeError):  # incompatible widths
        P.binary_reduce(h, O.named_config("u_add_v_add_v"), cuda(np.zeros((2, 4))),
                        cuda(np.zeros((2, 3))))
    with pytest.raises(P.ConfigError):
        P.binary_reduce(h, (O.U, O.U, O.MUL, O.SUM, O.V), cuda(np.zeros((2, 4))))


def test_degree_identity():  # test_kernels.cpp:339-352
    n, src, dst = O.random_small_graph(190)
    g = O.Graph(n, src, dst)
    out = gpu_reduce(g, O.named_config("u_copy_add_v"), u=np.ones((n, 1)))
    assert (out[:, 0] == np.bincount(dst, minlength=n)).all()


# ------------------------------------------- reference fixtures, bitwise
@pytest.mark.parametrize("seed", (101, 104, 107))
def test_reference_fixtures_bit_exact(golden, seed):
    p = f"s{seed}_"
    n = int(golden[p + "n"][0])
    g = O.Graph(n, golden[p + "src"], golden[p + "dst"])
    fu, fv, fe = golden[p + "fu"], golden[p + "fv"], golden[p + "fe"]
    for cname in O.APPLICATION_CONFIGS:
        cfg = O.named_config(cname)
        got = gpu_reduce(g, cfg, fu, fv, fe)
        assert O.bit_equal(got, golden[p + "spmm_" + cname]), cname
        if cfg[4] != O.E:
            want = golden[p + "oracle_" + cname]
            if O.is_exact_reduce(cfg[3]):
                assert O.bit_equal(got, want), cname
            else:
                assert O.max_rel_error(got, want) <= SUM_TOL, cname


def test_composed_fixtures_bit_exact(golden):
    n = int(golden["c_n"][0])
    g = O.Graph(n, golden["c_src"], golden["c_dst"])
    x, w, gy, a = golden["c_x"], golden["c_w"], golden["c_gy"], golden["c_att"]
    assert O.bit_equal(gpu_reduce(g, (O.U, O.E, O.MUL, O.SUM, O.V), u=x, e=w), golden["c_gcn_fwd"])
    assert O.bit_equal(gpu_reduce(g, (O.V, O.E, O.MUL, O.SUM, O.U), v=gy, e=w), golden["c_gcn_bwd"])
    assert O.bit_equal(gpu_reduce(g, (O.U, O.V, O.DOT, O.LAST, O.E), u=x, v=gy), golden["c_grad_w"])
    assert O.bit_equal(gpu_reduce(g, (O.U, O.NONE, O.COPY, P.MEAN, O.V), u=x), golden["c_mean"])
    assert O.bit_equal(gpu_reduce(g, (O.U, O.NONE, O.COPY, O.MAX, O.V), u=x), golden["c_max"])
    assert O.bit_equal(gpu_reduce(g, (O.U, O.E, O.MUL, O.SUM, O.V), u=x, e=a, heads=4),
                       golden["c_mh_fwd"])


# ------------------------------------- properties over random graphs
EXTRA = ["u_copy_max_v", "u_copy_min_v", "u_copy_mul_v", "u_copy_copy_v", "u_sub_v_add_v",
         "u_div_e_max_v", "e_mul_u_min_v", "v_add_e_add_v", "u_mul_v_mul_v", "e_copy_copy_v",
         "u_sub_e_copy_e", "u_dot_e_add_v", "v_dot_u_max_v"]


@pytest.mark.parametrize("seed", range(101, 141))
def test_all_configs_bit_exact_vs_oracle(seed):  # test_kernels.cpp:202-226
    n, src, dst = O.random_small_graph(seed)
    g = O.Graph(n, src, dst)
    dim = 1 + O.splitmix64_at(seed, 1) % 17
    fu = O.random_features(n, dim, seed)
    fv = O.random_features(n, dim, seed + 1)
    fe = O.random_features(g.m, dim, seed + 2)
    for cname in O.APPLICATION_CONFIGS + EXTRA:
        cfg = O.named_config(cname)
        want = O.binary_reduce(g, cfg, fu, fv, fe)
        got = gpu_reduce(g, cfg, fu, fv, fe)
        assert O.bit_equal(got, want), f"{cname} seed {seed}"


@pytest.mark.parametrize("seed", range(130, 135))
def test_scalar_edge_broadcast(seed):  # test_kernels.cpp:228-241
    n, src, dst = O.random_small_graph(seed)
    g = O.Graph(n, src, dst)
    fu = O.random_features(n, 9, seed)
    fe = O.random_features(g.m, 1, seed + 2)
    cfg = O.named_config("u_mul_e_add_v")
    got = gpu_reduce(g, cfg, u=fu, e=fe)
    assert O.bit_equal(got, O.binary_reduce(g, cfg, u=fu, e=fe))
    assert O.max_rel_error(got, O.oracle_aggregate(g, cfg, u=fu, e=fe)) <= SUM_TOL


@pytest.mark.parametrize("seed", range(150, 154))
def test_source_destined(seed):  # test_kernels.cpp:261-276
    n, src, dst = O.random_small_graph(seed)
    g = O.Graph(n, src, dst)
    fu = O.random_features(n, 4, seed)
    fv = O.random_features(n, 4, seed + 1)
    cfg = (O.U, O.V, O.MUL, O.SUM, O.U)
    got = gpu_reduce(g, cfg, u=fu, v=fv)
    assert O.bit_equal(got, O.binary_reduce(g, cfg, u=fu, v=fv))
    assert O.max_rel_error(got, O.oracle_aggregate(g, cfg, u=fu, v=fv)) <= SUM_TOL


def test_linearity():  # test_kernels.cpp:323-337
    n, src, dst = O.random_small_graph(180)
    g = O.Graph(n, src, dst)
    fu = O.random_features(n, 6, 180)
    cfg = O.named_config("u_copy_add_v")
    base = gpu_reduce(g, cfg, u=fu)
    scaled = gpu_reduce(g, cfg, u=fu * np.float32(3))
    assert O.max_rel_error(scaled, base * np.float32(3)) <= SUM_TOL


def test_deterministic_repeats():  # max bit-identical across runs (cf. :308-321)
    n, src, dst = O.random_small_graph(170)
    g = O.Graph(n, src, dst)
    fu = O.random_features(n, 8, 170)
    for name in ("u_copy_max_v", "u_copy_add_v"):
        a = gpu_reduce(g, O.named_config(name), u=fu)
        for _ in range(3):
            assert O.bit_equal(a, gpu_reduce(g, O.named_config(name), u=fu))


# ------------------------------------------------ layouts and widths
@pytest.mark.parametrize("dim", [1, 2, 3, 4, 5, 7, 8, 31, 33, 64, 100, 127, 128, 129, 256, 300,
                                 512, 602])
def test_widths_bit_exact(dim):
    src, dst = O.gen_rmat(3000, 40000, seed=dim)
    g = O.Graph(3000, src, dst)
    x = O.normal_features(3000, dim, dim)
    w = O.gcn_weights(3000, src, dst)
    fe = O.random_features(g.m, dim, 5)
    for cfg, kw in (((O.U, O.E, O.MUL, O.SUM, O.V), dict(u=x, e=w)),
                    ((O.U, O.E, O.SUB, O.MAX, O.V), dict(u=x, e=fe)),
                    ((O.U, O.NONE, O.COPY, O.SUM, O.V), dict(u=x)),
                    ((O.V, O.E, O.MUL, O.SUM, O.U), dict(v=x, e=w)),
                    ((O.U, O.V, O.DOT, O.LAST, O.E), dict(u=x, v=x))):
        assert O.bit_equal(gpu_reduce(g, cfg, **kw), O.binary_reduce(g, cfg, **kw)), (dim, cfg)


def test_padded_leading_dimension():
    # F=602 rows are not 16-byte aligned; a padded device ld=604 takes the
    # float4 path.  Results must not depend on the layout.
    src, dst = O.gen_rmat(2000, 30000, seed=3)
    g = O.Graph(2000, src, dst)
    x = O.normal_features(2000, 602, 1)
    want = O.mean(g, x)
    h = dev_graph(g, O.DST_MAJOR)
    xp = torch.zeros((2000, 604), dtype=torch.float32, device="cuda")
    xp[:, :602] = cuda(x)
    outp = torch.full((2000, 604), 7.0, device="cuda")
    P.binary_reduce(h, (O.U, O.NONE, O.COPY, P.MEAN, O.V), xp[:, :602], out=outp[:, :602])
    torch.cuda.synchronize()
    assert O.bit_equal(outp[:, :602].cpu().numpy(), want)
    assert (outp[:, 602:] == 7.0).all()  # padding untouched
    out = P.binary_reduce(h, (O.U, O.NONE, O.COPY, P.MEAN, O.V), cuda(x))
    assert O.bit_equal(out.cpu().numpy(), want)


def test_edge_operand_in_csr_order():
    src, dst = O.gen_rmat(2000, 30000, seed=4)
    g = O.Graph(2000, src, dst)
    x = O.normal_features(2000, 64, 1)
    w = O.gcn_weights(2000, src, dst)
    want = O.binary_reduce(g, (O.U, O.E, O.MUL, O.SUM, O.V), u=x, e=w)
    for orientation, cfg, kw in ((O.DST_MAJOR, (O.U, O.E, O.MUL, O.SUM, O.V), "u"),
                                 (O.SRC_MAJOR, (O.V, O.E, O.MUL, O.SUM, O.U), "v")):
        h = dev_graph(g, orientation)
        wp = h.permute_edges(cuda(w))
        args = {kw: cuda(x), "e": wp}
        got = P.binary_reduce(h, cfg, e_order=P.EDGE_BY_POS, **args).cpu().numpy()
        ref = O.binary_reduce(g, cfg, **{kw: x, "e": w})
        assert O.bit_equal(got, ref)
    assert O.bit_equal(gpu_reduce(g, (O.U, O.E, O.MUL, O.SUM, O.V), u=x, e=w), want)


def test_host_entry_matches_device_entry():
    src, dst = O.gen_rmat(1500, 20000, seed=6)
    g = O.Graph(1500, src, dst)
    x = O.normal_features(1500, 48, 1)
    w = O.gcn_weights(1500, src, dst)
    h = dev_graph(g, O.DST_MAJOR)
    cfg = (O.U, O.E, O.MUL, O.SUM, O.V)
    host = P.binary_reduce_host(h, cfg, u=x, e=w)
    assert O.bit_equal(host, O.binary_reduce(g, cfg, u=x, e=w))
    val, au, ae = P.binary_reduce_host(h, (O.U, O.NONE, O.COPY, O.MAX, O.V), u=x,
                                       want_arg_other=True, want_arg_edge=True)
    v2, au2, ae2 = O.copy_max_argmax(g, x)
    assert O.bit_equal(val, v2) and (au == au2).all() and (ae == ae2).all()


def test_async_host_entry_streams_steps():
    # gspmm_binary_reduce_host_async: forward and backward calls streamed on
    # two streams with alternating uploads (the bench's e2e schedule); every
    # step's outputs equal the synchronous entry's bit for bit
    src, dst = O.gen_rmat(2000, 30000, seed=8)
    g = O.Graph(2000, src, dst)
    w = O.gcn_weights(2000, src, dst)
    hd, hs = dev_graph(g, O.DST_MAJOR), dev_graph(g, O.SRC_MAJOR)
    cf, cb = (O.U, O.E, O.MUL, O.SUM, O.V), (O.V, O.E, O.MUL, O.SUM, O.U)
    sa, sb = torch.cuda.Stream(), torch.cuda.Stream()
    ea, eb = torch.cuda.Event(), torch.cuda.Event()
    ea.record(sa)
    eb.record(sb)
    wp = torch.from_numpy(w).pin_memory().numpy()
    outs = []
    for step in range(3):
        x = torch.from_numpy(O.normal_features(2000, 64, 10 + step)).pin_memory().numpy()
        gy = torch.from_numpy(O.normal_features(2000, 64, 20 + step)).pin_memory().numpy()
        of = torch.empty((2000, 64), pin_memory=True).numpy()
        ob = torch.empty((2000, 64), pin_memory=True).numpy()
        P.binary_reduce_host_async(hd, cf, u=x, e=wp, out=of, stream=sa,
                                   wait_event=eb if step else None, upload_event=ea)
        P.binary_reduce_host_async(hs, cb, v=gy, e=wp, out=ob, stream=sb, wait_event=ea,
                                   upload_event=eb)
        outs.append((x, gy, of, ob))
    sa.synchronize()
    sb.synchronize()
    for x, gy, of, ob in outs:
        assert O.bit_equal(of, P.binary_reduce_host(hd, cf, u=x, e=w))
        assert O.bit_equal(ob, P.binary_reduce_host(hs, cb, v=gy, e=w))
        assert O.bit_equal(of, O.binary_reduce(g, cf, u=x, e=w))


# ------------------------------------------- extensions
@pytest.mark.parametrize("seed", range(5))
def test_mean_and_mean_backward(seed):
    src, dst = O.gen_rmat(4000, 60000, seed=seed)
    g = O.Graph(4000, src, dst)
    x = O.random_features(4000, 100, seed)
    gy = O.normal_features(4000, 100, seed + 3)
    assert O.bit_equal(gpu_reduce(g, (O.U, O.NONE, O.COPY, P.MEAN, O.V), u=x), O.mean(g, x))
    # backward: v_copy_add_u scaled by 1/deg_in(v) of the gathered node
    deg = O.in_degree(g)
    inv = np.zeros(4000, np.float32)
    inv[deg > 0] = np.float32(1) / deg[deg > 0].astype(np.float32)
    h = dev_graph(g, O.SRC_MAJOR)
    got = P.binary_reduce(h, (O.V, O.NONE, O.COPY, O.SUM, O.U), v=cuda(gy),
                          other_scale=torch.from_numpy(inv).cuda()).cpu().numpy()
    assert O.bit_equal(got, O.mean_backward(g, gy))


@pytest.mark.parametrize("seed", range(5))
def test_max_argmax_and_backward(seed):
    src, dst = O.gen_rmat(3000, 50000, seed=seed)
    src, dst = O.symmetrize(src, dst)
    g = O.Graph(3000, src, dst)
    # few distinct values: ties between different sources and duplicate edges
    x = np.round(O.random_features(3000, 100, seed) * 4) / 4
    val, au, ae = gpu_reduce(g, (O.U, O.NONE, O.COPY, O.MAX, O.V), u=x, want_arg_other=True,
                             want_arg_edge=True)
    v2, au2, ae2 = O.copy_max_argmax(g, x)
    assert O.bit_equal(val, v2)
    assert O.bit_equal(val, O.binary_reduce(g, O.named_config("u_copy_max_v"), u=x))
    assert (au == au2).all() and (ae == ae2).all()
    # neighbour argmax alone: the kernels track the winning id directly
    val1, au1, _ = gpu_reduce(g, (O.U, O.NONE, O.COPY, O.MAX, O.V), u=x, want_arg_other=True)
    assert O.bit_equal(val1, v2) and (au1 == au2).all()
    gy = O.normal_features(3000, 100, seed + 3)
    grad = P.argmax_backward(torch.from_numpy(au).cuda(), cuda(gy), 3000).cpu().numpy()
    want = O.argmax_backward(au2, gy, 3000)
    assert O.max_rel_error(grad, want) <= 1e-6
    # min + argmin
    val, au, _ = gpu_reduce(g, (O.U, O.NONE, O.COPY, O.MIN, O.V), u=x, want_arg_other=True)
    assert O.bit_equal(val, O.binary_reduce(g, O.named_config("u_copy_min_v"), u=x))


def test_argmax_over_edge_features():
    src, dst = O.gen_rmat(500, 8000, seed=2)
    g = O.Graph(500, src, dst)
    fe = np.round(O.random_features(g.m, 16, 3) * 3) / 3
    val, au, ae = gpu_reduce(g, (O.E, O.NONE, O.COPY, O.MAX, O.V), e=fe, want_arg_other=True,
                             want_arg_edge=True)
    v2, au2, ae2 = O.copy_max_argmax(g, fe, lhs=O.E)
    assert O.bit_equal(val, v2) and (au == au2).all() and (ae == ae2).all()


@pytest.mark.parametrize("seed", range(3))
def test_multihead_forward_backward(seed):
    heads, d = 8, 64
    src, dst = O.gen_rmat(2000, 40000, seed=seed)
    g = O.Graph(2000, src, dst)
    x = O.normal_features(2000, heads * d, seed)
    a = O.softmax_attention(2000, dst, O.normal_features(g.m, heads, seed + 2))
    gy = O.normal_features(2000, heads * d, seed + 3)
    fwd = gpu_reduce(g, (O.U, O.E, O.MUL, O.SUM, O.V), u=x, e=a, heads=heads)
    assert O.bit_equal(fwd, O.multihead_u_mul_e_sum(g, x, a, heads))
    gx_want, ga_want = O.multihead_backward(g, x, a, gy, heads)
    gx = gpu_reduce(g, (O.V, O.E, O.MUL, O.SUM, O.U), v=gy, e=a, heads=heads)
    assert O.bit_equal(gx, gx_want)
    ga = gpu_reduce(g, (O.U, O.V, O.DOT, O.LAST, O.E), u=x, v=gy, heads=heads)
    assert O.bit_equal(ga, ga_want)


def test_long_rows_hub():
    # a hub with 60k in-edges and 40k out-edges exercises the long-row plan
    rng = np.random.default_rng(0)
    n = 5000
    src = np.concatenate([rng.integers(0, n, 60000), np.zeros(40000, np.int64),
                          rng.integers(0, n, 20000)]).astype(np.uint32)
    dst = np.concatenate([np.zeros(60000, np.int64), rng.integers(0, n, 40000),
                          rng.integers(0, n, 20000)]).astype(np.uint32)
    g = O.Graph(n, src, dst)
    x = O.normal_features(n, 128, 1)
    w = O.gcn_weights(n, src, dst)
    for cfg, kw in (((O.U, O.E, O.MUL, O.SUM, O.V), dict(u=x, e=w)),
                    ((O.V, O.E, O.MUL, O.SUM, O.U), dict(v=x, e=w)),
                    ((O.U, O.NONE, O.COPY, O.MAX, O.V), dict(u=x))):
        assert O.bit_equal(gpu_reduce(g, cfg, **kw), O.binary_reduce(g, cfg, **kw))
    assert dev_graph(g, O.DST_MAJOR).num_long_rows >= 1


@pytest.mark.parametrize("seg,long_", [(1, 2), (7, 16), (64, 100), (3, 100000)])
def test_plan_granularity_does_not_change_results(seg, long_):
    # tiny segments / long-row thresholds force every unit boundary case of
    # the planned kernels (rows split across units, empty rows at unit
    # edges, many long rows run as column units) -- results stay bitwise
    src, dst = O.gen_rmat(1500, 25000, seed=seg)
    src, dst = O.add_self_loops(1500, src, dst)
    g = O.Graph(1500, src, dst)
    g.plan = dict(seg_cost=seg, long_threshold=long_)
    for dim in (4, 100, 256, 300):
        x = O.normal_features(1500, dim, dim)
        w = O.gcn_weights(1500, src, dst)
        cases = [((O.U, O.E, O.MUL, O.SUM, O.V), dict(u=x, e=w)),
                 ((O.V, O.E, O.MUL, O.SUM, O.U), dict(v=x, e=w)),
                 ((O.U, O.NONE, O.COPY, O.MAX, O.V), dict(u=x)),
                 ((O.U, O.NONE, O.COPY, P.MEAN, O.V), dict(u=x))]
        for cfg, kw in cases:
            got = gpu_reduce(g, cfg, **kw)
            want = O.mean(g, x) if cfg[3] == P.MEAN else O.binary_reduce(g, cfg, **kw)
            assert O.bit_equal(got, want), (seg, long_, dim, cfg)
        g.__dict__.pop("_dev", None)  # rebuild handles with the next plan


def test_register_path_matches_planned_path():
    # the register kernel (rows.cu, plan kernel=1) and the planned kernels
    # (k_gather + k_long_rg) must agree bitwise, long rows included
    src, dst = O.gen_rmat(3000, 60000, seed=9)
    g = O.Graph(3000, src, dst)
    x = O.normal_features(3000, 256, 1)
    w = O.gcn_weights(3000, src, dst)
    h = P.Graph(*g.dst_major, orientation=P.DST_MAJOR)
    h.set_plan(long_threshold=200)
    assert h.num_long_rows > 0
    planned = P.binary_reduce(h, "u_mul_e_add_v", u=cuda(x), e=cuda(w)).cpu().numpy()
    h.set_plan(kernel=1)
    before = P.launch_count()
    reg = P.binary_reduce(h, "u_mul_e_add_v", u=cuda(x), e=cuda(w)).cpu().numpy()
    assert P.launch_count() - before == 1  # one rows.cu launch
    assert O.bit_equal(planned, reg)
    assert O.bit_equal(reg, O.binary_reduce(g, O.named_config("u_mul_e_add_v"), u=x, e=w))


def test_programmatic_dependent_pair_matches_serial_launches():
    # plan kernel=2: the segment kernel is a programmatic dependent of the
    # long-row kernel (its blocks start while long-row CTAs still run); the
    # outputs, the fused second reduction included, stay bitwise, call after
    # call on one stream
    src, dst = O.gen_rmat(4000, 90000, seed=11)
    g = O.Graph(4000, src, dst)
    x = O.normal_features(4000, 100, 2)
    h = P.Graph(*g.dst_major, orientation=P.DST_MAJOR)
    h.set_plan(long_threshold=150, kernel=2)
    assert h.num_long_rows > 0
    want_sum = O.binary_reduce(g, O.named_config("u_copy_add_v"), u=x)
    want_max = O.binary_reduce(g, O.named_config("u_copy_max_v"), u=x)
    xd = cuda(x)
    for _ in range(3):
        assert O.bit_equal(P.binary_reduce(h, "u_copy_add_v", u=xd).cpu().numpy(), want_sum)
        assert O.bit_equal(P.binary_reduce(h, "u_copy_max_v", u=xd).cpu().numpy(), want_max)


@pytest.mark.parametrize("edges", [64, 512, 100000])
def test_long_rows_split_by_edges(edges):
    # plan split_edges = N: long rows are folded as chunks of ~N edges and the
    # chunk partials combined in chunk order.  Max / Min values and both
    # argmax outputs keep the reference's bits (ties, first-wins).  Sums and
    # means are bit-identical on every row that is not split and the same
    # bits run after run; on a split row they are another fp32 summation
    # order, about as far (max_rel_error, compare.hpp:30-45) from the EXACT
    # f64 sum of the same fp32 messages as the reference's own fold is.  That
    # fold of a 40,000-edge row of N(0,1) values is ~3e-4 away from the exact
    # sum (partial sums reach a few hundred, each add rounds at 6e-8 of
    # that), so NO re-associated sum stays within 1e-5 of the reference on
    # hub rows -- which is why the default keeps the sequential order;
    # against the reference only a loose sanity bound is checked.  Scalar edge weights (by edge id and by CSR position),
    # per-head weights, the per-neighbour scale, the fused second reduction
    # and two-slice / wide widths all take the chunk path.
    rng = np.random.default_rng(5)
    n = 3000
    src = np.concatenate([rng.integers(0, n, 40000), rng.integers(0, n, 30000),
                          rng.integers(0, n, 5000)]).astype(np.uint32)
    dst = np.concatenate([np.zeros(40000, np.int64) + 5, rng.integers(0, n, 30000),
                          np.zeros(5000, np.int64) + 17]).astype(np.uint32)
    g = O.Graph(n, src, dst)
    g.plan = dict(long_threshold=1000, split_edges=edges)
    w = O.gcn_weights(n, src, dst)
    long_rows = np.array([5, 17])
    short = np.setdiff1d(np.arange(n), long_rows)

    in_edges = {r: np.nonzero(dst == r)[0] for r in long_rows}

    def check_sum(got, want, messages, div=False):
        assert O.bit_equal(got[short], want[short])
        assert O.max_rel_error(got, want) <= 2e-2  # sanity only
        for r in long_rows:  # the exact sum of the fp32 messages of row r
            exact = messages(in_edges[r]).astype(np.float64).sum(0)
            if div:
                exact = exact / len(in_edges[r])
            exact = exact.astype(np.float32)
            # the same order of rounding error as the reference's own fold
            assert O.max_rel_error(got[r], exact) <= \
                4 * max(O.max_rel_error(want[r], exact), SUM_TOL), r

    for dim in (4, 100, 256, 300, 512, 602):
        x = O.normal_features(n, dim, dim)
        xq = (np.round(x * 4) / 4).astype(np.float32)  # quantised: ties are real
        h = dev_graph(g, O.DST_MAJOR)
        assert h.num_long_rows == 2
        cfg = O.named_config("u_mul_e_add_v")
        got = gpu_reduce(g, cfg, u=x, e=w)
        check_sum(got, O.binary_reduce(g, cfg, u=x, e=w), lambda j: x[src[j]] * w[j].reshape(-1, 1))
        assert O.bit_equal(got, gpu_reduce(g, cfg, u=x, e=w))  # deterministic
        wp = h.permute_edges(cuda(w))
        got_pos = P.binary_reduce(h, cfg, u=cuda(x), e=wp, e_order=P.EDGE_BY_POS).cpu().numpy()
        assert O.bit_equal(got_pos, got)
        check_sum(gpu_reduce(g, O.named_config("u_copy_add_v"), u=x),
                  O.binary_reduce(g, O.named_config("u_copy_add_v"), u=x), lambda j: x[src[j]])
        check_sum(P.binary_reduce(h, (O.U, O.NONE, O.COPY, P.MEAN, O.V), u=cuda(x)).cpu().numpy(),
                  O.mean(g, x), lambda j: x[src[j]], div=True)
        for red in (O.MAX, O.MIN):
            c = (O.U, O.NONE, O.COPY, red, O.V)
            assert O.bit_equal(gpu_reduce(g, c, u=xq), O.binary_reduce(g, c, u=xq)), (dim, red)
        o2 = torch.empty((n, dim), device="cuda")
        v, ao, ae = P.binary_reduce(h, (O.U, O.NONE, O.COPY, O.MAX, O.V), u=cuda(xq), out2=o2,
                                    reduce2=P.MEAN, want_arg_other=True, want_arg_edge=True)
        wv, wa, we = O.copy_max_argmax(g, xq)
        assert O.bit_equal(v.cpu().numpy(), wv)
        assert np.array_equal(ao.cpu().numpy(), wa) and np.array_equal(ae.cpu().numpy(), we)
        check_sum(o2.cpu().numpy(), O.mean(g, xq), lambda j: xq[src[j]], div=True)
        res = P.binary_reduce(h, (O.U, O.NONE, O.COPY, O.MAX, O.V), u=cuda(xq),
                              want_arg_other=True)
        assert O.bit_equal(res[0].cpu().numpy(), wv) and np.array_equal(res[1].cpu().numpy(), wa)
        g.__dict__.pop("_dev", None)
    # per-head weights (8 heads x 64 columns) and the mean backward's scale
    x = O.normal_features(n, 512, 9)
    a = O.normal_features(len(src), 8, 10)
    got = gpu_reduce(g, (O.U, O.E, O.MUL, O.SUM, O.V), u=x, e=a, heads=8)
    want = O.multihead_u_mul_e_sum(g, x, a, 8)
    check_sum(got, want, lambda j: x[src[j]] * np.repeat(a[j], 64, axis=1))


@pytest.mark.parametrize("cols", [0, 4, 8, 12, 32, 64, 128, 132, 256, 512])
@pytest.mark.parametrize("split", [1, 0])  # 1: max on the long-row kernel; 0: max in edge chunks
def test_long_row_column_units(cols, split):
    # long rows run as column units of `cols` columns (0: the automatic
    # widths); every unit width, argmax and scalar / per-head / per-neighbour
    # small operands included, stays bitwise for every feature width
    rng = np.random.default_rng(cols + 7)
    n = 3000
    src = np.concatenate([rng.integers(0, n, 40000), rng.integers(0, n, 30000),
                          rng.integers(0, n, 5000)]).astype(np.uint32)
    dst = np.concatenate([np.zeros(40000, np.int64) + 5, rng.integers(0, n, 30000),
                          np.zeros(5000, np.int64) + 17]).astype(np.uint32)
    g = O.Graph(n, src, dst)
    g.plan = dict(long_threshold=1000, unit_cols=cols, split_edges=split)
    w = O.gcn_weights(n, src, dst)
    for dim in (4, 20, 100, 128, 256, 300, 512):
        x = O.normal_features(n, dim, dim)
        for cfg, kw in (((O.U, O.E, O.MUL, O.SUM, O.V), dict(u=x, e=w)),
                        ((O.U, O.NONE, O.COPY, O.SUM, O.V), dict(u=x)),
                        ((O.U, O.NONE, O.COPY, O.MAX, O.V), dict(u=x))):
            assert O.bit_equal(gpu_reduce(g, cfg, **kw), O.binary_reduce(g, cfg, **kw)), (cols, dim)
        assert dev_graph(g, O.DST_MAJOR).num_long_rows == 2
        val, au, ae = gpu_reduce(g, (O.U, O.NONE, O.COPY, O.MAX, O.V), u=x, want_arg_other=True,
                                 want_arg_edge=True)
        v2, au2, ae2 = O.copy_max_argmax(g, x)
        assert O.bit_equal(val, v2) and (au == au2).all() and (ae == ae2).all()
        if dim % 8 == 0 and dim >= 16:  # per-head weights (8 heads)
            a = O.normal_features(len(src), 8, dim + 1)
            want = O.multihead_u_mul_e_sum(g, x, a, 8)
            got = gpu_reduce(g, (O.U, O.E, O.MUL, O.SUM, O.V), u=x, e=a, heads=8)
            assert O.bit_equal(got, want), (cols, dim)
        # mean backward on the src-major handle: per-neighbour scale
        gy = O.normal_features(n, dim, dim + 2)
        deg = O.in_degree(g)
        inv = np.zeros(n, np.float32)
        inv[deg > 0] = np.float32(1) / deg[deg > 0].astype(np.float32)
        got = gpu_reduce(g, (O.V, O.NONE, O.COPY, O.SUM, O.U), v=gy,
                         other_scale=torch.from_numpy(inv).cuda())
        assert O.bit_equal(got, O.mean_backward(g, gy)), (cols, dim)
        g.__dict__.pop("_dev", None)


@pytest.mark.parametrize("nb", [2, 3, 7])
def test_source_blocks_bit_exact(nb):
    # Source blocking (the paper's Alg. 3): nb passes, each folding one
    # neighbour-id block into the partial rows of the previous passes, must
    # give the single-pass result bit for bit -- sums, mean, max / min with
    # the zero-degree fixup, per-edge weights by edge id, the mean backward's
    # per-neighbour scale, and long rows (the hub) on both kernels.
    rng = np.random.default_rng(nb)
    n = 3000
    src = np.concatenate([rng.integers(0, n, 40000), rng.integers(0, n, 3000),
                          np.full(2000, 7)]).astype(np.uint32)
    dst = np.concatenate([rng.integers(0, n // 2, 40000), np.zeros(3000, np.int64),
                          rng.integers(0, n, 2000)]).astype(np.uint32)
    g = O.Graph(n, src, dst)  # rows >= n/2 get few in-edges: empty block ranges
    g.plan = dict(long_threshold=300)
    x = O.normal_features(n, 200, nb)
    w = O.gcn_weights(n, src, dst)
    gy = O.normal_features(n, 200, nb + 3)
    deg = O.in_degree(g)
    inv = np.zeros(n, np.float32)
    inv[deg > 0] = np.float32(1) / deg[deg > 0].astype(np.float32)
    cases = [((O.U, O.E, O.MUL, O.SUM, O.V), dict(u=x, e=w), None),
             ((O.V, O.E, O.MUL, O.SUM, O.U), dict(v=x, e=w), None),
             ((O.U, O.NONE, O.COPY, O.MAX, O.V), dict(u=x), None),
             ((O.U, O.NONE, O.COPY, O.MIN, O.V), dict(u=x), None),
             ((O.U, O.NONE, O.COPY, P.MEAN, O.V), dict(u=x), O.mean(g, x)),
             ((O.V, O.NONE, O.COPY, O.SUM, O.U), dict(v=gy), O.mean_backward(g, gy))]
    for cfg, kw, want in cases:
        orientation = O.SRC_MAJOR if cfg[4] == O.U else O.DST_MAJOR
        h = dev_graph(g, orientation)
        extra = {}
        if want is not None and cfg[4] == O.U:
            extra["other_scale"] = torch.from_numpy(inv).cuda()
        h.set_source_blocks(1)
        plain = P.binary_reduce(h, cfg, *(cuda(kw.get(k)) for k in ("u", "v", "e")), **extra)
        torch.cuda.synchronize()
        h.set_source_blocks(nb)
        before = P.launch_count()
        got = P.binary_reduce(h, cfg, *(cuda(kw.get(k)) for k in ("u", "v", "e")), **extra)
        torch.cuda.synchronize()
        assert P.launch_count() - before >= nb, "blocked passes did not run"
        h.set_source_blocks(0)
        if want is None:
            want = O.binary_reduce(g, cfg, **kw)
        got, plain = got.cpu().numpy(), plain.cpu().numpy()
        assert O.bit_equal(plain, want), cfg
        assert O.bit_equal(got, want), (nb, cfg)


def test_row_shards_with_global_edge_ids():
    # a rank's handle over a row shard keeps global neighbour and edge ids
    # (bench.py / shard.py): edge operands in edge-id order must be permuted
    # to the shard's CSR positions (one row per shard edge), and the shard's
    # rows of every result equal the whole graph's, bit for bit
    from paper_2007_06354_b200.shard import balanced_row_ranges, slice_csr
    src, dst = O.gen_rmat(3000, 40000, seed=11)
    src, dst = O.add_self_loops(3000, src, dst)
    g = O.Graph(3000, src, dst)
    x = O.normal_features(3000, 64, 3)
    w = O.gcn_weights(3000, src, dst)
    cfg = (O.U, O.E, O.MUL, O.SUM, O.V)
    want = O.binary_reduce(g, cfg, u=x, e=w)
    ip, ix, ei = g.csr(O.DST_MAJOR)
    bounds = balanced_row_ranges(ip, 3)
    for k in range(3):
        lo, hi = int(bounds[k]), int(bounds[k + 1])
        sip, six, sei = slice_csr(ip, ix, ei, lo, hi)
        h = P.Graph(sip, six, sei, num_rows=hi - lo, num_cols=3000, orientation=P.DST_MAJOR)
        wp = h.permute_edges(cuda(w))
        assert wp.shape[0] == h.num_edges
        got = P.binary_reduce(h, cfg, u=cuda(x), e=wp, e_order=P.EDGE_BY_POS).cpu().numpy()
        assert O.bit_equal(got, want[lo:hi])
        got_h = P.binary_reduce_host(h, cfg, u=x, e=w[sei], e_order=P.EDGE_BY_POS)
        assert O.bit_equal(got_h, want[lo:hi])


def test_wide_rows_mean_and_mean_backward():
    # 602-column rows with a 16-byte leading dimension (cfg5's layout): one
    # wide segment unit per row (up to 640 columns), the fused mean
    # epilogue, and the mean backward's per-neighbour scale applied once per
    # gathered row -- all bit-exact
    src, dst = O.gen_rmat(2500, 60000, seed=4)
    g = O.Graph(2500, src, dst)
    x = O.normal_features(2500, 602, 7)
    gy = O.normal_features(2500, 602, 8)
    xp = torch.zeros((2500, 604), device="cuda")
    xp[:, :602] = cuda(x)
    gp = torch.zeros((2500, 604), device="cuda")
    gp[:, :602] = cuda(gy)
    op = torch.empty((2500, 604), device="cuda")
    hd, hs = dev_graph(g, O.DST_MAJOR), dev_graph(g, O.SRC_MAJOR)
    P.binary_reduce(hd, (O.U, O.NONE, O.COPY, P.MEAN, O.V), u=xp[:, :602], out=op[:, :602])
    assert O.bit_equal(op[:, :602].cpu().numpy(), O.mean(g, x))
    deg = O.in_degree(g)
    inv = np.zeros(2500, np.float32)
    inv[deg > 0] = np.float32(1) / deg[deg > 0].astype(np.float32)
    P.binary_reduce(hs, (O.V, O.NONE, O.COPY, O.SUM, O.U), v=gp[:, :602], out=op[:, :602],
                    other_scale=torch.from_numpy(inv).cuda())
    assert O.bit_equal(op[:, :602].cpu().numpy(), O.mean_backward(g, gy))


@pytest.mark.parametrize("dim,pad", [(100, 0), (128, 4), (37, 0), (64, 2)])
def test_argmax_backward_vector_and_scalar_paths(dim, pad):
    """a17.4 scatter through the argmax: dim % 4 == 0 with 16-byte rows takes
    the 4-column kernels, other widths / padded leading dims the scalar ones;
    -1 ids (rows without in-edges) contribute nothing."""
    rng = np.random.default_rng(dim + pad)
    rows, src_rows = 5000, 1200
    arg = rng.integers(-1, src_rows, size=(rows, dim), dtype=np.int32)
    arg[::7] = -1
    gy = O.normal_features(rows, dim, dim)
    want = O.argmax_backward(arg, gy, src_rows)
    a_full = torch.zeros((rows, dim + pad), dtype=torch.int32, device="cuda")
    g_full = torch.zeros((rows, dim + pad), dtype=torch.float32, device="cuda")
    a_full[:, :dim] = torch.from_numpy(arg).cuda()
    g_full[:, :dim] = cuda(gy)
    o_full = torch.full((src_rows, dim + pad), 7.0, dtype=torch.float32, device="cuda")
    got = P.argmax_backward(a_full[:, :dim], g_full[:, :dim], src_rows, out=o_full[:, :dim])
    assert O.max_rel_error(got.cpu().numpy(), want) <= 1e-6
    if pad:
        assert (o_full[:, dim:] == 7.0).all()


@pytest.mark.parametrize("long_", [0, 150])
def test_second_reduction_fused_and_fallback(long_):
    # out2 / reduce2: a second reduction of the same messages in the same
    # call -- fused into one gather for copy + max/min (argmax included, long
    # rows included), a second pass for any other config; always bitwise
    # equal to the separate call
    src, dst = O.gen_rmat(3000, 60000, seed=21)
    g = O.Graph(3000, src, dst)
    if long_:
        g.plan = dict(long_threshold=long_)
    w = O.gcn_weights(3000, src, dst)
    for dim in (7, 100, 128, 256):
        x = O.normal_features(3000, dim, dim)
        xd = cuda(x)
        h = dev_graph(g, O.DST_MAJOR)
        mean_want, sum_want = O.mean(g, x), O.binary_reduce(g, O.named_config("u_copy_add_v"), u=x)
        for red, arg in ((O.MAX, True), (O.MAX, False), (O.MIN, True)):
            for red2, want2 in ((P.MEAN, mean_want), (P.SUM, sum_want)):
                o2 = torch.empty((3000, dim), device="cuda")
                res = P.binary_reduce(h, (O.U, O.NONE, O.COPY, red, O.V), u=xd, out2=o2,
                                      reduce2=red2, want_arg_other=arg, want_arg_edge=arg)
                v = res[0] if arg else res
                want = O.binary_reduce(g, (O.U, O.NONE, O.COPY, red, O.V), u=x)
                assert O.bit_equal(v.cpu().numpy(), want), (dim, red, red2)
                assert O.bit_equal(o2.cpu().numpy(), want2), (dim, red, red2)
                if arg and red == O.MAX:
                    wv, wa, we = O.copy_max_argmax(g, x)
                    assert np.array_equal(res[1].cpu().numpy(), wa)
                    assert np.array_equal(res[2].cpu().numpy(), we)
        # fallback (second pass): u_mul_e + sum with a mean second output
        o2 = torch.empty((3000, dim), device="cuda")
        got = P.binary_reduce(h, "u_mul_e_add_v", u=xd, e=cuda(w), out2=o2, reduce2=P.MEAN)
        want = O.binary_reduce(g, O.named_config("u_mul_e_add_v"), u=x, e=w)
        deg = O.in_degree(g).astype(np.float32)[:, None]
        assert O.bit_equal(got.cpu().numpy(), want)
        assert O.bit_equal(o2.cpu().numpy(), np.where(deg > 0, want / np.maximum(deg, 1), 0)
                           .astype(np.float32))
        g.__dict__.pop("_dev", None)


@pytest.mark.parametrize("cols", [0, 8, 28, 100])
@pytest.mark.parametrize("split", [1, 0, 64])  # long-row kernel; default edge chunks; small chunks
def test_long_row_argmax_ties_zeros_and_nans(cols, split):
    # The long-row units take each 16-edge block's extremum from an FMNMX
    # tree and resolve the winner at the flush: the first-canonical-position
    # rule, the sign of a zero extremum (the reference's `a < m ? m : a`
    # keeps the EARLIER of -0 / +0), NaN never winning, and rows whose every
    # value is NaN or -inf must all come out bit for bit, max and min, with
    # and without the fused mean.  The same holds for the default path of a
    # plain max / min, long rows folded as chunks of edges and combined in
    # chunk order (split 0 and 64; the fused mean keeps the long-row kernel).
    rng = np.random.default_rng(91 + cols)
    n = 2000
    src = np.concatenate([rng.integers(0, n, 20000), rng.integers(0, n, 20000),
                          rng.integers(0, 40, 3000), rng.integers(0, n, 1500)]).astype(np.uint32)
    dst = np.concatenate([np.zeros(20000, np.int64) + 3, rng.integers(0, n, 20000),
                          np.zeros(3000, np.int64) + 11,
                          np.zeros(1500, np.int64) + 29]).astype(np.uint32)
    g = O.Graph(n, src, dst)
    g.plan = dict(long_threshold=1000, unit_cols=cols, split_edges=split)
    for dim in (8, 36, 100, 260):
        # few distinct values: -1, -0.0, +0.0, 0.5, NaN; column 1 only zeros
        # of both signs, column 2 only NaN, column 3 only -inf, column 4
        # nothing above -0.0
        pool = np.array([-1.0, -0.0, 0.0, 0.5, np.nan], np.float32)
        x = pool[rng.integers(0, len(pool), (n, dim))]
        x[:, 1] = np.where(rng.integers(0, 2, n) == 0, np.float32(-0.0), np.float32(0.0))
        x[:, 2] = np.nan
        x[:, 3] = -np.inf
        x[:, 4] = np.where(rng.integers(0, 2, n) == 0, np.float32(-0.0), np.float32(-1.0))
        for red in (O.MAX, O.MIN):
            cfg = (O.U, O.NONE, O.COPY, red, O.V)
            want = O.binary_reduce(g, cfg, u=x)
            val, au, ae = gpu_reduce(g, cfg, u=x, want_arg_other=True, want_arg_edge=True)
            assert val.tobytes() == want.tobytes(), (cols, dim, red)  # sign of zero included
            if red == O.MAX:
                v2, au2, ae2 = O.copy_max_argmax(g, x)
                assert val.tobytes() == v2.tobytes()
                assert np.array_equal(au, au2) and np.array_equal(ae, ae2), (cols, dim)
            else:  # the winner's feature is the extremum, bit for bit (or no winner)
                won = au >= 0
                picked = x[np.where(won, au, 0), np.arange(dim)[None, :]]
                assert (picked.view(np.uint32)[won] == val.view(np.uint32)[won]).all()
            # plain extremum (no argmax) and the fused second reduction
            assert gpu_reduce(g, cfg, u=x).tobytes() == want.tobytes()
        if split > 1:  # sums of split rows are not the reference's bits
            g.__dict__.pop("_dev", None)
            continue
        xz = np.nan_to_num(x, nan=0.25, neginf=-2.0)  # finite values for the mean
        o2 = torch.empty((n, dim), device="cuda")
        h = dev_graph(g, O.DST_MAJOR)
        res = P.binary_reduce(h, (O.U, O.NONE, O.COPY, O.MAX, O.V), u=cuda(xz), out2=o2,
                              reduce2=P.MEAN, want_arg_other=True, want_arg_edge=True)
        v2, au2, ae2 = O.copy_max_argmax(g, xz)
        assert res[0].cpu().numpy().tobytes() == v2.tobytes()
        assert np.array_equal(res[1].cpu().numpy(), au2) and np.array_equal(res[2].cpu().numpy(), ae2)
        assert o2.cpu().numpy().tobytes() == O.mean(g, xz).tobytes()
        g.__dict__.pop("_dev", None)


def test_zero_width_operands_give_rows_by_zero():
    # the reference returns a rows x 0 FeatureMatrix for zero-width operands
    # (binary_out_dim, ops.cpp:63-67); a dot or a 0-against-1 broadcast has
    # nothing to read there and is rejected
    g = g_of(4, [(0, 1), (2, 1), (3, 0)])
    h = dev_graph(g, O.DST_MAJOR)
    z = torch.empty((4, 0), device="cuda")
    ze = torch.empty((3, 0), device="cuda")
    assert tuple(P.out_shape(h, "u_copy_add_v", u=z)) == (4, 0)
    assert P.binary_reduce(h, "u_copy_add_v", u=z).shape == (4, 0)
    assert P.binary_reduce(h, "u_mul_e_add_v", u=z, e=ze).shape == (4, 0)
    assert P.binary_reduce(h, "u_add_v_copy_e", u=z, v=z).shape == (3, 0)
    with pytest.raises(P.ShapeError):
        P.binary_reduce(h, "u_dot_v_copy_e", u=z, v=z)
    with pytest.raises(P.ShapeError):
        P.binary_reduce(h, "u_mul_e_add_v", u=z, e=torch.ones((3, 1), device="cuda"))
    with pytest.raises(P.ShapeError):  # wrong row count is still reported first
        P.binary_reduce(h, "u_copy_add_v", u=torch.empty((5, 0), device="cuda"))


def test_large_table_geometry_all_operator_families():
    # <= 128-column segment units switch to the 4-edges x 5-blocks geometry
    # when the gathered table exceeds the L2 (gather_impl.cuh launch_k): a
    # 400k x 64 table (102 MB) puts every operator family on that instance --
    # copy, u_mul_e with scalar and per-head weights, add / sub / div, max +
    # argmax with the fused mean, the mean backward's per-neighbour scale,
    # copy_e -- bitwise against the oracle.
    n, m, F = 400_000, 2_500_000, 64
    src, dst = P.synth_rmat(n, m, 0.45, 0.22, 0.22, 0.11, 5)
    g = O.Graph(n, src, dst)
    x = O.normal_features(n, F, 1)
    v = O.random_features(n, F, 2) + np.float32(2.0)  # away from zero: a divisor
    w = O.gcn_weights(n, src, dst)
    for name, kw in (("u_copy_add_v", dict(u=x)), ("u_mul_e_add_v", dict(u=x, e=w)),
                     ("u_add_v_add_v", dict(u=x, v=v)), ("u_sub_v_add_v", dict(u=x, v=v)),
                     ("u_div_v_add_v", dict(u=x, v=v)), ("u_mul_v_max_v", dict(u=x, v=v)),
                     ("u_copy_min_v", dict(u=x)), ("v_mul_e_add_u", dict(v=x, e=w))):
        cfg = O.named_config(name)
        assert O.bit_equal(gpu_reduce(g, cfg, **kw), O.binary_reduce(g, cfg, **kw)), name
    a = O.normal_features(m, 8, 3)
    assert O.bit_equal(gpu_reduce(g, (O.U, O.E, O.MUL, O.SUM, O.V), u=x, e=a, heads=8),
                       O.multihead_u_mul_e_sum(g, x, a, 8))
    h = dev_graph(g, O.DST_MAJOR)
    o2 = torch.empty((n, F), device="cuda")
    val, au, ae = P.binary_reduce(h, (O.U, O.NONE, O.COPY, O.MAX, O.V), u=cuda(x), out2=o2,
                                  reduce2=P.MEAN, want_arg_other=True, want_arg_edge=True)
    v2, au2, ae2 = O.copy_max_argmax(g, x)
    assert O.bit_equal(val.cpu().numpy(), v2) and np.array_equal(au.cpu().numpy(), au2)
    assert np.array_equal(ae.cpu().numpy(), ae2) and O.bit_equal(o2.cpu().numpy(), O.mean(g, x))
    deg = O.in_degree(g)
    inv = np.zeros(n, np.float32)
    inv[deg > 0] = np.float32(1) / deg[deg > 0].astype(np.float32)
    got = gpu_reduce(g, (O.V, O.NONE, O.COPY, O.SUM, O.U), v=x, other_scale=torch.from_numpy(inv).cuda())
    assert O.bit_equal(got, O.mean_backward(g, x))
    ef = O.normal_features(m, F, 4)  # copy_e: the gathered table is the edge matrix (640 MB)
    cfg = O.named_config("e_copy_add_v")
    assert O.bit_equal(gpu_reduce(g, cfg, e=ef), O.binary_reduce(g, cfg, e=ef))
