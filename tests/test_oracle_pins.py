"""Pins the C restatement (oracle/) before it is trusted as the checker.

(a) hand goldens of the reference's own doctest suites
    (proj/tests/test_graph.cpp, test_kernels.cpp, test_oracle.cpp,
    test_generators.cpp, test_features.cpp), restated as pytest cases;
(b) fixtures produced by the unmodified reference library
    (tests/golden/reference_outputs.npz, made by tests/golden/make_golden.py);
(c) when oracle/_ref is present, a direct comparison on fresh seeds.
All CPU-only.
"""
import numpy as np
import pytest

from oracle import oracle as O


def g_of(n, edges):
    src = np.array([e[0] for e in edges], np.uint32)
    dst = np.array([e[1] for e in edges], np.uint32)
    return O.Graph(n, src, dst)


# ------------------------------------------------------- test_graph.cpp
def test_build_csr_dst_major_golden():  # test_graph.cpp:39-46
    ip, ix, ei = O.build_csr(3, [0, 1, 0], [2, 2, 1], O.DST_MAJOR)
    assert ip.tolist() == [0, 0, 1, 3]
    assert ix.tolist() == [0, 0, 1]
    assert ei.tolist() == [2, 0, 1]
    assert O.validate(3, 3, ip, ix, ei) == 0


def test_build_csr_empty_and_self_loop():  # test_graph.cpp:48-65
    ip, ix, ei = O.build_csr(2, [], [], O.DST_MAJOR)
    assert ip.tolist() == [0, 0, 0] and len(ix) == 0
    for o in (O.SRC_MAJOR, O.DST_MAJOR):
        ip, ix, ei = O.build_csr(1, [0], [0], o)
        assert ip.tolist() == [0, 1] and ix.tolist() == [0] and ei.tolist() == [0]


def test_build_csr_rejects_out_of_range():  # test_graph.cpp:67-70
    with pytest.raises(O.OracleError):
        O.build_csr(2, [0], [2])


def test_transpose_golden():  # test_graph.cpp:71-80
    ip, ix, ei = O.build_csr(3, [0, 1, 0], [2, 2, 1], O.DST_MAJOR)
    t = O.transpose(3, 3, ip, ix, ei)
    assert t[0].tolist() == [0, 2, 3, 3]
    assert t[1].tolist() == [1, 2, 2]
    assert t[2].tolist() == [2, 0, 1]


def test_validate_reports_violations():  # test_graph.cpp:95-119
    assert O.validate(2, 2, [0, 2, 1], [0], [0]) == 3       # not monotone
    assert O.validate(1, 2, [0, 2], [0, 1], [0, 0]) == 6    # eids not a permutation
    ok = O.build_csr(3, [0, 1], [2, 2])
    assert O.validate(3, 3, *ok) == 0


@pytest.mark.parametrize("seed", range(1, 26))
def test_csr_roundtrip_property(seed):  # test_graph.cpp:145-159 / 161-176
    n, src, dst = O.random_small_graph(seed)
    for o in (O.SRC_MAJOR, O.DST_MAJOR):
        ip, ix, ei = O.build_csr(n, src, dst, o)
        assert O.validate(n, n, ip, ix, ei) == 0
        rows = np.repeat(np.arange(n), np.diff(ip.astype(np.int64)))
        back_src = np.empty(len(src), np.uint32)
        back_dst = np.empty(len(src), np.uint32)
        if o == O.DST_MAJOR:
            back_src[ei], back_dst[ei] = ix, rows
        else:
            back_src[ei], back_dst[ei] = rows, ix
        assert (back_src == src).all() and (back_dst == dst).all()
    g = O.build_csr(n, src, dst, O.DST_MAJOR)
    tt = O.transpose(n, n, *O.transpose(n, n, *g))
    assert all((a == b).all() for a, b in zip(tt, g))


# -------------------------------------------------- test_kernels.cpp
def test_copy_sum_golden():  # test_kernels.cpp:49-66
    g = g_of(3, [(0, 2), (1, 2)])
    out = O.binary_reduce(g, O.named_config("u_copy_add_v"), u=np.array([[1, 2], [3, 4], [0, 0]]))
    assert out.tolist() == [[0, 0], [0, 0], [4, 6]]


def test_single_edge_copy():  # :68-78
    g = g_of(2, [(0, 1)])
    out = O.binary_reduce(g, O.named_config("u_copy_add_v"), u=np.array([[5, -3], [9, 9]]))
    assert out.tolist() == [[0, 0], [5, -3]]


def test_max_zero_rows():  # :80-90
    g = g_of(3, [(0, 1), (2, 1)])
    out = O.binary_reduce(g, O.named_config("u_copy_max_v"), u=np.array([[5], [-7], [2]]))
    assert out[:, 0].tolist() == [0, 5, 0]


def test_weighted_sum_eq2():  # :92-103
    g = g_of(2, [(0, 1)])
    out = O.binary_reduce(g, O.named_config("u_mul_e_add_v"), u=np.array([[2, 3], [0, 0]]),
                          e=np.array([[10, 10]]))
    assert out[1].tolist() == [20, 30]


def test_dot_and_add_to_edge():  # :105-127
    g = g_of(2, [(0, 1)])
    out = O.binary_reduce(g, O.named_config("u_dot_v_add_e"), u=np.array([[1, 2], [0, 0]]),
                          v=np.array([[0, 0], [3, 4]]))
    assert out.shape == (1, 1) and out[0, 0] == 11
    out = O.binary_reduce(g, O.named_config("u_add_v_copy_e"), u=np.array([[1], [0]]),
                          v=np.array([[0], [5]]))
    assert out[0, 0] == 6


def test_edge_max_duplicates():  # :129-137
    g = g_of(2, [(0, 1), (0, 1)])
    out = O.binary_reduce(g, O.named_config("e_copy_max_v"), e=np.array([[3], [7]]))
    assert out[1, 0] == 7


def test_validation_errors():  # :139-174
    g = g_of(2, [(0, 1)])
    cfg = O.named_config("u_copy_add_v")
    with pytest.raises(O.OracleError) as ex:  # wrong orientation
        O.binary_reduce(g, cfg, u=np.zeros((2, 4)), orientation=O.SRC_MAJOR)
    assert ex.value.status == O.SHAPE
    with pytest.raises(O.OracleError):  # missing operand
        O.binary_reduce(g, cfg)
    with pytest.raises(O.OracleError):  # row mismatch
        O.binary_reduce(g, cfg, u=np.zeros((3, 4)))
    with pytest.raises(O.OracleError):  # incompatible widths
        O.binary_reduce(g, O.named_config("u_add_v_add_v"), u=np.zeros((2, 4)), v=np.zeros((2, 3)))


def test_empty_graph_zero():  # :190-200
    g = O.Graph(4, np.array([], np.uint32), np.array([], np.uint32))
    for name in ("u_copy_add_v", "u_copy_max_v"):
        assert (O.binary_reduce(g, O.named_config(name), u=np.ones((4, 3))) == 0).all()


def test_degree_identity():  # :339-352
    n, src, dst = O.random_small_graph(190)
    g = O.Graph(n, src, dst)
    out = O.binary_reduce(g, O.named_config("u_copy_add_v"), u=np.ones((n, 1)))
    assert (out[:, 0] == np.bincount(dst, minlength=n)).all()


# --------------------------------------------------- test_oracle.cpp
def test_oracle_copy_last_canonical_winner():  # test_oracle.cpp:64-73
    g = g_of(3, [(2, 1), (0, 1)])
    out = O.oracle_aggregate(g, O.named_config("u_copy_copy_v"), u=np.array([[10], [0], [99]]))
    assert out[1, 0] == 99
    out = O.binary_reduce(g, O.named_config("u_copy_copy_v"), u=np.array([[10], [0], [99]]))
    assert out[1, 0] == 99


def test_oracle_refuses_large():  # test_oracle.cpp:75-83
    g = O.Graph(2, np.zeros(1000001, np.uint32), np.ones(1000001, np.uint32))
    with pytest.raises(O.OracleError):
        O.oracle_aggregate(g, O.named_config("u_copy_add_v"), u=np.zeros((2, 1)))


# ---------------------------------------------- test_generators.cpp
def test_er_p1_complete():  # test_generators.cpp:38-46
    src, dst = O.gen_er(4, 0, 1.0, 0)
    assert len(src) == 12 and (src != dst).all()


def test_sbm_disjoint():  # :48-58
    src, dst = O.gen_sbm(100, 2, 1.0, 0.0, 0)
    assert len(src) == 2 * 50 * 49 and ((src < 50) == (dst < 50)).all()


def test_rmat_count_and_range():  # :82-94
    src, dst = O.gen_rmat(1000, 5000, seed=3)
    assert len(src) == 5000 and (src < 1000).all() and (dst < 1000).all()


def test_random_features_range():  # :155-166
    f = O.random_features(200, 5, 7)
    assert (f >= -1).all() and (f < 1).all()
    assert (O.random_features(3, 2, 99) == O.random_features(3, 2, 99)).all()


def test_dot_equals_sum_of_mul():  # test_features.cpp:103-113
    g = g_of(2, [(0, 1)])
    for seed in range(20, 24):
        x = np.array([[O.LIB.or_unit_float_at(seed, i) for i in range(8)], [0] * 8], np.float32)
        y = np.array([[0] * 8, [O.LIB.or_unit_float_at(seed + 100, i) for i in range(8)]],
                     np.float32)
        d = O.binary_reduce(g, O.named_config("u_dot_v_add_e"), u=x, v=y)[0, 0]
        acc = np.float32(0)
        for i in range(8):
            acc = np.float32(acc + np.float32(x[0, i] * y[1, i]))
        assert d == acc


# -------------------------------------- fixtures from the reference
@pytest.mark.parametrize("seed", (101, 104, 107))
def test_restatement_matches_reference_fixtures(golden, seed):
    p = f"s{seed}_"
    n = int(golden[p + "n"][0])
    src, dst = golden[p + "src"], golden[p + "dst"]
    # generator restatement reproduces the reference's edges
    regen = O.random_small_graph(seed)
    assert regen[0] == n and (regen[1] == src).all() and (regen[2] == dst).all()
    for o in (0, 1):
        mine = O.build_csr(n, src, dst, o)
        for a, k in zip(mine, ("indptr", "indices", "eids")):
            assert (a == golden[p + f"csr{o}_{k}"]).all()
    g = O.Graph(n, src, dst)
    fu, fv, fe = golden[p + "fu"], golden[p + "fv"], golden[p + "fe"]
    assert (O.random_features(n, fu.shape[1], seed) == fu).all()
    for cname in O.APPLICATION_CONFIGS:
        cfg = O.named_config(cname)
        got = O.binary_reduce(g, cfg, fu, fv, fe)
        assert O.bit_equal(got, golden[p + "spmm_" + cname]), cname
        if cfg[4] != O.E:
            want = golden[p + "oracle_" + cname]
            assert O.bit_equal(O.oracle_aggregate(g, cfg, fu, fv, fe), want), cname
            # the reference's own acceptance criterion between the two
            if O.is_exact_reduce(cfg[3]):
                assert O.bit_equal(got, want)
            else:
                assert O.max_rel_error(got, want) <= 1e-5


def test_composed_ops_match_reference_fixtures(golden):
    n = int(golden["c_n"][0])
    g = O.Graph(n, golden["c_src"], golden["c_dst"])
    x, w, gy = golden["c_x"], golden["c_w"], golden["c_gy"]
    assert (O.normal_features(n, x.shape[1], 1) == x).all()
    assert (O.gcn_weights(n, g.src, g.dst) == w).all()
    assert O.bit_equal(O.binary_reduce(g, (O.U, O.E, O.MUL, O.SUM, O.V), u=x, e=w),
                       golden["c_gcn_fwd"])
    assert O.bit_equal(O.sum_backward(g, gy, w), golden["c_gcn_bwd"])
    assert O.bit_equal(O.edge_grad(g, x, gy), golden["c_grad_w"])
    assert O.bit_equal(O.mean(g, x), golden["c_mean"])
    val, arg_u, arg_e = O.copy_max_argmax(g, x)
    assert O.bit_equal(val, golden["c_max"])
    # argmax consistency: the winner's feature equals the max
    has = arg_u >= 0
    cols = np.nonzero(has)[1]
    assert (x[arg_u[has], cols] == val[has]).all()
    a = O.softmax_attention(n, g.dst, O.normal_features(g.m, 4, 2))
    assert (a == golden["c_att"]).all()
    assert O.bit_equal(O.multihead_u_mul_e_sum(g, x, a, 4), golden["c_mh_fwd"])


# -------------------------- direct comparison (container with the reference)
@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("seed", range(1, 21))
def test_restatement_matches_reference_library(seed):
    n, src, dst = O.random_small_graph(seed)
    g = O.Graph(n, src, dst)
    dim = 1 + O.splitmix64_at(seed, 2) % 17
    fu = O.random_features(n, dim, seed)
    fv = O.random_features(n, dim, seed + 1000)
    fe = O.random_features(g.m, dim, seed + 2000)
    for cname in O.APPLICATION_CONFIGS + ["u_copy_max_v", "u_copy_min_v", "u_copy_mul_v",
                                          "u_copy_copy_v", "u_sub_v_add_v", "u_div_e_max_v",
                                          "e_mul_u_min_v"]:
        cfg = O.named_config(cname)
        mine = O.binary_reduce(g, cfg, fu, fv, fe)
        for strategy in (O.SPMM, O.PULL):
            assert O.bit_equal(mine, O.ref_binary_reduce(g, cfg, fu, fv, fe, strategy=strategy))
        assert O.bit_equal(O.oracle_aggregate(g, cfg, fu, fv, fe),
                           O.ref_oracle_aggregate(g, cfg, fu, fv, fe))


@pytest.mark.parametrize("seed", (101, 107))
def test_fault_injection_fails_the_checks(golden, seed):
    # the checker must catch one corrupted element (the reference's
    # --inject-fault, tools/main.cpp:201-204): a single ulp for the bitwise
    # reducers, a 1e-3 relative change for the tolerance check
    p = f"s{seed}_"
    n = int(golden[p + "n"][0])
    g = O.Graph(n, golden[p + "src"], golden[p + "dst"])
    fu, fv, fe = golden[p + "fu"], golden[p + "fv"], golden[p + "fe"]
    for cname in ("u_mul_e_add_v", "e_copy_max_v"):
        cfg = O.named_config(cname)
        got = O.binary_reduce(g, cfg, fu, fv, fe)
        want = golden[p + "spmm_" + cname]
        assert O.bit_equal(got, want)
        i = int(np.argmax(np.abs(got).reshape(-1)))
        bad = got.reshape(-1).copy()
        bad[i] = np.nextafter(bad[i], np.float32(np.inf))
        assert not O.bit_equal(bad.reshape(got.shape), want), cname
        bad[i] = got.reshape(-1)[i] + np.float32(1e-3) * max(1.0, abs(float(got.reshape(-1)[i])))
        assert O.max_rel_error(bad.reshape(got.shape), want) > 1e-5, cname
