"""Generates tests/golden/*.npz from the UNMODIFIED reference library.

Run in the container that has /root/reference (it needs oracle/_ref, built by
`make -C oracle`).  The fixtures pin the C restatement in oracle/ and the GPU
path to the reference's own outputs; they are committed so the tests need no
reference checkout at run time.

  python tests/golden/make_golden.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "..", ".."))
from oracle import oracle as O  # noqa: E402

assert O.ref_available(), "oracle/_ref/libgspmm_ref.so missing: run make -C oracle"

KIND = {0: "er", 1: "rmat", 2: "sbm"}


def small_graph_via_ref(seed):
    """test_util.hpp:30-61 random_small_graph, drawn with the reference's own
    generate()."""
    pick = O.splitmix64_at(seed, 9000)
    n = 8 + O.splitmix64_at(seed, 9001) % 193
    degree = 1.0 + float(O.splitmix64_at(seed, 9002) % 10)
    kind = pick % 3
    if kind == 0:
        src, dst = O.ref_generate(0, n, 0, min(1.0, degree / (n - 1.0)), seed=seed)
    elif kind == 1:
        src, dst = O.ref_generate(1, n, min(2000, int(degree * n)), a=0.40, b=0.25, c=0.25,
                                  d=0.10, seed=seed)
    else:
        blocks = 1 + int(O.splitmix64_at(seed, 9004) % 4)
        p_in = min(1.0, degree * blocks / float(n))
        src, dst = O.ref_generate(2, n, 0, blocks=blocks, p_in=p_in, p_out=p_in / 20.0,
                                  seed=seed)
    return int(n), src, dst


def app_configs():
    out = {}
    for seed in (101, 104, 107):
        n, src, dst = small_graph_via_ref(seed)
        g = O.Graph(n, src, dst)
        dim = 1 + O.splitmix64_at(seed, 1) % 17
        fu = O.ref_random_features(n, dim, seed)
        fv = O.ref_random_features(n, dim, seed + 1)
        fe = O.ref_random_features(g.m, dim, seed + 2)
        p = f"s{seed}_"
        out[p + "n"] = np.array([n])
        out[p + "src"], out[p + "dst"] = src, dst
        for o, name in ((0, "src"), (1, "dst")):
            ip, ix, ei = O.ref_build_csr(n, src, dst, o)
            out[p + f"csr{o}_indptr"], out[p + f"csr{o}_indices"], out[p + f"csr{o}_eids"] = ip, ix, ei
        out[p + "fu"], out[p + "fv"], out[p + "fe"] = fu, fv, fe
        for cname in O.APPLICATION_CONFIGS:
            cfg = O.named_config(cname)
            out[p + "spmm_" + cname] = O.ref_binary_reduce(g, cfg, fu, fv, fe)
            if cfg[4] != O.E:
                out[p + "oracle_" + cname] = O.ref_oracle_aggregate(g, cfg, fu, fv, fe)
    return out


def composed():
    """a17 ops composed from reference calls on one RMAT graph."""
    out = {}
    n = 300
    src, dst = O.ref_generate(1, n, 4000, a=0.57, b=0.19, c=0.19, d=0.05, seed=5)
    src, dst = O.add_self_loops(n, src, dst)
    g = O.Graph(n, src, dst)
    x = O.normal_features(n, 24, 1)
    w = O.gcn_weights(n, src, dst)
    gy = O.normal_features(n, 24, 3)
    out["c_n"], out["c_src"], out["c_dst"] = np.array([n]), src, dst
    out["c_x"], out["c_w"], out["c_gy"] = x, w, gy
    out["c_gcn_fwd"] = O.ref_binary_reduce(g, (O.U, O.E, O.MUL, O.SUM, O.V), u=x, e=w)
    out["c_gcn_bwd"] = O.ref_binary_reduce(g, (O.V, O.E, O.MUL, O.SUM, O.U), v=gy, e=w)
    out["c_grad_w"] = O.ref_binary_reduce(g, (O.U, O.V, O.DOT, O.LAST, O.E), u=x, v=gy)
    deg = O.in_degree(g)
    s = O.ref_binary_reduce(g, (O.U, O.NONE, O.COPY, O.SUM, O.V), u=x)
    mean = np.where(deg[:, None] > 0, s / np.maximum(deg, 1).astype(np.float32)[:, None], 0)
    out["c_mean"] = mean.astype(np.float32)
    out["c_max"] = O.ref_binary_reduce(g, (O.U, O.NONE, O.COPY, O.MAX, O.V), u=x)
    # multi-head: 4 heads x 6 columns, one reference call per head
    heads = 4
    logits = O.normal_features(g.m, heads, 2)
    a = O.softmax_attention(n, dst, logits)
    out["c_att"] = a
    mh = np.empty_like(x)
    for h in range(heads):
        xh = np.ascontiguousarray(x[:, h * 6:(h + 1) * 6])
        mh[:, h * 6:(h + 1) * 6] = O.ref_binary_reduce(g, (O.U, O.E, O.MUL, O.SUM, O.V), u=xh,
                                                       e=np.ascontiguousarray(a[:, h:h + 1]))
    out["c_mh_fwd"] = mh
    return out


if __name__ == "__main__":
    data = {}
    data.update(app_configs())
    data.update(composed())
    path = os.path.join(HERE, "reference_outputs.npz")
    np.savez_compressed(path, **data)
    print(path, os.path.getsize(path), "bytes,", len(data), "arrays")
