"""Kernel micro-benchmark: one aggregation pass on synthetic graphs, CUDA-event
timed, algorithmic GB/s vs the measured HBM peak.  Development tool (not the
driver's bench): python scripts/kbench.py [--cases er128,rmat256,...]"""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2007_06354_b200 as P  # noqa: E402

PEAK = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
    os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0


PLAN = {}


def graph(kind, n, m, seed=0, loops=False, sym=False):
    if kind == "powerlaw":
        return P.synth_powerlaw(n, 90, 21000, seed)
    if kind in ("er", "star"):
        src, dst = P.synth_er(n, m, -1.0, seed)
    else:
        src, dst = P.synth_rmat(n, m, 0.57, 0.19, 0.19, 0.05, seed)
    if sym:
        src, dst = np.concatenate([src, dst]), np.concatenate([dst, src])
    if kind == "rmatcap":  # drop the in-edges of rows above 4096
        deg = np.bincount(dst, minlength=n)
        keep = deg[dst] <= 4096
        src, dst = src[keep], dst[keep]
    if kind == "star":  # uniform graph + one 66k in-edge hub at row 7
        hub = np.random.default_rng(0).integers(0, n, 66394).astype(np.uint32)
        src = np.concatenate([src, hub])
        dst = np.concatenate([dst, np.full(len(hub), 7, np.uint32)])
    if loops:
        ar = np.arange(n, dtype=np.uint32)
        src, dst = np.concatenate([src, ar]), np.concatenate([dst, ar])
    return src, dst


def time_pass(fn, iters=10, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters


CASES = {
    "er128": ("er", 100_000, 1_600_000, 128, False, False, "copy"),
    "er256": ("er", 1_000_000, 16_000_000, 256, False, False, "gcn"),
    "rmat256": ("rmat", 1_000_000, 16_000_000, 256, True, False, "gcn"),
    "rmatcap256": ("rmatcap", 1_000_000, 16_000_000, 256, True, False, "gcn"),
    "star256": ("star", 1_000_000, 16_000_000, 256, False, False, "gcn"),
    "rmat100sym": ("rmat", 2_449_029, 61_859_140, 100, False, True, "mean"),
    "rmat512h": ("rmat", 1_000_000, 32_000_000, 512, False, False, "heads"),
    "cfg3max": ("rmat", 2_449_029, 61_859_140, 100, False, True, "maxarg"),
    "cfg5mean": ("powerlaw", 232_965, 0, 602, False, False, "mean604"),
    "cfg2dot": ("rmat", 1_000_000, 16_000_000, 256, True, False, "dot"),
    "cfg4dot": ("rmat", 1_000_000, 32_000_000, 512, False, False, "dotheads"),
    "cfg4softmax": ("rmat", 1_000_000, 32_000_000, 8, False, False, "softmax"),
    # backward passes (src-major handle)
    "cfg2bwd": ("rmat", 1_000_000, 16_000_000, 256, True, False, "gcnbwd"),
    "cfg3meanbwd": ("rmat", 2_449_029, 61_859_140, 100, False, True, "meanbwd"),
    "cfg3maxbwd": ("rmat", 2_449_029, 61_859_140, 100, False, True, "maxbwd"),
    "cfg4bwdx": ("rmat", 1_000_000, 32_000_000, 512, False, False, "headsbwd"),
    "cfg5meanbwd": ("powerlaw", 232_965, 0, 602, False, False, "meanbwd604"),
    "cfg4softmaxbwd": ("rmat", 1_000_000, 32_000_000, 8, False, False, "softmaxbwd"),
}


def run(name):
    kind, n, m, F, loops, sym, op = CASES[name]
    t0 = time.time()
    src, dst = graph(kind, n, m, loops=loops, sym=sym)
    E = len(src)
    dcsr = P.build_csr(n, src, dst, P.DST_MAJOR)
    g = P.Graph(*dcsr, orientation=P.DST_MAJOR)
    deg = np.diff(dcsr[0].astype(np.int64))
    x = torch.randn(n, F, device="cuda")
    out = torch.empty(n, F, device="cuda")
    if op == "gcn":
        w = torch.from_numpy(P.synth_gcn_weights(n, src, dst)).cuda()
        wp = g.permute_edges(w)
        fn = lambda: P.binary_reduce(g, "u_mul_e_add_v", u=x, e=wp, out=out, e_order=P.EDGE_BY_POS)
        eb = E * 4
    elif op == "heads":
        a = torch.rand(E, 8, device="cuda")
        ap = g.permute_edges(a)
        fn = lambda: P.binary_reduce(g, "u_mul_e_add_v", u=x, e=ap, out=out, e_order=P.EDGE_BY_POS,
                                     heads=8)
        eb = E * 32
    elif op == "mean":
        fn = lambda: P.binary_reduce(g, (P.U, P.NONE, P.COPY, P.MEAN, P.V), u=x, out=out)
        eb = 0
    elif op == "mean604":  # F=602 rows padded to a 16-byte leading dimension
        xp = torch.zeros(n, 604, device="cuda")
        xp[:, :F] = x
        op_ = torch.empty(n, 604, device="cuda")
        fn = lambda: P.binary_reduce(g, (P.U, P.NONE, P.COPY, P.MEAN, P.V), u=xp[:, :F],
                                     out=op_[:, :F])
        eb = 0
    elif op == "maxarg":
        fn = lambda: P.binary_reduce(g, "u_copy_max_v", u=x, out=out, want_arg_other=True)
        eb = 0
    elif op in ("dot", "dotheads"):
        # edge grads: grad_e[e, h] = dot(x[u_e, h], y[v_e, h]) (u_dot_v_copy_e)
        y = torch.randn(n, F, device="cuda")
        heads = 8 if op == "dotheads" else 1
        oe = torch.empty(E, heads, device="cuda")
        fn = lambda: P.binary_reduce(g, (P.U, P.V, P.DOT, P.COPY_LAST, P.E), u=x, v=y, out=oe,
                                     heads=heads)
        eb = E * heads * 4 - n * F * 4  # writes E x heads, reads y rows per edge (cached)
    elif op in ("softmax", "softmaxbwd"):
        # GAT attention over 8 heads: logits in CSR order, E x 8
        lg = torch.randn(E, F, device="cuda")
        a = P.edge_softmax(g, lg, e_order=P.EDGE_BY_POS)
        ga = torch.randn(E, F, device="cuda")
        if op == "softmax":
            fn = lambda: P.edge_softmax(g, lg, out=a, e_order=P.EDGE_BY_POS)
            eb = 0
        else:
            gl = torch.empty_like(a)
            fn = lambda: P.edge_softmax_backward(g, a, ga, out=gl, e_order=P.EDGE_BY_POS)
            eb = E * F * 4  # reads a and grad_a
    elif op in ("gcnbwd", "meanbwd", "headsbwd", "meanbwd604"):
        # grad_u = sum over out-edges (u -> v) of grad_out[v] (x a weight), on
        # the transposed CSR
        scsr = P.transpose(n, n, *dcsr)
        gs = P.Graph(*scsr, orientation=P.SRC_MAJOR)
        del g
        cfg = (P.V, P.E, P.MUL, P.SUM, P.U)
        if op == "gcnbwd":
            w = torch.from_numpy(P.synth_gcn_weights(n, src, dst)).cuda()
            wp = gs.permute_edges(w)
            fn = lambda: P.binary_reduce(gs, cfg, v=x, e=wp, out=out, e_order=P.EDGE_BY_POS)
            eb = E * 4
        elif op == "headsbwd":
            a = torch.rand(E, 8, device="cuda")
            ap = gs.permute_edges(a)
            fn = lambda: P.binary_reduce(gs, cfg, v=x, e=ap, out=out, e_order=P.EDGE_BY_POS,
                                         heads=8)
            eb = E * 32
        else:
            inv = torch.from_numpy(np.where(deg > 0, 1.0 / np.maximum(deg, 1), 0).astype(np.float32)).cuda()
            cfgc = (P.V, P.NONE, P.COPY, P.SUM, P.U)
            if op == "meanbwd":
                fn = lambda: P.binary_reduce(gs, cfgc, v=x, out=out, other_scale=inv)
            else:
                xp = torch.zeros(n, 604, device="cuda")
                xp[:, :F] = x
                op_ = torch.empty(n, 604, device="cuda")
                fn = lambda: P.binary_reduce(gs, cfgc, v=xp[:, :F], out=op_[:, :F], other_scale=inv)
            eb = E * 4
        g = gs
    elif op == "maxbwd":
        _, au, _ = P.binary_reduce(g, "u_copy_max_v", u=x, want_arg_other=True)
        gy = torch.randn(n, F, device="cuda")
        fn = lambda: P.argmax_backward(au, gy, n)
        eb = 0
    else:
        fn = lambda: P.binary_reduce(g, "u_copy_add_v", u=x, out=out)
        eb = 0
    if PLAN:
        g.set_plan(**PLAN)
    ms = time_pass(fn)
    byts = E * F * 4 + (n + 1) * 4 + E * 4 + eb + n * F * 4
    if op == "maxbwd":  # read arg + grad_out, write grad (scatter): N x F each
        byts = n * F * 4 * 3
    if op in ("softmax", "softmaxbwd"):  # read logits (a, grad_a) once, write once; indptr
        byts = E * F * 4 * 2 + eb + (n + 1) * 4
    gbs = byts / ms / 1e6
    res = dict(case=name, E=E, F=F, ms=round(ms, 4), gbs=round(gbs, 1), frac=round(gbs / PEAK, 3),
               max_deg=int(deg.max()), long_rows=g.num_long_rows, plan=PLAN,
               setup_s=round(time.time() - t0, 1))
    print(json.dumps(res), flush=True)
    return res


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--cases", default="er128,er256,rmat256")
    ap.add_argument("--plans", default="", help="plan options k=v ..., several plans separated by /")
    args = ap.parse_args()
    for plan in args.plans.split("/"):
        PLAN = {k: int(v) for k, v in (t.split("=") for t in plan.split() if t)}
        for c in args.cases.split(","):
            run(c)
