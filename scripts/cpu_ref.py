"""The reference CPU path timed beside the GPU kernels, per configuration
shape ("shown next to the reference CPU path timed on the same
box's host cores").  For each kbench case: the unmodified reference library
(oracle/_ref, binary_reduce RowParallelSpmm with every host thread, its own
steady_clock around each call) on inputs of the same shape, composed as
SURVEY 8a a17 specifies where the reference has no single call (mean =
copy-sum then a division; multi-head = one call per head on copied head
slices), then the GPU pass of the same case (scripts/kbench.py).
python scripts/cpu_ref.py --cases er128,rmat256,...  (one JSON line each)"""
import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import kbench  # noqa: E402
from oracle import oracle as O  # noqa: E402

P = kbench.P
R = O.REF


def feats(rows, dim, seed):
    return np.random.default_rng(seed).standard_normal((rows, dim), dtype=np.float32)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cases", default="er128,rmat256,rmat100sym,cfg3max,rmat512h,cfg5mean")
    ap.add_argument("--iters", type=int, default=1)
    ap.add_argument("--no-gpu", action="store_true")
    args = ap.parse_args()
    if R is None:
        print(json.dumps({"unavailable": "oracle/_ref/libgspmm_ref.so not built"}))
        return
    threads = os.cpu_count() or 1
    for name in args.cases.split(","):
        kind, n, m, F, loops, sym, op = kbench.CASES[name]
        src, dst = kbench.graph(kind, n, m, loops=loops, sym=sym)
        E = len(src)
        t0 = time.time()
        views = R.ref_views_create(n, E, src.ctypes.data, dst.ctypes.data)
        setup = time.time() - t0
        keep = []

        def fm(a):
            a = np.ascontiguousarray(a, np.float32)
            keep.append(a)
            return R.ref_feat_create(a.shape[0], a.shape[1], a.ctypes.data)

        deg = np.bincount(dst, minlength=n)
        calls = []  # (lhs, rhs, op, red, out, u, v, e)
        extra = 0.0  # composition work outside the reference calls, timed here
        if op in ("copy", "mean", "mean604", "maxarg"):
            fx = fm(feats(n, F, 1))
            red = O.MAX if op == "maxarg" else O.SUM
            calls.append((O.U, O.NONE, O.COPY, red, O.V, fx, None, None))
        elif op in ("gcn", "gcnbwd", "meanbwd", "meanbwd604"):
            fx = fm(feats(n, F, 1))
            if op in ("meanbwd", "meanbwd604"):  # e = 1 / deg_in(dst(e))
                w = np.where(deg[dst] > 0, 1.0 / np.maximum(deg[dst], 1), 0).astype(np.float32)
            else:
                w = P.synth_gcn_weights(n, src, dst)
            fw = fm(w.reshape(-1, 1))
            if op == "gcn":
                calls.append((O.U, O.E, O.MUL, O.SUM, O.V, fx, None, fw))
            else:
                calls.append((O.V, O.E, O.MUL, O.SUM, O.U, None, fx, fw))
        elif op in ("heads", "headsbwd"):
            x = feats(n, F, 1)
            a = np.random.default_rng(2).random((E, 8), dtype=np.float32)
            t1 = time.time()
            xs = [np.ascontiguousarray(x[:, 64 * h:64 * h + 64]) for h in range(8)]
            as_ = [np.ascontiguousarray(a[:, h:h + 1]) for h in range(8)]
            extra += time.time() - t1
            for h in range(8):
                if op == "heads":
                    calls.append((O.U, O.E, O.MUL, O.SUM, O.V, fm(xs[h]), None, fm(as_[h])))
                else:
                    calls.append((O.V, O.E, O.MUL, O.SUM, O.U, None, fm(xs[h]), fm(as_[h])))
        elif op in ("dot", "dotheads"):
            x, y = feats(n, F, 1), feats(n, F, 2)
            heads = 8 if op == "dotheads" else 1
            D = F // heads
            for h in range(heads):
                calls.append((O.U, O.V, O.DOT, O.LAST, O.E,
                              fm(x[:, D * h:D * h + D]), fm(y[:, D * h:D * h + D]), None))
        else:
            print(json.dumps({"case": name, "skipped": "no reference composition"}), flush=True)
            R.ref_views_free(views)
            continue

        def run_all():
            tot = 0.0
            for (lhs, rhs, bop, red, out, fu, fv, fe) in calls:
                t = R.ref_run(views, O.SPMM, lhs, rhs, bop, red, out, fu, fv, fe, threads, None)
                if t < 0:
                    raise RuntimeError(f"reference failed on {name}")
                tot += t
            return tot

        run_all()  # warm-up
        ts = [run_all() for _ in range(args.iters)]
        ref_s = min(ts) + extra
        if op in ("mean", "mean604"):  # the division by the degree (a17.1)
            y = np.empty((n, F), np.float32)
            t1 = time.time()
            np.divide(y, np.maximum(deg, 1)[:, None].astype(np.float32), out=y)
            ref_s += time.time() - t1
        for (_, _, _, _, _, fu, fv, fe) in calls:
            for f in (fu, fv, fe):
                if f:
                    R.ref_feat_free(f)
        R.ref_views_free(views)
        res = {"case": name, "E": E, "F": F, "ref_ms": round(ref_s * 1e3, 1), "threads": threads,
               "ref_calls": len(calls), "ref_views_s": round(setup, 1)}
        if not args.no_gpu:
            g = kbench.run(name)
            res["gpu_ms"] = g["ms"]
            res["speedup"] = round(ref_s * 1e3 / g["ms"], 1)
        print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
