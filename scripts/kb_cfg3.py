"""Config-3 forward / backward passes on their own (development tool): the
max+argmax and mean forward passes, the mean backward and the max backward,
10 timed repetitions each after 3 warm-ups, CUDA events.  Arguments: a
library path to load instead of the in-tree one (variant sweeps, or '-'),
then plan options as k=v (gspmm_graph_set_plan) -- several plans separated
by '/' are timed one after the other."""
import json
import os
import shutil
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
if len(sys.argv) > 1 and sys.argv[1] != "-":  # variant library, copied in before import
    shutil.copy(sys.argv[1], os.path.join(ROOT, "paper_2007_06354_b200", "_lib",
                                          "libgspmm_b200.so"))
import torch  # noqa: E402

import paper_2007_06354_b200 as P  # noqa: E402

n, F = 2_449_029, 100
src, dst = P.synth_rmat(n, 61_859_140, 0.57, 0.19, 0.19, 0.05, 0)
src, dst = np.concatenate([src, dst]), np.concatenate([dst, src])
dcsr = P.build_csr(n, src, dst, P.DST_MAJOR)
scsr = P.transpose(n, n, *dcsr)
deg = np.diff(dcsr[0].astype(np.int64))
inv = np.zeros(n, np.float32)
inv[deg > 0] = np.float32(1) / deg[deg > 0].astype(np.float32)
gd = P.Graph(*dcsr, orientation=P.DST_MAJOR)
gs = P.Graph(*scsr, orientation=P.SRC_MAJOR)
x = torch.from_numpy(P.synth_uniform(n, F, 1)).cuda()
gy = torch.from_numpy(P.synth_normal(n, F, 3)).cuda()
invd = torch.from_numpy(inv).cuda()
mx = torch.empty((n, F), device="cuda")
au = torch.empty((n, F), dtype=torch.int32, device="cuda")
mean = torch.empty((n, F), device="cuda")
gxm = torch.empty((n, F), device="cuda")
gmax = torch.empty((n, F), device="cuda")
passes = {
    "max+argmax": lambda: P.binary_reduce(gd, (P.U, P.NONE, P.COPY, P.MAX, P.V), u=x, out=mx,
                                          arg_other_out=au),
    "mean": lambda: P.binary_reduce(gd, (P.U, P.NONE, P.COPY, P.MEAN, P.V), u=x, out=mean),
    "max+argmax+mean (one gather)": lambda: P.binary_reduce(
        gd, (P.U, P.NONE, P.COPY, P.MAX, P.V), u=x, out=mx, arg_other_out=au, out2=mean,
        reduce2=P.MEAN),
    "mean_bwd": lambda: P.binary_reduce(gs, (P.V, P.NONE, P.COPY, P.SUM, P.U), v=gy, out=gxm,
                                        other_scale=invd),
    "max_bwd": lambda: P.argmax_backward(au, gy, n, out=gmax),
}
plans = " ".join(sys.argv[2:]).split("/") if len(sys.argv) > 2 else [""]
for plan in plans:
    kw = {k: int(v) for k, v in (t.split("=") for t in plan.split() if t)}
    for h in (gd, gs):
        h.set_plan(**kw)
    res = {"lib": sys.argv[1] if len(sys.argv) > 1 else "in-tree", "plan": kw}
    for name, fn in passes.items():
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(10):
            fn()
        b.record()
        torch.cuda.synchronize()
        res[name] = round(a.elapsed_time(b) / 10, 4)
    print(json.dumps(res), flush=True)
