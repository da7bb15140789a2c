"""Micro-benchmark of the max backward (argmax scatter) at config-3 size:
the real cfg3 argmax (max forward on the symmetrised R-MAT graph) and a
uniform random argmax, CUDA-event timed.  Development tool."""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2007_06354_b200 as P  # noqa: E402

n, F = 2_449_029, 100
src, dst = P.synth_rmat(n, 61_859_140, 0.57, 0.19, 0.19, 0.05, 0)
src, dst = np.concatenate([src, dst]), np.concatenate([dst, src])
g = P.Graph(*P.build_csr(n, src, dst, P.DST_MAJOR), orientation=P.DST_MAJOR)
x = torch.from_numpy(P.synth_uniform(n, F, 1)).cuda()
gy = torch.from_numpy(P.synth_normal(n, F, 3)).cuda()
_, au, _ = P.binary_reduce(g, "u_copy_max_v", u=x, want_arg_other=True)
rnd = torch.randint(0, n, (n, F), dtype=torch.int32, device="cuda")
rnd[au < 0] = -1
out = torch.empty((n, F), device="cuda")
for name, arg in (("cfg3 argmax", au), ("uniform", rnd)):
    for _ in range(3):
        P.argmax_backward(arg, gy, n, out=out)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(10):
        P.argmax_backward(arg, gy, n, out=out)
    e.record()
    torch.cuda.synchronize()
    print(f"{name}: {s.elapsed_time(e) / 10:.3f} ms", flush=True)
