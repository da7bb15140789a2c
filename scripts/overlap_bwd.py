"""Config-3 step with the two backward passes (independent of each other) on
two streams against the serial step (development tool, r04g).  Setup as in
scripts/kb_cfg3.py: the
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

fwd, mbwd, xbwd = passes["max+argmax+mean (one gather)"], passes["mean_bwd"], passes["max_bwd"]
s1 = torch.cuda.Stream()
s2 = torch.cuda.Stream()


def serial():
    fwd(); mbwd(); xbwd()


def overlap(order):
    # forward on the current stream; then the two backward passes on two streams
    cur = torch.cuda.current_stream()
    fwd()
    ev = torch.cuda.Event(); ev.record(cur)
    first, second = (s1, s2)
    first.wait_event(ev); second.wait_event(ev)
    a, b = (mbwd, xbwd) if order == 0 else (xbwd, mbwd)
    with torch.cuda.stream(first):
        a()
    with torch.cuda.stream(second):
        b()
    cur.wait_stream(first); cur.wait_stream(second)


def bwd_under_fwd():
    # the mean backward does not depend on the forward at all: run it beside the forward
    cur = torch.cuda.current_stream()
    ev = torch.cuda.Event(); ev.record(cur)
    s1.wait_event(ev)
    with torch.cuda.stream(s1):
        mbwd()
    fwd()
    xbwd()
    cur.wait_stream(s1)


def fwd_then_xbwd_beside_mbwd_late():
    # max backward launched AFTER the mean backward's kernels are queued (other stream)
    cur = torch.cuda.current_stream()
    fwd()
    ev = torch.cuda.Event(); ev.record(cur)
    s1.wait_event(ev)
    mbwd()
    with torch.cuda.stream(s1):
        xbwd()
    cur.wait_stream(s1)


res = {}
for name, fn in (("serial", serial), ("overlap mean_bwd first", lambda: overlap(0)),
                 ("overlap max_bwd first", lambda: overlap(1)),
                 ("mean_bwd beside forward", bwd_under_fwd),
                 ("max_bwd on side stream after mean_bwd queued", fwd_then_xbwd_beside_mbwd_late),
                 ("serial again", serial)):
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
