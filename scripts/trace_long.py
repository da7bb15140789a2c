"""Per-unit timeline of the long-row kernel on config 3 (development tool):
loads a library built with -DLG_TRACE=1 (argv[1]), runs ONE mean-backward-
shaped pass (copy + sum over the src-major graph) and ONE fused max + argmax
+ mean pass, and summarises the LGU lines the kernel prints."""
import os
import shutil
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
if len(sys.argv) > 1 and sys.argv[1] != "-":
    shutil.copy(sys.argv[1], os.path.join(ROOT, "paper_2007_06354_b200", "_lib", "libgspmm_b200.so"))
import torch  # noqa: E402

import paper_2007_06354_b200 as P  # noqa: E402

n, F = 2_449_029, 100
src, dst = P.synth_rmat(n, 61_859_140, 0.57, 0.19, 0.19, 0.05, 0)
src, dst = np.concatenate([src, dst]), np.concatenate([dst, src])
dcsr = P.build_csr(n, src, dst, P.DST_MAJOR)
gd = P.Graph(*dcsr, orientation=P.DST_MAJOR)
x = torch.from_numpy(P.synth_uniform(n, F, 1)).cuda()
mean = torch.empty((n, F), device="cuda")
mx = torch.empty((n, F), device="cuda")
au = torch.empty((n, F), dtype=torch.int32, device="cuda")
which = sys.argv[2] if len(sys.argv) > 2 else "mean"
torch.cuda.synchronize()
print("TRACE BEGIN", which, flush=True)
if which == "mean":
    P.binary_reduce(gd, (P.U, P.NONE, P.COPY, P.MEAN, P.V), u=x, out=mean)
else:
    P.binary_reduce(gd, (P.U, P.NONE, P.COPY, P.MAX, P.V), u=x, out=mx, arg_other_out=au, out2=mean,
                    reduce2=P.MEAN)
torch.cuda.synchronize()
print("TRACE END", flush=True)
