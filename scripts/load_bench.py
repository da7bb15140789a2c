"""CSR1 / FMAT1 loader timings at config-3 size (development tool): the
device loader (gspmm_graph_load_csr1: pinned ring, device narrowing and
validation) against the host reader followed by an upload, and the FMAT1
device loader against a host read + copy.  Files go to a temp directory."""
import json
import os
import sys
import tempfile
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2007_06354_b200 as P  # noqa: E402

n, F = 2_449_029, 100
src, dst = P.synth_rmat(n, 61_859_140, 0.57, 0.19, 0.19, 0.05, 0)
src, dst = np.concatenate([src, dst]), np.concatenate([dst, src])
dcsr = P.build_csr(n, src, dst, P.DST_MAJOR)
x = P.synth_uniform(n, F, 1)
d = tempfile.mkdtemp()
t0 = time.time()
P.save_csr(d + "/g.csr", P.DST_MAJOR, n, n, *dcsr)
P.save_feature_matrix(d + "/x.fmat", x)
res = {"edges": len(src), "csr1_bytes": os.path.getsize(d + "/g.csr"),
       "fmat1_bytes": os.path.getsize(d + "/x.fmat"), "write_s": round(time.time() - t0, 2)}
torch.cuda.init()
torch.zeros(1, device="cuda")
for rep in range(2):  # second repetition: page cache warm
    t0 = time.time()
    g = P.Graph.load(d + "/g.csr")
    torch.cuda.synchronize()
    res[f"device_loader_s_{rep}"] = round(time.time() - t0, 3)
    g.close()
    t0 = time.time()
    o, r, c, ip, ix, ei = P.load_csr(d + "/g.csr")
    t1 = time.time()
    g = P.Graph(ip, ix, ei, num_rows=r, num_cols=c, orientation=o)
    torch.cuda.synchronize()
    res[f"host_reader_s_{rep}"] = round(t1 - t0, 3)
    res[f"host_upload_s_{rep}"] = round(time.time() - t1, 3)
    g.close()
    t0 = time.time()
    xd = P.load_feature_matrix(d + "/x.fmat", device=0)
    torch.cuda.synchronize()
    res[f"fmat_device_loader_s_{rep}"] = round(time.time() - t0, 3)
    t0 = time.time()
    xh = torch.from_numpy(P.load_feature_matrix(d + "/x.fmat")).cuda()
    torch.cuda.synchronize()
    res[f"fmat_host_read_copy_s_{rep}"] = round(time.time() - t0, 3)
    assert torch.equal(xd, xh)
print(json.dumps(res))
for f in ("g.csr", "x.fmat"):
    os.remove(os.path.join(d, f))
