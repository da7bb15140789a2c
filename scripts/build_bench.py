"""Host vs device CSR build + transpose at config-3 scale (development aid)."""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2007_06354_b200 as P  # noqa: E402

n, m = 2_449_029, 61_859_140
src, dst = P.synth_rmat(n, m, 0.57, 0.19, 0.19, 0.05, 0)
src, dst = np.concatenate([src, dst]), np.concatenate([dst, src])
t0 = time.time()
h = P.build_csr(n, src, dst, P.DST_MAJOR)
t1 = time.time()
ht = P.transpose(n, n, *h)
t2 = time.time()
s_d = torch.from_numpy(src.view(np.int32)).cuda()
d_d = torch.from_numpy(dst.view(np.int32)).cuda()
for rep in range(2):
    torch.cuda.synchronize()
    a = time.time()
    d = P.build_csr_device(n, s_d, d_d)
    torch.cuda.synchronize()
    b = time.time()
    dt = P.transpose_device(n, n, *d)
    torch.cuda.synchronize()
    c = time.time()
same = all(np.array_equal(x, y.cpu().numpy().view(np.uint32)) for x, y in zip(h, d))
same_t = all(np.array_equal(x, y.cpu().numpy().view(np.uint32)) for x, y in zip(ht, dt))
print(json.dumps({"edges": len(src), "host_build_s": t1 - t0, "host_transpose_s": t2 - t1,
                  "host_threads": os.cpu_count(), "device_build_s": b - a,
                  "device_transpose_s": c - b, "identical": same and same_t}))
