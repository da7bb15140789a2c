"""Concurrent per-unit timeline of one aggregation pass (development aid).

Like trace_case.py, but with GSPMM_UNIT_TRACE_CONCURRENT=1 the long-row and
segment launches of a call run concurrently as in production; both traces
share the global timer, so this prints, per 100-us bin, how many segment
units (warps) and long-row units (CTAs) were active, and when each kernel
drained.  python scripts/trace_conc.py rmat256"""
import os
import sys
import tempfile

import numpy as np

path = os.path.join(tempfile.mkdtemp(), "trace.bin")
os.environ["GSPMM_UNIT_TRACE"] = path
os.environ["GSPMM_UNIT_TRACE_CONCURRENT"] = "1"
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import kbench  # noqa: E402
import torch  # noqa: E402

name = sys.argv[1]
kbench.time_pass = lambda fn, iters=0, warm=0: (fn(), fn(), torch.cuda.synchronize(), 1.0)[-1]
kbench.run(name)
raw = np.fromfile(path, dtype=np.uint64)
i = 0
launches = []
while i < len(raw):
    assert raw[i] == 0xC0FFEE
    n_units, n_long, mode = int(raw[i + 1]), int(raw[i + 2]), int(raw[i + 3])
    t = raw[i + 4: i + 4 + 4 * max(n_units, 1)].reshape(-1, 4)[:n_units].astype(np.int64)
    i += 4 + 4 * max(n_units, 1)
    launches.append((mode, t))
last = {}
for mode, t in launches:
    last[mode] = t
t0 = min(t[:, 0].min() for t in last.values())
for mode, t in sorted(last.items()):
    s, e = (t[:, 0] - t0) / 1e3, (t[:, 1] - t0) / 1e3
    sms = len(set((t[:, 2] >> 32).tolist()))
    print(f"mode {mode} ({'long' if mode else 'seg'}): units {len(t)} start {s.min():.0f} "
          f"end {e.max():.0f} us, SMs {sms}, edges {t[:, 3].sum()}")
end = max(((t[:, 1] - t0) / 1e3).max() for t in last.values())
bins = np.arange(0, end + 100, 100)
print("bin_us  seg_active  long_active  long_SMs")
for b0 in bins:
    row = [f"{b0:6.0f}"]
    for mode in (0, 1):
        if mode not in last:
            row.append("-")
            continue
        t = last[mode]
        s, e = (t[:, 0] - t0) / 1e3, (t[:, 1] - t0) / 1e3
        act = (s < b0 + 100) & (e > b0)
        row.append(f"{act.sum():6d}")
        if mode == 1:
            row.append(f"{len(set((t[act, 2] >> 32).tolist())):4d}")
    print("  ".join(row))
