"""Per-unit timing of one aggregation pass of a kbench case (development aid).

GSPMM_UNIT_TRACE makes every planned launch append (start, end, sm, edges)
per work unit; this runs the case once (after one untraced warm-up in a
separate process is not possible: the trace switch is read once, so the
first pass is traced and the second is reported) and summarises the long-row
units by slice class.  python scripts/trace_case.py cfg5mean"""
import os
import sys
import tempfile

import numpy as np

path = os.path.join(tempfile.mkdtemp(), "trace.bin")
os.environ["GSPMM_UNIT_TRACE"] = path
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
    launches.append((mode, n_units, n_long, t))
# the second pass: the last launch of each mode
for mode in (1, 0):
    ls = [x for x in launches if x[0] == mode]
    if not ls:
        continue
    _, n_units, n_long, t = ls[-1]
    t0 = t[:, 0].min()
    start, end = (t[:, 0] - t0) / 1e3, (t[:, 1] - t0) / 1e3
    dur = end - start
    edges = t[:, 3]
    sms = t[:, 2] >> 32
    print(f"mode {mode}: units {n_units} span {end.max():.1f} us busy-sum {dur.sum():.0f} us "
          f"SMs {len(set(sms.tolist()))}")
    rate = edges / np.maximum(dur, 1e-3)
    q = np.quantile(end, [0.5, 0.9, 0.99, 1.0])
    print(f"  unit end quantiles (us) 50/90/99/100: {np.round(q, 1)}")
    if mode == 1:
        # classes by edges (long-row units are listed heaviest first)
        for lo, hi in ((0, 4096), (4096, 8192), (8192, 16384), (16384, 1 << 40)):
            m = (edges >= lo) & (edges < hi)
            if m.any():
                print(f"  rows {lo:>6}-{hi if hi < 1 << 40 else 'inf':>6}: units {m.sum():6d} "
                      f"edges/us median {np.median(rate[m]):7.1f} p10 {np.quantile(rate[m], .1):7.1f} "
                      f"dur median {np.median(dur[m]):8.1f} us")
    else:
        print(f"  seg edges/us median {np.median(rate):.1f}, dur median {np.median(dur):.1f} us")
