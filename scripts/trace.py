"""Summarise a GSPMM_UNIT_TRACE file (development aid)."""
import sys
import numpy as np

raw = np.fromfile(sys.argv[1], dtype=np.uint64)
i = 0
launch = 0
while i < len(raw):
    assert raw[i] == 0xC0FFEE, raw[i]
    n_units, n_long = int(raw[i + 1]), int(raw[i + 2])
    t = raw[i + 4: i + 4 + 4 * max(n_units, 1)].reshape(-1, 4)[:n_units]
    i += 4 + 4 * max(n_units, 1)
    launch += 1
    t0 = t[:, 0].min()
    start = (t[:, 0] - t0) / 1e3
    end = (t[:, 1] - t0) / 1e3
    dur = end - start
    edges = t[:, 3].astype(np.int64)
    kind = np.where(np.arange(n_units) < n_long, "long", "seg")
    print(f"launch {launch}: units {n_units} (long {n_long}) span {end.max():.1f} us, "
          f"sum-dur {dur.sum():.0f} us, warps {len(set(t[:, 2].tolist()))}")
    for k in ("long", "seg"):
        m = kind == k
        if m.any():
            rate = edges[m] / np.maximum(dur[m], 1e-3)
            print(f"  {k}: n={m.sum()} dur mean {dur[m].mean():.1f} max {dur[m].max():.1f} us; "
                  f"edges/us median {np.median(rate):.1f}; start max {start[m].max():.1f} us")
    top = np.argsort(-dur)[:8]
    for u in top:
        print(f"    unit {u:6d} {kind[u]:4s} edges {edges[u]:7d} start {start[u]:8.1f} dur {dur[u]:8.1f} us "
              f"rate {edges[u] / max(dur[u], 1e-3):7.1f} e/us sm {t[u, 2] >> 32}")
