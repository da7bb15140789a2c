"""Summarise the LGU lines of scripts/trace_long.py: kernel span, the units
on the critical path, per-unit rates by slice width."""
import collections
import re
import sys

U = []
W = {}
for line in open(sys.argv[1]):
    m = re.match(r"LGW (\d+) full (-?\d+) empty (-?\d+) idbar (-?\d+) ld (-?\d+) st (-?\d+) ar (-?\d+)", line)
    if m:
        W[int(m.group(1))] = tuple(int(v) / 1.965e3 for v in m.groups()[1:])  # us at 1.965 GHz
    m = re.match(r"LGU (\d+) row (\d+) c0 (\d+) cw (\d+) n (\d+) t0 (\d+) t1 (\d+) cta (\d+)", line)
    if m:
        U.append(tuple(int(v) for v in m.groups()))
t0 = min(u[5] for u in U)
t1 = max(u[6] for u in U)
print(f"{len(U)} units, span {(t1 - t0) / 1e3:.1f} us, {len(set(u[7] for u in U))} CTAs")
by = collections.defaultdict(list)
for u in U:
    by[u[3]].append(u)
for cw, us in sorted(by.items()):
    ns = sum(u[6] - u[5] for u in us)
    ed = sum(u[4] for u in us)
    print(f"cw {cw:4d}: {len(us):5d} units, {ed / 1e6:8.2f} M edges, {ns / ed:6.2f} ns/edge, "
          f"{ed * cw * 4 / ns:6.1f} GB/s per CTA, mean unit {ns / len(us) / 1e3:7.1f} us"
          + (f"; waits (us, mean): consumer on full {sum(W[u[0]][0] for u in us) / len(us):7.1f}, "
             f"producer on empty {sum(W[u[0]][1] for u in us) / len(us):7.1f}, "
             f"ids + barrier {sum(W[u[0]][2] for u in us) / len(us):7.1f}, load issue "
             f"{sum(W[u[0]][3] for u in us) / len(us):7.1f}, STS (data wait) "
             f"{sum(W[u[0]][4] for u in us) / len(us):7.1f}, arrive {sum(W[u[0]][5] for u in us) / len(us):7.1f}"
             if W else ""))
print("last units to finish:")
for u in sorted(U, key=lambda u: -u[6])[:8]:
    print(f"  unit {u[0]} row {u[1]} cw {u[3]} n {u[4]}: start {(u[5] - t0) / 1e3:.1f} us, "
          f"{(u[6] - u[5]) / 1e3:.1f} us, {(u[6] - u[5]) / u[4]:.2f} ns/edge, cta {u[7]}")
print("longest units:")
for u in sorted(U, key=lambda u: -(u[6] - u[5]))[:8]:
    print(f"  unit {u[0]} row {u[1]} cw {u[3]} n {u[4]}: start {(u[5] - t0) / 1e3:.1f} us, "
          f"{(u[6] - u[5]) / 1e3:.1f} us, {(u[6] - u[5]) / u[4]:.2f} ns/edge, cta {u[7]}")
busy = collections.defaultdict(int)
for u in U:
    busy[u[7]] += u[6] - u[5]
b = sorted(busy.values())
print(f"CTA busy time: min {b[0] / 1e3:.1f} median {b[len(b) // 2] / 1e3:.1f} max {b[-1] / 1e3:.1f} us")
