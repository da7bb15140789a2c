"""Summarise an `ncu --metrics ... --csv` launch list: one line per launch
(or, with --group, per kernel name) with duration, DRAM bytes, L2 hit rate."""
import collections
import csv
import sys


def load(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    launches = collections.OrderedDict()
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            key = (int(d["ID"]), d["Kernel Name"])
            launches.setdefault(key, {})[d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
    return launches


def main():
    path = sys.argv[1]
    skip = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    L = load(path)
    items = list(L.items())[skip:]
    tot_t = 0
    for (i, name), m in items:
        t = m.get("gpu__time_duration.sum", 0) / 1e3
        rd = m.get("dram__bytes_read.sum", 0) / 1e9
        wr = m.get("dram__bytes_write.sum", 0) / 1e9
        hit = m.get("lts__t_sector_hit_rate.pct", 0)
        l2 = m.get("lts__t_bytes.sum", 0) / 1e9
        tot_t += t
        short = name.split("(")[0][-60:]
        print(f"{i:4d} {short:60s} {t:9.1f} us  dram r {rd:6.3f} w {wr:6.3f} GB "
              f"({(rd + wr) / max(t, 1e-9) * 1e3:6.2f} TB/s)  L2 {l2:6.2f} GB hit {hit:5.1f}%")
    print(f"total {tot_t:.1f} us")


if __name__ == "__main__":
    main()
