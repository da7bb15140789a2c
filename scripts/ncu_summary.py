"""Key metrics of every launch in an .ncu-rep (ncu --set full), as text for
profiles/: duration, DRAM / L2 bytes and throughput, occupancy, issue and the
top warp-stall reasons.  Usage: ncu_summary.py <rep> [> profiles/x.txt]"""
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_bytes.sum",
        "lts__t_sector_hit_rate.pct", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__t_sector_hit_rate.pct",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__inst_executed.sum",
        "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
        "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
        "sm__cycles_elapsed.max"]
raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
for vals in rows[2:]:
    d = dict(zip(hdr, vals))
    u = dict(zip(hdr, units))
    print("==", d.get("Kernel Name"), "(launch id", d.get("ID"), ")")
    for k in KEYS:
        if k in d:
            print(f"  {k:62s} {d[k]:>16s} {u[k]}")
    stalls = sorted(((float(d[h] or 0), h) for h in hdr
                     if h.startswith("smsp__average_warps_issue_stalled_") and
                     h.endswith("_per_issue_active.ratio")), reverse=True)[:6]
    for v, h in stalls:
        print(f"  stall {h[len('smsp__average_warps_issue_stalled_'):-len('_per_issue_active.ratio')]:30s} "
              f"{v:8.3f} warps per issue")
