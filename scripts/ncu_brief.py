"""Key ncu metrics + top stall reasons of one .ncu-rep (development aid):
python scripts/ncu_brief.py <report.ncu-rep>"""
import csv
import io
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True,
                     text=True, check=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[0]
for r in rows[2:]:
    v = dict(zip(h, r))
    print("==", v.get("Kernel Name", "")[:90])
    for w in ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
              "lts__t_sector_hit_rate.pct", "smsp__issue_active.avg.pct_of_peak_sustained_active",
              "sm__warps_active.avg.pct_of_peak_sustained_active",
              "l1tex__throughput.avg.pct_of_peak_sustained_active",
              "lts__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum",
              "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "launch__registers_per_thread",
              "launch__occupancy_limit_shared_mem", "launch__occupancy_limit_registers"]:
        if w in v:
            print(f"  {w} = {v[w]} {rows[1][h.index(w)]}")
    st = []
    for k, x in v.items():
        if k.startswith("smsp__pcsamp_warps_issue_stalled") and not k.endswith("not_issued"):
            try:
                st.append((float(x), k.replace("smsp__pcsamp_warps_issue_stalled_", "")))
            except ValueError:
                pass
    tot = sum(a for a, _ in st) or 1
    print("  stalls:", ", ".join(f"{k} {a / tot:.0%}" for a, k in sorted(st, reverse=True)[:8]))
