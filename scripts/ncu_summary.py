"""Summarise ncu --set full reports of the bench's kernels into profiles/
(development tool, run in the container: ncu -i reads the .ncu-rep files).

python scripts/ncu_summary.py <round-tag> fwd:<gather.ncu-rep> fwd:<long.ncu-rep> \
    bwd:<gather.ncu-rep> bwd:<long.ncu-rep>
writes profiles/<tag>_ncu_full.txt and profiles/traffic.json (per pass =
k_gather + k_long_ws of that pass, dram read + write bytes per launch)."""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
METRICS = ["dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
           "launch__block_size", "launch__grid_size", "launch__registers_per_thread",
           "lts__t_sector_hit_rate.pct", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
           "sm__warps_active.avg.pct_of_peak_sustained_active",
           "dram__throughput.avg.pct_of_peak_sustained_elapsed",
           "smsp__issue_active.avg.pct_of_peak_sustained_active"]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return [dict(zip(rows[0], zip(rows[1], r))) for r in rows[2:]]


def main():
    tag, reps = sys.argv[1], sys.argv[2:]
    lines = [f"# {tag} ncu --set full summaries (one launch each, bench.py cfg2 forward / "
             f"backward pass)"]
    per_pass = {"fwd": {}, "bwd": {}}
    for spec in reps:
        pas, rep = spec.split(":", 1) if ":" in spec else ("fwd", spec)
        for d in raw(rep):
            name = d["Kernel Name"][1]
            short = "k_long_ws" if "k_long_ws" in name else "k_long" if "k_long" in name else \
                "k_gather" if "k_gather" in name else name[:30]
            lines.append(f"## {pas} {short}")
            lines.append(f"  Kernel Name = {name}")
            byt = 0.0
            for m in METRICS:
                if m in d:
                    unit, val = d[m]
                    lines.append(f"  {m} = {val} {unit}")
                    if m.startswith("dram__bytes_"):
                        byt += float(val.replace(",", "")) * SCALE.get(unit, 1)
            per_pass[pas][short] = byt
    open(os.path.join(ROOT, "profiles", f"{tag}_ncu_full.txt"), "w").write("\n".join(lines) + "\n")
    json.dump({"fwd": sum(per_pass["fwd"].values()) or None,
               "bwd": sum(per_pass["bwd"].values()) or None, "per_kernel": per_pass,
               "note": f"dram__bytes_read.sum + dram__bytes_write.sum per launch, ncu --set full, "
                       f"cfg2 pass = k_gather + k_long_ws of that pass ({tag})"},
              open(os.path.join(ROOT, "profiles", "traffic.json"), "w"), indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main()
