"""profiles/traffic_cfg3.json from an ncu metrics launch list of `bench.py
--steps 1` (scripts/gpu/*.sh: --metrics ...dram__bytes_read.sum,
dram__bytes_write.sum...): DRAM bytes of the LAST step's kernels summed per
pass of the cfg3 step.  Usage: traffic_from_ncu.py <csv> <source label>"""
import json
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from ncu_metrics import load  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PASSES = ["fwd copy_u+max+argmax and copy_u+mean (one gather)", "bwd mean (grad_x)",
          "bwd max (argmax scatter)"]


def pass_of(name, state):
    if "k_argmax_scatter" in name or "k_round_f64" in name:
        return 2
    if "k_scale_rows" in name:
        state["bwd"] = True
        return 1
    return 1 if state.get("bwd") else 0


def main():
    L = list(load(sys.argv[1]).items())
    # the last step = the launches after the last k_round_f64 but one
    ends = [i for i, ((_, n), _) in enumerate(L) if "k_round_f64" in n]
    first = ends[-2] + 1 if len(ends) > 1 else 0
    state, out, kern = {}, {p: 0.0 for p in PASSES}, []
    for (_, name), m in L[first:]:
        k = pass_of(name, state)
        b = m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0)
        out[PASSES[k]] += b
        kern.append({"kernel": name.split("(")[0], "pass": k, "dram_bytes": b,
                     "us": m.get("gpu__time_duration.sum", 0) / 1e3,
                     "l2_bytes": m.get("lts__t_bytes.sum", 0)})
    head = subprocess.run(["git", "rev-parse", "--short", "HEAD"], cwd=ROOT, capture_output=True,
                          text=True).stdout.strip()
    json.dump({"source": sys.argv[2] if len(sys.argv) > 2 else sys.argv[1], "head": head,
               "config": "cfg3", "passes": out, "kernels": kern},
              open(os.path.join(ROOT, "profiles", "traffic_cfg3.json"), "w"), indent=1)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
