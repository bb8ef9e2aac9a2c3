"""ncu --metrics CSV of tools/ncu_kernels.py -> profiles/{plan_sweep,latent,route}_ncu_summary.json
(the per-launch figures bench.py's sub-leg rooflines read). Uses the LAST
launch of each kernel (the warm round).

    python tools/ncu_summarize.py gpurun_out/r2l_kernels.csv [tag]
"""
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
src = sys.argv[1]
tag = sys.argv[2] if len(sys.argv) > 2 else os.path.basename(src)
rows = [r for r in csv.reader(open(src)) if len(r) > 14 and r[0] != "ID"]
by = {}
for r in rows:
    kid, name, metric, unit, val = r[0], r[4], r[12], r[13], r[14]
    key = ("plan_sweep" if "plan_sweep_kernel" in name else
           "latent" if "latent_kernel" in name else "route" if "route_kernel" in name else None)
    if key is None:
        continue
    by.setdefault(key, {}).setdefault(int(kid), {})[metric] = (unit, val, r[7], r[8])


def num(unit, v):
    x = float(v.replace(",", ""))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "us": 1.0,
             "ms": 1e3, "usecond": 1.0, "nsecond": 1e-3, "msecond": 1e3}
    return x * scale.get(unit, 1.0)


for key, launches in by.items():
    kid = max(launches)
    m = launches[kid]
    out = {"source": f"ncu --metrics (tools/ncu_kernels.py, launch id {kid}, {tag})",
           "block": m["gpu__time_duration.sum"][2], "grid": m["gpu__time_duration.sum"][3],
           "duration_us_under_ncu": num(*m["gpu__time_duration.sum"][:2]),
           "warp_inst_per_launch": num(*m["smsp__inst_executed.sum"][:2]),
           "dram_bytes_read": num(*m["dram__bytes_read.sum"][:2]),
           "dram_bytes_write": num(*m["dram__bytes_write.sum"][:2]),
           "issue_active_pct": num(*m["smsp__issue_active.avg.pct_of_peak_sustained_active"][:2]),
           "warps_active_pct": num(*m["sm__warps_active.avg.pct_of_peak_sustained_active"][:2]),
           "sm_cycles_elapsed": num(*m["sm__cycles_elapsed.avg"][:2]),
           "sm_cycles_active": num(*m["sm__cycles_active.avg"][:2]),
           "sms": 148}
    out["dram_bytes_per_launch"] = out["dram_bytes_read"] + out["dram_bytes_write"]
    path = os.path.join(ROOT, "profiles", f"{key}_ncu_summary.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1)
    print(path, json.dumps(out))
