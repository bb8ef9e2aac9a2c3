"""Key figures of an `ncu --set full` capture (first kernel): duration, clock,
issue/IPC, pipe utilisation, occupancy, memory, the top stall reasons.

    python tools/ncu_details.py gpurun_out/x.ncu-rep
"""
import csv
import io
import subprocess
import sys

KEYS = ["Duration", "SM Frequency", "Elapsed Cycles", "Executed Ipc Active", "Issue Slots Busy",
        "Compute (SM) Throughput", "Memory Throughput", "DRAM Throughput", "L2 Hit Rate",
        "Achieved Occupancy", "Registers Per Thread", "Warp Cycles Per Issued Instruction",
        "No Eligible", "Active Warps Per Scheduler", "Eligible Warps Per Scheduler",
        "Block Size", "Grid Size"]
raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "details", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr = rows[0]
ci = {k: hdr.index(k) for k in ("ID", "Kernel Name", "Section Name", "Metric Name", "Metric Unit",
                                "Metric Value")}
first = rows[1][ci["ID"]]
print(rows[1][ci["Kernel Name"]][:110])
seen = set()
for r in rows[1:]:
    if r[ci["ID"]] != first:
        break
    name = r[ci["Metric Name"]]
    if name in KEYS and name not in seen:
        seen.add(name)
        print(f"  {name}: {r[ci['Metric Value']]} {r[ci['Metric Unit']]}")
raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, vals = rows[0], rows[1], rows[2]
pipes = [(h, v) for h, v in zip(hdr, vals)
         if h.startswith("sm__inst_executed_pipe_") and h.endswith("avg.pct_of_peak_sustained_active")]
pipes = sorted(((float(v.replace(",", "")), h) for h, v in pipes if v), reverse=True)[:8]
print("  pipes (inst executed, % of peak sustained active):",
      ", ".join(f"{h[len('sm__inst_executed_pipe_'):].split('.')[0]} {v:.1f}" for v, h in pipes))
stalls = [(h, v) for h, v in zip(hdr, vals)
          if h.startswith("smsp__average_warp_latency_issue_stalled_") and h.endswith(".ratio")]
if not stalls:
    stalls = [(h, v) for h, v in zip(hdr, vals)
              if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio")]
st = sorted(((float(v.replace(",", "")), h) for h, v in stalls if v), reverse=True)[:6]
print("  top stalls (cycles per issued instruction):",
      ", ".join(f"{h.split('issue_stalled_')[1].split('_per_issue')[0].split('.')[0]} {v:.2f}"
                for v, h in st))
