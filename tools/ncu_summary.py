"""Print the key metrics of an .ncu-rep (first kernel ID) in a compact form."""
import csv
import subprocess
import sys

KEYS = ["Duration", "Elapsed Cycles", "Memory Throughput", "DRAM Throughput", "L2 Hit Rate", "L1/TEX Hit Rate",
        "Compute (SM) Throughput", "Registers Per Thread", "Achieved Occupancy", "Executed Ipc Active",
        "Issue Slots Busy", "Warp Cycles Per Issued Instruction", "No Eligible", "Eligible Warps Per Scheduler",
        "Active Warps Per Scheduler", "L2 Cache Throughput", "L1/TEX Cache Throughput", "Dynamic Shared Memory Per Block",
        "Executed Instructions", "Block Limit Shared Mem"]
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "details", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[0]
ix = {h: i for i, h in enumerate(hdr)}
want = sys.argv[2] if len(sys.argv) > 2 else rows[1][0]
seen = set()
print(next(r for r in rows[1:] if r[0] == want)[ix["Kernel Name"]][:60])
for r in rows[1:]:
    if r[0] != want:
        continue
    m = r[ix["Metric Name"]]
    if any(k == m for k in KEYS) and m not in seen:
        seen.add(m)
        print(f"  {m:40s} {r[ix['Metric Value']]:>14s} {r[ix['Metric Unit']]}")
