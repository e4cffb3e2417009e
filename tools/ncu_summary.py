"""Key metrics of every kernel in an ncu report (details page).
  python tools/ncu_summary.py report.ncu-rep [regex]"""
import csv
import re
import subprocess
import sys

KEYS = ["Duration", "Elapsed Cycles", "SM Active Cycles", "Compute (SM) Throughput", "Memory Throughput",
        "DRAM Throughput", "L2 Hit Rate", "Issue Slots Busy", "Executed Ipc Active", "Registers Per Thread",
        "Grid Size", "Block Size", "Achieved Occupancy", "No Eligible", "Warp Cycles Per Issued Instruction"]
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "details", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[0]
pat = re.compile(sys.argv[2]) if len(sys.argv) > 2 else None
cur = None
for r in rows[1:]:
    d = dict(zip(h, r))
    name = f"{d['ID']} {d['Kernel Name'][:40]}"
    if pat and not pat.search(name):
        continue
    if name != cur:
        print(name)
        cur = name
    if d["Metric Name"] in KEYS:
        print(f"   {d['Metric Name']:38s} {d['Metric Value']:>14s} {d['Metric Unit']}")
