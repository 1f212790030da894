"""Key metrics of one kernel in an ncu report (details page), one per line.

    python tools/ncu_summary.py report.ncu-rep [kernel-substring]
"""
import csv
import io
import subprocess
import sys

KEYS = ["Duration", "DRAM Throughput", "Memory Throughput", "L1/TEX Hit Rate", "L2 Hit Rate",
        "Achieved Occupancy", "Registers Per Thread", "Compute (SM) Throughput", "Executed Ipc Active",
        "Issue Slots Busy", "Warp Cycles Per Issued Instruction", "No Eligible", "Active Warps Per Scheduler",
        "Dynamic Shared Memory Per Block", "L2 Compression", "Mem Busy", "Max Bandwidth", "Mem Pipes Busy",
        "Local Memory Spilling", "Shared Memory Configuration Size"]
rep = sys.argv[1]
kern = sys.argv[2] if len(sys.argv) > 2 else ""
out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[0]
ki, si, mi, ui, vi = (hdr.index(c) for c in ("Kernel Name", "Section Name", "Metric Name", "Metric Unit", "Metric Value"))
for r in rows[1:]:
    if kern in r[ki] and any(r[mi].startswith(k) for k in KEYS):
        print(f"{r[si][:28]:28s} {r[mi]:45s} {r[vi]:>14s} {r[ui]}")
