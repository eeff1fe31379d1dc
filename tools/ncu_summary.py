"""Print the key metrics of an ncu report (details page) per kernel:
   python tools/ncu_summary.py report.ncu-rep [more metric substrings]"""
import csv
import io
import subprocess
import sys

WANT = ["Duration", "DRAM Throughput", "Memory Throughput", "L1/TEX Hit Rate", "L2 Hit Rate",
        "Compute (SM) Throughput", "Achieved Occupancy", "Issue Slots Busy", "Executed Ipc Active",
        "Registers Per Thread", "L1/TEX Cache Throughput", "L2 Cache Throughput", "Mem Busy", "Max Bandwidth",
        "Mem Pipes Busy", "No Eligible", "One or More Eligible", "Active Warps Per Scheduler",
        "Eligible Warps Per Scheduler", "Warp Cycles Per Issued Instruction", "SM Frequency", "Shared Memory"]
rep = sys.argv[1]
want = WANT + sys.argv[2:]
out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[0]
ki, mi, ui, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Unit"), hdr.index("Metric Value")
seen = set()
for r in rows[1:]:
    if len(r) <= vi:
        continue
    key = (r[0], r[mi])
    if key in seen:
        continue
    if any(w in r[mi] for w in want):
        seen.add(key)
        print(f"{r[0]:>2} {r[ki][:40]:40s} {r[mi]:45s} {r[vi]:>14s} {r[ui]}")
