"""Key per-kernel metrics from an ncu report (details page)."""
import csv, subprocess, sys
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "details", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[0]
ki = hdr.index("Kernel Name"); mi = hdr.index("Metric Name"); vi = hdr.index("Metric Value"); ui = hdr.index("Metric Unit")
idi = hdr.index("ID")
want = ["Duration", "DRAM Throughput", "Compute (SM) Throughput", "Executed Ipc Active", "Issue Slots Busy",
        "Registers Per Thread", "Achieved Occupancy", "Theoretical Occupancy", "Block Limit Registers",
        "Block Limit Shared Mem", "Warp Cycles Per Issued Instruction", "Eligible Warps Per Scheduler",
        "L1/TEX Hit Rate", "L2 Hit Rate", "Mem Busy"]
cur = None
seen = set()
for r in rows[1:]:
    key = (r[idi], r[ki])
    if key != cur:
        cur = key; seen = set(); print("====", r[idi], r[ki][:80])
    if r[mi] in want and r[mi] not in seen:
        seen.add(r[mi]); print(f"    {r[mi]:40s} {r[vi]} {r[ui]}")
