"""Hottest SASS instructions of an ncu report (source page, SASS view): samples, stall columns."""
import csv, subprocess, sys
rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[1]
si, ni, ai = h.index("Source"), h.index("# Samples"), h.index("Address")
stall = h.index("Warp Stall Sampling (All Samples)")
data = []
for idx, r in enumerate(rows[2:]):
    try:
        data.append((int(r[ni]), idx, r[ai], r[si], r[stall]))
    except (ValueError, IndexError):
        pass
tot = sum(d[0] for d in data) or 1
print("total samples", tot)
for d in sorted(data, reverse=True)[:top]:
    print(f"{d[0]:6d} {100*d[0]/tot:5.1f}%  #{d[1]:5d} {d[3][:70]:70s} {d[4][:80]}")
