"""Summarise an `ncu --page source --csv --print-source sass` export:
instruction mix and the hottest SASS lines (by samples and by executed instructions)."""
import csv, sys, collections
lines = open(sys.argv[1]).read().splitlines()
rows = list(csv.reader(lines[1:]))
hdr = rows[0]
ix = {h: i for i, h in enumerate(hdr)}
data = rows[1:]
def f(r, k):
    try: return float(r[ix[k]].replace(",", "") or 0)
    except: return 0.0
tot_inst = sum(f(r, "Instructions Executed") for r in data)
tot_samp = sum(f(r, "Warp Stall Sampling (All Samples)") for r in data)
print(f"warp-level instructions executed: {tot_inst:.4g}; samples {tot_samp:.4g}")
ops = collections.Counter()
for r in data:
    op = r[ix["Source"]].split()[0] if r[ix["Source"]].split() else "?"
    if op.startswith("@"): op = r[ix["Source"]].split()[1]
    ops[op.split(".")[0]] += f(r, "Instructions Executed")
print("mix:", ", ".join(f"{k} {v/tot_inst*100:.1f}%" for k, v in ops.most_common(18)))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
print("--- hottest by samples")
for r in sorted(data, key=lambda r: -f(r, "Warp Stall Sampling (All Samples)"))[:top]:
    st = sorted(((f(r, c), c[6:]) for c in stall_cols), reverse=True)[:2]
    print(f"{r[ix['Address']]:>6} {f(r,'Warp Stall Sampling (All Samples)')/tot_samp*100:5.1f}%  inst {f(r,'Instructions Executed'):.3g}  {r[ix['Source']][:60]:60s} {st}")
