"""Per-kernel table from an ncu --csv --metrics launch list (tools/r02_full.sh):
duration, DRAM read/write bytes, GB/s, fraction of the measured HBM peak, algorithmic
bytes (a read and a write of the keys a pass moves; given per kernel
on the command line), and shared-memory bank-conflict wavefronts next to total
wavefronts for ld / st / atom.

  python tools/ncu_kernel_table.py ncu_C3.csv --n 268435456 --ksize 4 [--last-call]
Only the second hs_sort call of tools/one_call.py is summarised with --last-call
(launches after the midpoint of the list).
"""
import argparse
import collections
import csv
import json
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

ap = argparse.ArgumentParser()
ap.add_argument("csv")
ap.add_argument("--n", type=int, required=True)
ap.add_argument("--ksize", type=int, required=True)
ap.add_argument("--last-call", action="store_true")
ap.add_argument("--levels", type=int, default=3, help="active merge levels per step (for the alg. bytes)")
ap.add_argument("--counted", type=float, default=0.0,
                help="share of the keys in counted (not padded) split buckets: the count pass reads only those")
args = ap.parse_args()

rows = list(csv.DictReader(l for l in open(args.csv) if not l.startswith("==")))
launches = collections.OrderedDict()
for r in rows:
    launches.setdefault((int(r["ID"]), r["Kernel Name"]), {})[r["Metric Name"]] = (r["Metric Value"], r["Metric Unit"])
items = list(launches.items())
if args.last_call:
    items = items[len(items) // 2:]
UNIT = {"ns": 1e-9, "us": 1e-6, "ms": 1e-3, "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1.0, "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6,
        "Gbyte": 1e9, "%": 1.0, "": 1.0}


def v(m, k):
    val, unit = m.get(k, ("0", ""))
    return float(val.replace(",", "")) * UNIT.get(unit, 1.0)


peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
    os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0
nb = args.n * args.ksize
ALG = {"k_tile_hist": nb, "k_scatter": 2 * nb, "k_split_count": nb * args.counted, "k_split_scatter": 2 * nb, "k_tile_sort": 2 * nb,
       "k_merge_level": 2 * nb}
agg = collections.OrderedDict()
for (i, name), m in items:
    short = name.split("(")[0].replace("void ", "").replace("hs::", "").split("<")[0]
    a = agg.setdefault(short, collections.Counter())
    a["launches"] += 1
    t = v(m, "gpu__time_duration.sum")
    a["t"] += t
    if t > 20e-6:
        a["active"] += 1
    for k in ("dram__bytes_read.sum", "dram__bytes_write.sum",
              "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
              "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum",
              "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_atom.sum",
              "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum",
              "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum",
              "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum"):
        a[k] += v(m, k)
tot = sum(a["t"] for a in agg.values())
print(f"{'kernel':22s} {'launch':>6s} {'us':>9s} {'share':>6s} {'DRAM R GB':>9s} {'W GB':>7s} {'GB/s':>7s} "
      f"{'alg GB':>7s} {'alg/meas':>8s} {'frac':>5s}  {'ld conf/wavef (M)':>18s} {'st conf/wavef (M)':>18s} {'atom conf/wavef (M)':>20s}")
for k, a in sorted(agg.items(), key=lambda kv: -kv[1]["t"]):
    rd, wr, t = a["dram__bytes_read.sum"], a["dram__bytes_write.sum"], a["t"]
    alg = ALG.get(k)
    if alg is not None and k == "k_merge_level":
        alg = alg * args.levels
    gbs = (rd + wr) / t / 1e9 if t else 0
    fr = (alg / t / 1e9 / peak) if (alg and t) else None

    def cw(op):
        return (f"{a['l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_' + op + '.sum'] / 1e6:7.1f}/"
                f"{a['l1tex__data_pipe_lsu_wavefronts_mem_shared_op_' + op + '.sum'] / 1e6:7.1f}")
    print(f"{k:22s} {a['launches']:6d} {t * 1e6:9.1f} {t / tot:6.1%} {rd / 1e9:9.3f} {wr / 1e9:7.3f} {gbs:7.0f} "
          f"{(alg or 0) / 1e9:7.3f} {((rd + wr) / alg) if alg else 0:8.2f} {fr if fr else 0:5.2f}  {cw('ld'):>18s} "
          f"{cw('st'):>18s} {cw('atom'):>20s}")
print(f"total {tot * 1e3:.3f} ms (serialised, cold-cache ncu replay: compare shares); peak {peak} GB/s (measured copy)")
