"""Summarise an ncu --csv launch list: per launch name, time, DRAM bytes, GB/s."""
import csv, sys, collections
rows = list(csv.DictReader(l for l in open(sys.argv[1]) if not l.startswith("==")))
skip = int(sys.argv[2]) if len(sys.argv) > 2 else 0
launches = collections.OrderedDict()
for r in rows:
    key = (int(r["ID"]), r["Kernel Name"])
    launches.setdefault(key, {})[r["Metric Name"]] = (r["Metric Value"].replace(",", ""), r["Metric Unit"])
def val(m, name):
    v, u = m.get(name, ("0", ""))
    v = float(v)
    scale = {"nsecond": 1e-9, "ns": 1e-9, "usecond": 1e-6, "us": 1e-6, "msecond": 1e-3, "ms": 1e-3, "second": 1, "s": 1, "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
    return v * scale
tot = 0
items = list(launches.items())[skip:]
for (i, name), m in items:
    t = val(m, "gpu__time_duration.sum")
    rd = val(m, "dram__bytes_read.sum"); wr = val(m, "dram__bytes_write.sum")
    tot += t
    short = name.split("(")[0][:60]
    print(f"{i:4d} {short:60s} {t*1e6:9.1f} us  R {rd/1e9:7.3f} GB W {wr/1e9:7.3f} GB  {(rd+wr)/t/1e9 if t else 0:7.0f} GB/s")
print(f"total {tot*1e3:.3f} ms over {len(items)} launches")
