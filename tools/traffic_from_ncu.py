"""profiles/traffic_<cfg>.json from an ncu --set full report of tools/one_call.py: per kernel kind,
DRAM read + write bytes of its first captured launch (bench.py puts the dominant kernel's in
roofline.traffic).  usage: python tools/traffic_from_ncu.py full.ncu-rep C3"""
import csv
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
KIND = {"k_merge_level": "merge_level", "k_tile_sort": "tile_sort", "k_split_scatter": "split_scatter",
        "k_scatter": "scatter", "k_split_count": "split_count", "k_tile_hist": "tile_hist",
        "k_merge_partition": "merge_partition"}
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h, units = rows[0], rows[1]
ki, r, w = h.index("Kernel Name"), h.index("dram__bytes_read.sum"), h.index("dram__bytes_write.sum")
res = {}
for row in rows[2:]:
    kind = KIND.get(row[ki].split("(")[0].replace("void ", "").split("<")[0])
    if kind and kind not in res:
        res[kind] = sum(float(row[i].replace(",", "")) * UNIT.get(units[i], 1) for i in (r, w))
with open(os.path.join(ROOT, "profiles", f"traffic_{sys.argv[2]}.json"), "w") as f:
    json.dump(res, f, indent=1)
print(res)
