"""Write profiles/<out>.json with the DRAM bytes per cell of one kernel from an ncu --set full report.
Usage: python tools/traffic_json.py REPORT KERNEL_REGEX CELLS_PER_LAUNCH OUT_JSON"""
import csv
import json
import re
import subprocess
import sys

rep, kre, cells, out = sys.argv[1], sys.argv[2], float(sys.argv[3]), sys.argv[4]
txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(txt.splitlines()))
h = rows[0]
iname = h.index("Kernel Name")
for r in rows[2:]:
    if re.search(kre, r[iname]):
        get = lambda n: float(r[h.index(n)])
        scale = lambda n: {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}[rows[1][h.index(n)]]
        rd = get("dram__bytes_read.sum") * scale("dram__bytes_read.sum")
        wr = get("dram__bytes_write.sum") * scale("dram__bytes_write.sum")
        tu = rows[1][h.index("gpu__time_duration.sum")]
        t = get("gpu__time_duration.sum") * {"ns": 1e-6, "us": 1e-3, "ms": 1.0}[tu]
        json.dump({"kernel": r[iname][:120], "source": rep, "cells_per_launch": cells, "dram_bytes_read": rd,
                   "dram_bytes_write": wr, "dram_bytes_per_launch": rd + wr, "dram_bytes_per_cell": (rd + wr) / cells,
                   "ncu_ms": t}, open(out, "w"), indent=1)
        print(open(out).read())
        break
else:
    sys.exit("kernel not found")
