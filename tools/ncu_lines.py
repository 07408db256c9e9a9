"""Attribute ncu warp-stall samples (source page, SASS) to CUDA source lines using a locally compiled cubin with
-lineinfo of the same source.  Usage: ncu_lines.py SASS_CSV CUBIN KERNEL_MANGLED [top]"""
import collections
import csv
import re
import subprocess
import sys

sass_csv, cubin, kern = sys.argv[1], sys.argv[2], sys.argv[3]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 30
dis = subprocess.run(["nvdisasm", "--print-line-info", cubin], capture_output=True, text=True).stdout.split("\n")
start = next(i for i, l in enumerate(dis) if ".section" in l and ".text." + kern in l)
off2line, cur = {}, None
for l in dis[start + 1:]:
    if ".section" in l and ".text." in l:
        break
    m = re.search(r"line (\d+)", l)
    if "//## File" in l and m:
        f = re.search(r'File "([^"]+)"', l)
        cur = (f.group(1).split("/")[-1] if f else "?") + ":" + m.group(1)
    mm = re.match(r"\s+/\*([0-9a-f]{4,})\*/", l)
    if mm:
        off2line[int(mm.group(1), 16)] = cur
rows = list(csv.reader(open(sass_csv)))
h, data = rows[1], rows[2:]
ix = {n: i for i, n in enumerate(h)}
base = int(data[0][ix["Address"]], 16)
f = lambda r, n: float(r[ix[n]] or 0) if r[ix[n]] not in ("", "-") else 0.0
reasons = [n for n in h if n.startswith("stall_") and "Not Issued" not in n]
tot = sum(f(r, "Warp Stall Sampling (All Samples)") for r in data)
byline = collections.defaultdict(collections.Counter)
miss = 0
for r in data:
    ln = off2line.get(int(r[ix["Address"]], 16) - base)
    if ln is None:
        miss += 1
        continue
    for n in reasons:
        byline[ln][n] += f(r, n)
    byline[ln]["all"] += f(r, "Warp Stall Sampling (All Samples)")
print(f"# unmapped {miss} of {len(data)} SASS rows; share of all stall samples per source line")
for ln, c in sorted(byline.items(), key=lambda kv: -kv[1]["all"])[:top]:
    t = [(n[6:], round(100 * v / tot, 1)) for n, v in c.most_common(5) if n != "all"][:3]
    print(f"{ln:26s} {100 * c['all'] / tot:5.1f}%  {t}")
