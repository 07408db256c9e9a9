"""Attribute ncu warp-stall samples and executed instructions of the N = 32 term-loop kernel to its warp roles
(Y, X, Z, setup) through the inlining chain of each SASS instruction (nvdisasm -gi of a locally compiled cubin of
the same source).  Usage: ncu_roles.py SASS_CSV CUBIN KERNEL_MANGLED SRC_FILE Y0-Y1 X0-X1 Z0-Z1
(line ranges of the kernel body that belong to each role)"""
import collections
import csv
import re
import subprocess
import sys

sass_csv, cubin, kern, src = sys.argv[1:5]
rng = {name: tuple(map(int, r.split("-"))) for name, r in zip("YXZ", sys.argv[5:8])}
dis = subprocess.run(["nvdisasm", "--print-line-info-inline", cubin], capture_output=True, text=True).stdout.split("\n")
start = next(i for i, l in enumerate(dis) if ".section" in l and ".text." + kern in l)
off2role, cur = {}, "setup"
for l in dis[start + 1:]:
    if ".section" in l and ".text." in l:
        break
    if "//## File" in l:
        lines = [int(x) for f, x in re.findall(r'File "([^"]+)", line (\d+)', l) if f.endswith(src)]
        lines += [int(x) for f, x in re.findall(r'inlined at "([^"]+)", line (\d+)', l) if f.endswith(src)]
        cur = "setup"
        for ln in lines:
            for name, (a, b) in rng.items():
                if a <= ln <= b:
                    cur = name
    mm = re.match(r"\s+/\*([0-9a-f]{4,})\*/", l)
    if mm:
        off2role[int(mm.group(1), 16)] = cur
rows = list(csv.reader(open(sass_csv)))
h, data = rows[1], rows[2:]
ix = {n: i for i, n in enumerate(h)}
base = int(data[0][ix["Address"]], 16)
f = lambda r, n: float(r[ix[n]] or 0) if r[ix[n]] not in ("", "-") else 0.0
reasons = [n for n in h if n.startswith("stall_") and "Not Issued" not in n]
agg = collections.defaultdict(collections.Counter)
for r in data:
    role = off2role.get(int(r[ix["Address"]], 16) - base, "?")
    agg[role]["samples"] += f(r, "Warp Stall Sampling (All Samples)")
    agg[role]["inst"] += f(r, "Instructions Executed")
    src_txt = r[ix["Source"]]
    if re.search(r"\bD(FMA|ADD|MUL)\b", src_txt):
        agg[role]["fp64"] += f(r, "Instructions Executed")
    for n in reasons:
        agg[role][n] += f(r, n)
tot_s = sum(a["samples"] for a in agg.values())
tot_i = sum(a["inst"] for a in agg.values())
for role, a in sorted(agg.items(), key=lambda kv: -kv[1]["samples"]):
    top = sorted(((a[n], n[6:]) for n in reasons), reverse=True)[:4]
    print(f"{role:6s} stall samples {100 * a['samples'] / tot_s:5.1f} %  warp-instructions {100 * a['inst'] / tot_i:5.1f} %"
          f"  fp64 {a['fp64'] / 1e9:6.2f} G  top: " + ", ".join(f"{n} {100 * v / tot_s:.1f}" for v, n in top))
