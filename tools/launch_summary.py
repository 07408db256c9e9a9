"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list: launches, total ms and share per kernel
(torch kernels excluded).  Usage: launch_summary.py CSV [header line]"""
import collections
import csv
import re
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 14 and r[0] != "ID"]
tot = collections.defaultdict(float)
cnt = collections.Counter()
for r in rows:
    name = r[4]
    if "at::" in name or "torch" in name or "elementwise" in name or "vectorized" in name:
        continue
    m = re.search(r"(?:fks::)?(?:\w+::)*(\w+)(?:<[^(]*>)?\(", name)
    key = m.group(1) if m else name[:40]
    scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "nsecond": 1e-6, "msecond": 1.0}[r[13]]
    tot[key] += float(r[14].replace(",", "")) * scale
    cnt[key] += 1
allt = sum(tot.values())
if len(sys.argv) > 2:
    print(sys.argv[2])
for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
    print(f"{k:40s} launches={cnt[k]:3d} total={v:9.2f} ms  share={100 * v / allt:5.1f}%")
