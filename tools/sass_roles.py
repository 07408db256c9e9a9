"""Static SASS size of each warp role of the N = 32 term-loop kernel (instruction-cache working set): instructions
attributed to the Y / X / Z sections of fast32.cu through their inlining chains.  Usage: sass_roles.py CUBIN"""
import collections
import re
import subprocess
import sys

src = open(__file__.rsplit("/", 2)[0] + "/paper_1701_01608_b200/csrc/fast32.cu").read().split("\n")
find = lambda s: next(i + 1 for i, l in enumerate(src) if s in l)
y0, x0, z0 = find("// ---------------- Y warp"), find("// ---------------- X warp"), find("-------- Z warps ---")
rng = {"Y": (y0, x0 - 1), "X": (x0, z0 - 1), "Z": (z0, len(src))}
dis = subprocess.run(["nvdisasm", "--print-line-info-inline", sys.argv[1]], capture_output=True, text=True).stdout.split("\n")
kern = "_ZN3fks3f322v413hot_kernel_v4ENS1_4ArgsE"
start = next(i for i, l in enumerate(dis) if ".section" in l and ".text." + kern in l)
cnt, cur = collections.Counter(), "setup"
for l in dis[start + 1:]:
    if ".section" in l and ".text." in l:
        break
    if "//## File" in l:
        lines = [int(x) for f, x in re.findall(r'"([^"]+)", line (\d+)', l) if f.endswith("fast32.cu")]
        cur = "setup"
        for ln in lines:
            for n, (a, b) in rng.items():
                if a <= ln <= b:
                    cur = n
    if re.match(r"\s+/\*[0-9a-f]{4,}\*/", l):
        cnt[cur] += 1
print({k: f"{v} instr = {v * 16 / 1024:.1f} KB" for k, v in cnt.items()}, f"total {sum(cnt.values()) * 16 / 1024:.1f} KB")
