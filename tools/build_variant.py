"""Build a variant of libfks.so with extra nvcc defines into build_variants/libfks_<name>.so (for A/B timing on
the GPU box via FKS_LIB=...).  Usage: python tools/build_variant.py NAME [-DMACRO=V ...]"""
import os
import subprocess
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_1701_01608_b200"))
import build  # noqa: E402

name, extra = sys.argv[1], sys.argv[2:]
out_dir = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "build_variants")
os.makedirs(out_dir, exist_ok=True)
out = os.path.join(out_dir, f"libfks_{name}.so")
r = subprocess.run([build.NVCC] + build.FLAGS + extra + build.sources() + ["-o", out], capture_output=True, text=True)
if r.returncode != 0:
    sys.stderr.write(r.stderr[-4000:])
    sys.exit(1)
for ln in r.stderr.splitlines():
    if "spill" in ln and "hot_kernel_v4" in r.stderr:
        pass
print(out)
