"""Collision timing through the raw C ABI (fks_collision_init / fks_collision_batch only), so that libraries of
older revisions can be timed side by side: FKS_LIB=path python tools/ab_time_raw.py [n_cells] [reps]"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1701_01608_b200 import inputs  # noqa: E402
from paper_1701_01608_b200.configs import CONFIGS  # noqa: E402

path = os.environ.get("FKS_LIB") or os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                                 "paper_1701_01608_b200", "libfks.so")
lib = C.CDLL(path)
lib.fks_collision_init.argtypes = [C.POINTER(C.c_void_p), C.c_int, C.c_double, C.c_int, C.c_int, C.c_int]
lib.fks_collision_batch.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_longlong, C.c_void_p]
cfg = CONFIGS[os.environ.get("FKS_CFG", "c3")]
n = int(sys.argv[1]) if len(sys.argv) > 1 else 4320
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
f = inputs.make_f(cfg, device="cuda", cells=list(range(n)))
Q = torch.empty_like(f)
h = C.c_void_p()
assert lib.fks_collision_init(C.byref(h), cfg.N, cfg.L, cfg.M, cfg.M_r, cfg.kernel) == 0
st = torch.cuda.current_stream().cuda_stream
assert lib.fks_collision_batch(h, f.data_ptr(), Q.data_ptr(), n, st) == 0
torch.cuda.synchronize()
ts = []
for _ in range(reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    lib.fks_collision_batch(h, f.data_ptr(), Q.data_ptr(), n, st)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
print(f"lib {os.path.basename(path)} {cfg.name} cells {n}: {np.median(ts):.3f} ms -> full {cfg.name} "
      f"{np.median(ts) * cfg.n_cells / n:.3f} ms; "
      f"checksum {Q[:256].abs().sum().item():.15e}")
