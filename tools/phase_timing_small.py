"""Per-phase cycle counts of the small-N term kernel (FKS_PHASE_TIMING=1): for the first unit of CTAs 0..31, every
warp's busy time (work before the phase barrier) and the phase length (barrier exit to barrier exit).
Needs the instrumented build: FKS_LIB=$(python tools/build_variant.py ptime -DFKS_SMALL_PHASE_TIMING) python
tools/phase_timing_small.py [config]"""
import os
import sys

os.environ["FKS_PHASE_TIMING"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1701_01608_b200 import binding as B  # noqa: E402
from paper_1701_01608_b200 import inputs  # noqa: E402
from paper_1701_01608_b200.configs import CONFIGS  # noqa: E402

cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c1"]
f = inputs.make_f(cfg, device="cuda")
col = B.Collision(cfg.N, cfg.L, cfg.M, cfg.M_r, cfg.kernel)
col.collision_batch(f)
torch.cuda.synchronize()
ts = B.fks_debug_timestamps(col.h, 65536).reshape(32, 16, 64, 2)
W = 12 if cfg.N == 24 else 8
names = ["A (Z+X2)", "B (Y0)", "C (X0+Y1)", "D (X1+Y2)"]
busy = {n: [] for n in names}
length = {n: [] for n in names}
for cta in range(32):
    t = ts[cta, :W]
    if (t[:, :, 1] == 0).all():
        continue
    for k in range(1, 60):
        if (t[:, k, 1] == 0).any() or (t[:, k - 1, 1] == 0).any():
            break
        ph = names[k % 4]
        start = t[:, k - 1, 1].max()
        busy[ph].append(np.median(t[:, k, 0] - t[:, k - 1, 1]))
        busy[ph + " max"] = busy.get(ph + " max", []) + [np.max(t[:, k, 0] - t[:, k - 1, 1])]
        length[ph].append(t[:, k, 1].max() - start)
for n in names:
    print(f"{n:12s} phase median {np.median(length[n]):8.0f} cycles   warp busy median {np.median(busy[n]):8.0f}"
          f"   slowest warp median {np.median(busy[n + ' max']):8.0f}")
tot = sum(np.median(length[n]) for n in names)
print(f"term period ~ {tot:.0f} cycles")
