"""Per-phase cycle counts of the v4 term-loop kernel (FKS_PHASE_TIMING=1; needs the instrumented build variant: FKS_LIB=$(python tools/build_variant.py ptime4 -DFKS_V4_PHASE_TIMING)): YX group 0 and Z warps of every CTA,
terms 2..5 of the first cell of each team.  Usage: python tools/phase_timing_v4.py [config] [n_cells]"""
import os
import sys

os.environ["FKS_PHASE_TIMING"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1701_01608_b200 import binding as B  # noqa: E402
from paper_1701_01608_b200 import inputs  # noqa: E402
from paper_1701_01608_b200.configs import CONFIGS  # noqa: E402

cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
n = int(sys.argv[2]) if len(sys.argv) > 2 else cfg.n_cells
f = inputs.make_f(cfg, device="cuda", cells=list(range(n)))
col = B.Collision(cfg.N, cfg.L, cfg.M, cfg.M_r, cfg.kernel)
print("layout", col.info)
Q = col.collision_batch(f)
torch.cuda.synchronize()
buf = B.fks_debug_timestamps(col.h)
raw = buf[: 144 * 128].reshape(144, 8, 16)[:, :4, :]  # [cta][term][slot]
raw = raw[raw[:, 0, 0] > 0]
yx, z = raw[:, :, :8].astype(float), raw[:, :, 8:].astype(float)
print("CTAs sampled:", len(raw))
for name, a, b in [("Y: wait W1 (poll + TMA)", 0, 1), ("Y: slot wait + 2 tasks", 1, 2),
                   ("X: wait Y", 3, 4), ("X: park", 4, 5), ("X: 3 tasks", 5, 6)]:
    d = yx[:, :, b] - yx[:, :, a]
    print(f"{name:28s} median {np.median(d):8.0f}  p10 {np.percentile(d, 10):8.0f}  p90 {np.percentile(d, 90):8.0f}")
d = yx[:, 1:, 3] - yx[:, :-1, 3]
print(f"{'X term period':28s} median {np.median(d):8.0f}")
d = yx[:, 1:, 0] - yx[:, :-1, 0]
print(f"{'YX term period':28s} median {np.median(d):8.0f}")
for name, a, b in [("Z: products (zt 0)", 0, 1), ("Z: barrier + publish", 1, 2), ("Z: wait W1 buffer free", 2, 3),
                   ("Z: class tasks + stores", 3, 4)]:
    d = z[:, :, b] - z[:, :, a]
    print(f"{name:28s} median {np.median(d):8.0f}  p10 {np.percentile(d, 10):8.0f}  p90 {np.percentile(d, 90):8.0f}")
d = z[:, 1:, 0] - z[:, :-1, 0]
print(f"{'Z term period':28s} median {np.median(d):8.0f}")
