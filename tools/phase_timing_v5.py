"""Per-round cycle counts of the v5 term-loop kernel (FKS_PHASE_TIMING=1): CTA leader stamps for terms 2..5 of
the team's term sequence.  Usage: python tools/phase_timing_v5.py [config] [n_cells]"""
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
raw = buf[: 144 * 128].reshape(144, 8, 16)[:, :4, :4].astype(float)
raw = raw[raw[:, 0, 0] > 0]
print("CTAs sampled:", len(raw))
for name, a, b in [("wait W1", 0, 1), ("R1 (Y + Z part B)", 1, 2), ("R2 (X + Z part A)", 2, 3)]:
    d = raw[:, :, b] - raw[:, :, a]
    print(f"{name:24s} median {np.median(d):8.0f}  p10 {np.percentile(d, 10):8.0f}  p90 {np.percentile(d, 90):8.0f}")
d = raw[:, 1:, 0] - raw[:, :-1, 0]
print(f"{'term period':24s} median {np.median(d):8.0f}")
