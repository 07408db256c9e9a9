"""Per-phase cycle counts of the fused hot kernel (debug build path: FKS_PHASE_TIMING=1)."""
import os
import sys

os.environ["FKS_PHASE_TIMING"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1701_01608_b200 import binding as B  # noqa: E402
from paper_1701_01608_b200 import inputs  # noqa: E402
from paper_1701_01608_b200.configs import CONFIGS  # noqa: E402

cfg = CONFIGS["c2"]
f = inputs.make_f(cfg, device="cuda")
col = B.Collision(cfg.N, cfg.L, cfg.M, cfg.M_r, cfg.kernel)
print("layout", col.info)
Q = col.collision_batch(f)
torch.cuda.synchronize()
raw = B.fks_debug_timestamps(col.h).reshape(-1, 64)[:, :32].reshape(-1, 4, 8)
raw = raw[raw[:, 0, 0] > 0]
ts = raw[:, :, :6]
sub = np.stack([raw[:, :, 6] - raw[:, :, 0], raw[:, :, 7] - raw[:, :, 6], raw[:, :, 1] - raw[:, :, 7]], -1).astype(float)
for i, n in enumerate(["Z: stage wait", "Z: product pass", "Z: tasks+stores"]):
    print(f"{n:16s} median {np.median(sub[:, :, i]):9.0f} clk")
d = np.diff(ts, axis=2).astype(float)  # Z, barrier, Y, sync, X
names = ["Z", "cluster barrier", "Y", "syncthreads", "X"]
print("CTAs sampled:", len(ts))
for i, n in enumerate(names):
    print(f"{n:16s} median {np.median(d[:, :, i]):9.0f} clk   p10 {np.percentile(d[:, :, i], 10):9.0f}  p90 {np.percentile(d[:, :, i], 90):9.0f}")
tot = np.median(ts[:, 1:, 0] - ts[:, :-1, 0])
print(f"term period (median) {tot:.0f} clk")
