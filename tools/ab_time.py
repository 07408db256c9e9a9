"""A/B timing of the collision operator on a c3 subset: python tools/ab_time.py [n_cells] [reps].
Select the library with FKS_LIB=...; prints ms per call (median) and the per-phase split of fks_profile."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1701_01608_b200 import binding as B  # noqa: E402
from paper_1701_01608_b200 import inputs  # noqa: E402
from paper_1701_01608_b200.configs import CONFIGS  # noqa: E402

cfg = CONFIGS["c3"]
n = int(sys.argv[1]) if len(sys.argv) > 1 else 4320
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
f = inputs.make_f(cfg, device="cuda", cells=list(range(n)))
col = B.Collision(cfg.N, cfg.L, cfg.M, cfg.M_r, cfg.kernel)
Q = col.collision_batch(f)
torch.cuda.synchronize()
ts = []
for _ in range(reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    col.collision_batch(f, Q)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
print(f"lib {os.environ.get('FKS_LIB', 'default')} cells {n}: {np.median(ts):.2f} ms (min {min(ts):.2f}) "
      f"-> full c3 {np.median(ts) * 32768 / n:.1f} ms")
q = Q[:256].double()
print(f"  checksum sum|Q| {q.abs().sum().item():.17e}  sum Q {q.sum().item():.6e}")
