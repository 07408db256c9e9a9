"""Run one collision batch of n cells of a config and report time (debugging aid for the persistent kernels)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1701_01608_b200 import binding as B  # noqa: E402
from paper_1701_01608_b200 import inputs  # noqa: E402
from paper_1701_01608_b200.configs import CONFIGS  # noqa: E402

cfg = CONFIGS[sys.argv[1]]
n = int(sys.argv[2])
f = inputs.make_f(cfg, device="cuda", cells=list(range(n)))
col = B.Collision(cfg.N, cfg.L, cfg.M, cfg.M_r, cfg.kernel)
t0 = time.time()
Q = col.collision_batch(f)
torch.cuda.synchronize()
print(cfg.name, n, "ok", round(time.time() - t0, 3), "s", float(Q.abs().max()), flush=True)
