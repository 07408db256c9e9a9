"""Small, fixed workload for ncu: one fks_step on the c2 slab (512 cells x 32^3, fast path) after one warm-up."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1701_01608_b200 import binding as B  # noqa: E402
from paper_1701_01608_b200 import inputs  # noqa: E402
from paper_1701_01608_b200.configs import CONFIGS  # noqa: E402

cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
n = int(sys.argv[2]) if len(sys.argv) > 2 else cfg.n_cells
f = inputs.make_f(cfg, device="cuda", cells=list(range(n)))
out = torch.empty_like(f)
col = B.Collision(cfg.N, cfg.L, cfg.M, cfg.M_r, cfg.kernel)
col.transport_setup((n, 1, 1), cfg.cfl_num, cfg.cfl_den)
for _ in range(2):
    col.step(f, out, cfg.coll_scale)
torch.cuda.synchronize()
print("ok path", col.info["path"], "launches", col.launches())
