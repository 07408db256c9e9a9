"""BJ.configs[4]: ten fks_step on the c4 box (48^3 cells x 32^3, HS, M = 64, CFL 1/8, Kn = 0.01), timed with CUDA
events, with the total mass after every step (A24: relative change per step <= 1e-12; transport is a
permutation, so only the collision's rounding moves it).  Usage: python tools/c4_ten_steps.py [steps]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1701_01608_b200 import binding as B  # noqa: E402
from paper_1701_01608_b200 import inputs  # noqa: E402
from paper_1701_01608_b200.configs import CONFIGS  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
cfg = CONFIGS["c4"]
f = inputs.make_f(cfg, device="cuda")
g = torch.empty_like(f)
col = B.Collision(cfg.N, cfg.L, cfg.M, cfg.M_r, cfg.kernel)
col.transport_setup(cfg.shape, cfg.cfl_num, cfg.cfl_den)
mass0 = f.sum().item()
absm = f.abs().sum().item()
rows = []
bufs = [f, g]
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for i in range(steps):
    e0.record()
    col.step(bufs[i % 2], bufs[(i + 1) % 2], cfg.coll_scale)
    e1.record()
    torch.cuda.synchronize()
    m = bufs[(i + 1) % 2].sum().item()
    rows.append({"step": i + 1, "ms": e0.elapsed_time(e1), "mass_rel_change_total": (m - mass0) / absm})
    mass_prev = m
per_step = [abs(rows[0]["mass_rel_change_total"])] + [abs(rows[i]["mass_rel_change_total"] - rows[i - 1]["mass_rel_change_total"]) for i in range(1, steps)]
print(json.dumps({"config": "c4", "steps": rows, "max_rel_mass_change_per_step": max(per_step),
                  "cell_vp_per_s": cfg.n_cells * cfg.N ** 3 * steps / (sum(r["ms"] for r in rows) / 1e3)}))
