"""fks_step vs fks_step_moments on the full c3 box (NEXT-1 cost): median of K steps each, CUDA events."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import json  # noqa: E402

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1701_01608_b200 import binding as B  # noqa: E402
from paper_1701_01608_b200 import inputs  # noqa: E402
from paper_1701_01608_b200.configs import CONFIGS  # noqa: E402

cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c3"]
K = int(sys.argv[2]) if len(sys.argv) > 2 else 3
f = inputs.make_f(cfg, device="cuda")
out = torch.empty_like(f)
col = B.Collision(cfg.N, cfg.L, cfg.M, cfg.M_r, cfg.kernel)
col.transport_setup(cfg.shape, cfg.cfl_num, cfg.cfl_den)
U = torch.empty((cfg.n_cells, 5), dtype=torch.float64, device="cuda")
W = torch.empty_like(U)
res = {}
for name in ["step", "step_moments", "step", "step_moments"]:
    ts = []
    for _ in range(K + 1):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        if name == "step":
            B.fks_step(col.h, f, out, cfg.coll_scale)
        else:
            B.fks_step_moments(col.h, f, out, cfg.coll_scale, U, W)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    res.setdefault(name, []).append(float(np.median(ts[1:])))
res["added_pct"] = 100.0 * (min(res["step_moments"]) / min(res["step"]) - 1.0)
print(json.dumps({"config": cfg.name, **res}))
