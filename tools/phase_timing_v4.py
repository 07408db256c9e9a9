"""Steady-state phase accounting of the N = 32 term-loop kernel: cycles per term spent in each phase by lane 0 of
Y warps 6 (class 0) and 7 (class 1), X warp 0 and Z warps 12 / 13 of every CTA, summed over the terms of each team's third cell (needs the
instrumented build variant: FKS_LIB=$(python tools/build_variant.py ptime4 -DFKS_V4_PHASE_TIMING)).
Usage: python tools/phase_timing_v4.py [config] [n_cells]   (n_cells >= 3 x 12 teams)"""
import os
import sys

os.environ["FKS_PHASE_TIMING"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1701_01608_b200 import binding as B  # noqa: E402
from paper_1701_01608_b200 import inputs  # noqa: E402
from paper_1701_01608_b200.configs import CONFIGS  # noqa: E402

cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c3"]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 1440
f = inputs.make_f(cfg, device="cuda", cells=list(range(n)))
col = B.Collision(cfg.N, cfg.L, cfg.M, cfg.M_r, cfg.kernel)
Q = col.collision_batch(f)
torch.cuda.synchronize()
T1 = col.info["T"] + 1
buf = B.fks_debug_timestamps(col.h)[: 144 * 128].reshape(144, 128).astype(float) / T1
roles = [("Y warp 6", 0, ["W1 issue/wait/ack", "2 transforms", "slot wait", "2 x 16 stores", "signal/prefetch"]),
         ("Y warp 7", 32, ["W1 issue/wait/ack", "2 transforms", "slot wait", "2 x 16 stores", "signal/prefetch"]),
         ("X warp 0", 8, ["wait for Y", "park", "3 class tasks", "G write-out"]),
         ("Z warp 13", 16, ["products", "barrier", "class tasks + barrier"]),
         ("Z warp 12", 24, ["publish + ring poll", "barrier", "class tasks + barrier"])]
print(f"cycles per term (median over {len(buf)} CTAs; terms of each team's third cell), T+1 = {T1}")
for name, off, labels in roles:
    tot = buf[:, off:off + len(labels)].sum(1)
    parts = "  ".join(f"{lab} {np.median(buf[:, off + i]):6.0f}" for i, lab in enumerate(labels))
    print(f"{name:10s} period {np.median(tot):6.0f} | {parts}")
