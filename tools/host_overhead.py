"""Host cost per fks_step call vs the device step time (is a small config host-bound?).
Usage: python tools/host_overhead.py [config] [profile 0|1]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1701_01608_b200 import binding as B  # noqa: E402
from paper_1701_01608_b200 import inputs  # noqa: E402
from paper_1701_01608_b200.configs import CONFIGS  # noqa: E402

cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c1"]
prof = len(sys.argv) > 2 and sys.argv[2] == "1"
f = inputs.make_f(cfg, device="cuda")
g = torch.empty_like(f)
col = B.Collision(cfg.N, cfg.L, cfg.M, cfg.M_r, cfg.kernel)
col.transport_setup(cfg.shape, cfg.cfl_num, cfg.cfl_den)
for i in range(5):
    col.step(f, g, cfg.coll_scale)
torch.cuda.synchronize()
if prof:
    B.fks_profile(col.h, True)
for trial in range(3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    hs = []
    e0.record()
    t0 = time.perf_counter()
    for i in range(20):
        h0 = time.perf_counter()
        col.step(f if i % 2 == 0 else g, g if i % 2 == 0 else f, cfg.coll_scale)
        hs.append(time.perf_counter() - h0)
    t1 = time.perf_counter()
    e1.record()
    torch.cuda.synchronize()
    print(f"{cfg.name} profile={int(prof)}: host per call {1e3 * sum(hs) / 20:.3f} ms (max {1e3 * max(hs):.3f}), "
          f"device {e0.elapsed_time(e1) / 20:.3f} ms/step")
