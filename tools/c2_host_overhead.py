import os, sys, time
sys.path.insert(0, os.getcwd())
import torch
from paper_1701_01608_b200 import binding as B
from paper_1701_01608_b200 import inputs
from paper_1701_01608_b200.configs import CONFIGS
cfg = CONFIGS["c2"]
f = inputs.make_f(cfg, device="cuda"); g = torch.empty_like(f)
col = B.Collision(cfg.N, cfg.L, cfg.M, cfg.M_r, cfg.kernel)
col.transport_setup(cfg.shape, cfg.cfl_num, cfg.cfl_den)
for i in range(3): col.step(f, g, cfg.coll_scale)
torch.cuda.synchronize()
import ctypes
for trial in range(2):
    t0 = time.perf_counter()
    hs = []
    for i in range(10):
        h0 = time.perf_counter(); col.step(f if i % 2 == 0 else g, g if i % 2 == 0 else f, cfg.coll_scale); hs.append(time.perf_counter() - h0)
    t1 = time.perf_counter(); torch.cuda.synchronize(); t2 = time.perf_counter()
    print(f"host per call {1e3*sum(hs)/10:.3f} ms (max {1e3*max(hs):.3f}), enqueue {1e3*(t1-t0)/10:.3f} ms/step, total {1e3*(t2-t0)/10:.3f} ms/step")
