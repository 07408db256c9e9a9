"""Time the HBM-bound kernels on the full c3 box: transport alone, BGK step (fused), BGK operator, moments.
Usage: python tools/bgk_time.py [reps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1701_01608_b200 import binding as B  # noqa: E402
from paper_1701_01608_b200 import inputs  # noqa: E402
from paper_1701_01608_b200.configs import CONFIGS  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
cfg = CONFIGS["c3"]
f = inputs.make_f(cfg, device="cuda")
g = torch.empty_like(f)
n = cfg.n_cells
U = torch.empty((n, 5), dtype=torch.float64, device="cuda")
col = B.Collision(cfg.N, cfg.L, cfg.M, cfg.M_r, cfg.kernel)
col.transport_setup(cfg.shape, cfg.cfl_num, cfg.cfl_den)
nbytes = f.numel() * 8


def t(name, fn, traffic):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    print(f"{name:28s} {ms:8.3f} ms  {traffic / ms / 1e6:8.1f} GB/s algorithmic")


t("transport_step", lambda: col.transport_step(f, g), 2 * nbytes)
t("bgk_step (fused)", lambda: col.bgk_step(f, g, 0.0236), 2 * nbytes)
t("bgk_step + U", lambda: col.bgk_step(f, g, 0.0236, U), 2 * nbytes)
t("bgk_batch", lambda: col.bgk_batch(f, 10.0, g), 2 * nbytes)
t("moments", lambda: B.fks_moments(col.h, f, U, None, n), nbytes)
t("torch copy_", lambda: g.copy_(f), 2 * nbytes)
