"""Library baseline for the collision operator (SURVEY §8(d) "cuFFT comparison"): the same Galerkin computation
with batched cuFFT 3D transforms (torch.fft) and element-wise PyTorch kernels, every intermediate (zero-padded
Z_t, z_t, G) materialised in HBM.  Uses the library's own tables (fks_get_tables) so the numbers are comparable;
checks Q against fks_collision_batch, then times it on c3 cells.  Comparison only: not a product path.

  python tools/cufft_baseline.py [batch] [reps]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1701_01608_b200 import binding as B  # noqa: E402
from paper_1701_01608_b200 import inputs  # noqa: E402
from paper_1701_01608_b200.configs import CONFIGS  # noqa: E402


def main():
    batch = int(sys.argv[1]) if len(sys.argv) > 1 else 64
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    cfg = CONFIGS["c3"]
    N, dev = cfg.N, torch.device("cuda:0")
    col = B.Collision(cfg.N, cfg.L, cfg.M, cfg.M_r, cfg.kernel)
    P, T = col.info["P"], col.info["T"]
    K = N - 1
    a, b, _, w = B.fks_get_tables(col.h, N, cfg.M)
    ab = torch.complex(torch.as_tensor(a), torch.as_tensor(b)).to(dev)  # (T+1, K, K, K): a_t + i b_t
    kp = np.arange(-(N // 2 - 1), N // 2)
    iN = torch.as_tensor(kp % N, device=dev)      # K' in the N-point spectrum
    iP = torch.as_tensor(kp % P, device=dev)      # K' in the P-point spectrum
    f = inputs.make_f(cfg, device=dev, cells=list(range(batch)))

    def collide(fb):
        fh = torch.fft.fftn(fb, dim=(1, 2, 3)) / N ** 3                           # f^ on the N-grid
        fh = fh[:, iN][:, :, iN][:, :, :, iN]                                      # K'^3
        G = torch.zeros((fb.shape[0], P, P, P), dtype=torch.float64, device=dev)
        Zp = torch.zeros((fb.shape[0], P, P, P), dtype=torch.complex128, device=dev)
        for t in range(T + 1):
            Zp[:, iP[:, None, None], iP[None, :, None], iP[None, None, :]] = ab[t] * fh
            z = torch.fft.ifftn(Zp, dim=(1, 2, 3)) * P ** 3                        # unnormalised inverse
            G += z.real * z.imag
        Gh = torch.fft.fftn(G, dim=(1, 2, 3)) / P ** 3
        Qh = torch.zeros((fb.shape[0], N, N, N), dtype=torch.complex128, device=dev)
        Qh[:, iN[:, None, None], iN[None, :, None], iN[None, None, :]] = Gh[:, iP][:, :, iP][:, :, :, iP]
        return (torch.fft.ifftn(Qh, dim=(1, 2, 3)) * N ** 3).real

    # same numbers as the library (tables are identical; only the summation order differs)
    q_lib = col.collision_batch(f[:4])
    q_ref = collide(f[:4])
    err = ((q_ref - q_lib).abs().amax(dim=(1, 2, 3)) / q_lib.abs().amax(dim=(1, 2, 3))).max().item()
    collide(f)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        collide(f)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    # ours on the same batch size and on a large batch (the persistent kernel needs >= 12 cells per team wave)
    res = {"batch": batch, "cufft_ms_per_batch": ms, "cufft_cell_vp_per_s": batch * N ** 3 / (ms / 1e3),
           "max_rel_err_vs_libfks": err}
    for nb in (batch, 4320):
        fb = f if nb == batch else inputs.make_f(cfg, device=dev, cells=list(range(nb)))
        Q = col.collision_batch(fb)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(reps):
            col.collision_batch(fb, Q)
        e1.record()
        torch.cuda.synchronize()
        m2 = e0.elapsed_time(e1) / reps
        res[f"libfks_cell_vp_per_s_batch{nb}"] = nb * N ** 3 / (m2 / 1e3)
    res["speedup_libfks_vs_cufft_large_batch"] = res["libfks_cell_vp_per_s_batch4320"] / res["cufft_cell_vp_per_s"]
    print(json.dumps(res))


if __name__ == "__main__":
    main()
