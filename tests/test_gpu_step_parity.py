"""GPU parity of `fks_step` (transport → collision → explicit Euler, Eq. disc_relax; A17, A18)
against the CPU oracle on the configurations BASELINE.json names, including the exact configuration `bench.py`
times (c3: 32³ cells × 32³, CFL 1, Kn 1, transport fused into the fast path's first and last kernels).

Comparison (A23): per sampled cell, (f_out − f*) against s·Q_oracle(f*), where f* is the exact transport of the
GPU input with the ORACLE's own generic-cell shifts (`oracle.GenericCell`, `oracle.source_cells`).  Bound:
TOL_Q·max|s·Q_oracle| plus the rounding of the Euler sum itself (f_out is stored in fp64, so f_out − f* carries
up to one ulp of f*: 2^-52·max|f*|).  Sampling: blocks of 12 consecutive cells at the start, middle and end of
the grid; the hot kernel assigns the cells of a chunk round-robin to its 12 teams, so every block covers every
team, and the three blocks fall into the three chunks c3 runs as (≤ 24 GB of workspace per chunk).
"""
import numpy as np
import pytest
import torch

from oracle import fks_oracle as o
from paper_1701_01608_b200 import binding as B
from paper_1701_01608_b200 import dist as D
from paper_1701_01608_b200 import inputs
from paper_1701_01608_b200.configs import CONFIGS
from tests._common import TOL_Q, cfg_tables

pytestmark = pytest.mark.gpu

EPS = 2.0 ** -52


def make(cfg, **kw):
    return B.Collision(cfg.N, cfg.L, cfg.M, cfg.M_r, cfg.kernel, **kw)


def team_blocks(n_cells: int, width: int = 12, nblocks: int = 3):
    """Blocks of `width` consecutive cells (every team of a chunk) at nblocks evenly spaced starts, first and last
    cells included."""
    if nblocks == 3:
        starts = sorted({0, max(0, n_cells // 2 - width // 2), max(0, n_cells - width)})
    else:
        starts = sorted({min(max(0, n_cells - width), (n_cells - width) * i // (nblocks - 1)) for i in range(nblocks)})
    return sorted({c for s in starts for c in range(s, min(n_cells, s + width))})


def gather_fstar(cur: torch.Tensor, j: int, shape, delta: np.ndarray) -> np.ndarray:
    """f*_j = f[(j − δ(k)) mod n][k] on the device (a permutation, no arithmetic), with the oracle's sources."""
    N = cur.shape[-1]
    flat = cur.view(cur.shape[0], -1)
    src = torch.as_tensor(o.source_cells(int(j), shape, delta).reshape(-1), device=cur.device)
    idx = torch.arange(N ** 3, device=cur.device)
    return flat[src, idx].view(N, N, N).cpu().numpy()


def check_step_cells(cur, nxt, cells, shape, delta, tb, s):
    worst = 0.0
    for j in cells:
        fstar = gather_fstar(cur, j, shape, delta)
        dq_ref = s * o.collision_fast(fstar, tb)
        got = nxt[int(j)].cpu().numpy()
        err = np.abs((got - fstar) - dq_ref).max()
        bound = TOL_Q * np.abs(dq_ref).max() + EPS * np.abs(fstar).max()
        worst = max(worst, err / bound)
        assert err <= bound, (int(j), err, bound)
    return worst


@pytest.mark.parametrize("name", ["c2", "c3"])
def test_step_bench_configuration(cuda_device, name):
    """The step bench.py times (c3; and the c2 slab): fused transport on the fast path, two consecutive steps
    (the generic cell advances), 36 sampled cells per step, and box mass to 1e-12 per step (A24)."""
    cfg = CONFIGS[name]
    f = inputs.make_f(cfg, device=cuda_device)
    g = torch.empty_like(f)
    col = make(cfg)
    assert B.fks_get_path(col.h) == B.FKS_PATH_FAST
    col.transport_setup(cfg.shape, cfg.cfl_num, cfg.cfl_den)
    cell = o.GenericCell(N=cfg.N, c_num=cfg.cfl_num, c_den=cfg.cfl_den)
    tb = cfg_tables(name)
    s = cfg.coll_scale
    cells = team_blocks(cfg.n_cells)
    cur, nxt = f, g
    for _ in range(2):
        m0 = cur.sum(dtype=torch.float64).item()
        col.step(cur, nxt, s)
        torch.cuda.synchronize()
        d = cell.advance()
        assert np.array_equal(col.last_shift(), d)
        assert np.abs(d).max() >= 1            # the step really moves particles across cells
        check_step_cells(cur, nxt, cells, cfg.shape, d, tb, s)
        m1 = nxt.sum(dtype=torch.float64).item()
        assert abs(m1 - m0) / cur.abs().sum(dtype=torch.float64).item() <= 1e-12
        cur, nxt = nxt, cur
    del f, g


def test_step_c1_homogeneous_all_cells(cuda_device):
    """c1 (BKW, Maxwell molecules, N = 24, T + 1 = 257, homogeneous: c = 0, s = 0.01): every cell."""
    cfg = CONFIGS["c1"]
    f = inputs.make_f(cfg, device=cuda_device)
    out = torch.empty_like(f)
    col = make(cfg)
    col.transport_setup(cfg.shape, 0, 1)
    s = cfg.coll_scale
    col.step(f, out, s)
    torch.cuda.synchronize()
    assert not np.any(col.last_shift())
    worst = check_step_cells(f, out, range(cfg.n_cells), cfg.shape, col.last_shift(), cfg_tables("c1"), s)
    assert worst <= 1.0
    fh = f.cpu().numpy()
    assert abs(out.cpu().numpy().sum() - fh.sum()) / np.abs(fh).sum() <= 1e-12


def test_step_c4_two_steps_dense_sample(cuda_device):
    """c4 (48³ cells, M = 64, c = 1/8, Kn = 0.01) at full size: two steps, 12 blocks of 12 cells per step, so that
    every workspace chunk (about 11 per step) and both slots of the chunk pipeline are sampled."""
    cfg = CONFIGS["c4"]
    f = inputs.make_f(cfg, device=cuda_device)
    g = torch.empty_like(f)
    col = make(cfg)
    col.transport_setup(cfg.shape, cfg.cfl_num, cfg.cfl_den)
    cell = o.GenericCell(N=cfg.N, c_num=cfg.cfl_num, c_den=cfg.cfl_den)
    tb = cfg_tables("c4")
    cur, nxt = f, g
    for _ in range(2):
        col.step(cur, nxt, cfg.coll_scale)
        torch.cuda.synchronize()
        d = cell.advance()
        check_step_cells(cur, nxt, team_blocks(cfg.n_cells, nblocks=12), cfg.shape, d, tb, cfg.coll_scale)
        cur, nxt = nxt, cur
    del f, g


def test_slab_step_vs_oracle(cuda_device):
    """Slab-decomposed fks_step (ranks emulated in one process, gathers through the plane-pointer table) against
    the ORACLE's fks_step on the whole grid (not only against the single-domain GPU step): 3 slabs, CFL 3/2."""
    cfg = CONFIGS["c0"]
    shape, cfl, size = (7, 2, 2), (3, 2), 3
    nx, ny, nz = shape
    n = nx * ny * nz
    f = inputs.make_f(cfg, device=cuda_device, cells=[c % cfg.n_cells for c in range(n)])
    per = ny * nz
    doms = [D.SlabDomain(nx, ny, nz, r, size) for r in range(size)]
    bufs_a = [f[d.x0 * per:d.x1 * per].clone() for d in doms]
    bufs_b = [torch.empty_like(x) for x in bufs_a]
    cols = [make(cfg) for _ in doms]
    steppers = [D.SlabStepper(cols[r], doms[r], bufs_a[r], bufs_b[r], *cfl,
                              ptrs_a=[x.data_ptr() for x in bufs_a], ptrs_b=[x.data_ptr() for x in bufs_b])
                for r in range(size)]
    cell = o.GenericCell(N=cfg.N, c_num=cfl[0], c_den=cfl[1])
    tb = cfg_tables("c0")
    s = cfg.coll_scale
    cur = f
    for _ in range(2):
        outs = [st.step(s) for st in steppers]
        got = torch.cat(outs)
        torch.cuda.synchronize()
        d = cell.advance()
        check_step_cells(cur, got, range(n), shape, d, tb, s)
        cur = got.clone()


def test_two_streams_one_handle_are_ordered(cuda_device):
    """Two asynchronous calls on one handle from different streams share its workspace: the second must wait
    for the first.  Results equal the same calls made on one stream."""
    cfg = CONFIGS["c2"]
    col = make(cfg)
    fa = inputs.make_f(cfg, device=cuda_device, cells=list(range(0, 300)))
    fb = inputs.make_f(cfg, device=cuda_device, cells=list(range(200, 500)))
    qa_ref = col.collision_batch(fa).clone()
    qb_ref = col.collision_batch(fb).clone()
    torch.cuda.synchronize()
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    qa, qb = torch.empty_like(fa), torch.empty_like(fb)
    torch.cuda.synchronize()
    B.fks_collision_batch(col.h, fa, qa, stream=s1)
    B.fks_collision_batch(col.h, fb, qb, stream=s2)
    torch.cuda.synchronize()
    assert torch.equal(qa, qa_ref) and torch.equal(qb, qb_ref)


def test_slab_plane_table_checks(cuda_device):
    cfg = CONFIGS["c0"]
    col = make(cfg)
    B.fks_transport_setup_slab(col.h, 4, 1, 1, 1, 2, 1, 1)
    H = B.fks_slab_halo(col.h)
    assert B.fks_slab_plane_count(col.h) == 2 + 2 * H
    f = torch.zeros(6, cfg.N, cfg.N, cfg.N, dtype=torch.float64, device=cuda_device)
    g = torch.zeros(2, cfg.N, cfg.N, cfg.N, dtype=torch.float64, device=cuda_device)
    planes = [f[i].data_ptr() for i in range(2 + 2 * H)]
    with pytest.raises(B.FksError):                      # too short: refused by the binding
        B.fks_transport_step_slab(col.h, planes[:-1], g)
    hostbuf = torch.zeros(cfg.N ** 3, dtype=torch.float64)
    with pytest.raises(B.FksError) as ei:                # a host pointer among the planes
        B.fks_transport_step_slab(col.h, planes[:-1] + [hostbuf.data_ptr()], g)
    assert ei.value.status == B.FKS_ERR_INVALID
    B.fks_transport_step_slab(col.h, planes, g)
    B.fks_sync(col.h)
