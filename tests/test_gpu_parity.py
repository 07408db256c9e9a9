"""GPU parity: libfks (through the C ABI) vs the CPU oracle on the same seeded inputs.

Tolerances: tables ≤ 1e-13·max|table| (P17); Q per cell ≤ 1e-10 relative L∞ (BJ.north_star, A23);
transport bit-exact (A25); mass defect |ΣQ|/Σ|Q_loss| ≤ 1e-11 (A24).
"""
import numpy as np
import pytest
import torch

from oracle import fks_oracle as o
from paper_1701_01608_b200 import binding as B
from paper_1701_01608_b200 import inputs
from paper_1701_01608_b200.configs import CONFIGS, L_BOX
from tests._common import TOL_Q, TOL_TABLE, cfg_tables, oracle_tables, oracle_Q, rel_err_per_cell

pytestmark = pytest.mark.gpu


def make(cfg, path=B.FKS_PATH_AUTO, **kw):
    return B.Collision(cfg.N, cfg.L, cfg.M, cfg.M_r, cfg.kernel, path=path, **kw)


# ---------------- P17: tables -------------------------------------------------------------------------

@pytest.mark.parametrize("name", ["c0", "c1", "c2", "c4"])
def test_tables_match_oracle(cuda_device, name):
    cfg = CONFIGS[name]
    col = make(cfg)
    ref = cfg_tables(name)
    e, w = o.directions(*o.split_angles(cfg.M))
    a, b, dirs, ww = B.fks_get_tables(col.h, cfg.N, len(w))
    assert np.abs(dirs - e).max() < 1e-15 and np.abs(ww - w).max() < 1e-15
    assert a.shape == ref.a.shape
    assert np.abs(a - ref.a).max() <= TOL_TABLE * np.abs(ref.a).max()
    assert np.abs(b - ref.b).max() <= TOL_TABLE * np.abs(ref.b).max()


@pytest.mark.parametrize("kw", [dict(quad_rule=1), dict(cutoff_ratio=1.5), dict(n_theta=2, n_phi=3)])
def test_tables_variants(cuda_device, kw):
    col = B.Collision(12, L_BOX, 16, 16, 0, **kw)
    ref = oracle_tables(12, L_BOX, 16, 16, 0, n_theta=kw.get("n_theta", 0), n_phi=kw.get("n_phi", 0),
                        rule=kw.get("quad_rule", 0), cutoff_ratio=kw.get("cutoff_ratio", 1.0))
    nd = ref.w.size
    a, b, _, _ = B.fks_get_tables(col.h, 12, nd)
    assert np.abs(a - ref.a).max() <= TOL_TABLE * np.abs(ref.a).max()
    assert np.abs(b - ref.b).max() <= TOL_TABLE * np.abs(ref.b).max()


# ---------------- collision: small configs in full ----------------------------------------------------

@pytest.mark.parametrize("name", ["c0", "c1"])
def test_collision_config_full(cuda_device, name):
    cfg = CONFIGS[name]
    f = inputs.make_f(cfg, device=cuda_device)
    col = make(cfg)
    Q = col.collision_batch(f)
    torch.cuda.synchronize()
    fh, qh = f.cpu().numpy(), Q.cpu().numpy()
    tb = cfg_tables(name)
    ref = oracle_Q(fh, tb)
    err = rel_err_per_cell(qh, ref)
    assert err.max() <= TOL_Q, err.max()
    loss = np.stack([np.abs(o.loss_part(x, tb)).sum() for x in fh])
    assert (np.abs(qh.reshape(len(fh), -1).sum(1)) / loss).max() <= 1e-11


@pytest.mark.parametrize("N", [4, 6, 8, 12, 16])
@pytest.mark.parametrize("kernel", [0, 1])
def test_collision_random_fields_vs_direct_sum(cuda_device, N, kernel):
    M_r = 4
    f = inputs.random_field(3, N, seed=N + 10 * kernel, signed=(N % 4 == 0)).to(cuda_device)
    col = B.Collision(N, L_BOX, 16, M_r, kernel)
    Q = col.collision_batch(f).cpu().numpy()
    tb = oracle_tables(N, L_BOX, 16, M_r, kernel)
    ref = np.stack([o.collision_direct(x, tb) for x in f.cpu().numpy()])
    assert rel_err_per_cell(Q, ref).max() <= TOL_Q


@pytest.mark.parametrize("pad", [0, 22, 32])
def test_collision_pad_and_projection(cuda_device, pad):
    N = 16
    cfg = CONFIGS["c0"]
    f = inputs.make_f(cfg, device=cuda_device)[:3]
    col = B.Collision(N, L_BOX, 16, 16, 0, pad=pad, project_mass=1)
    Q = col.collision_batch(f).cpu().numpy()
    ref = oracle_Q(f.cpu().numpy(), cfg_tables("c0"), P=pad or None, project_mass=True)
    assert rel_err_per_cell(Q, ref).max() <= TOL_Q
    assert np.abs(Q.reshape(3, -1).sum(1)).max() <= 1e-13 * np.abs(Q).max() * Q[0].size


@pytest.mark.parametrize("N", [6, 8, 12, 16])
def test_collision_aliased_variant_vs_direct_sum(cuda_device, N):
    """pad P < 3N/2 - 2 is the aliased collocation operator (P = N: classical collocation),
    compared with the oracle's brute-force sum over l + m = k mod P (pinned, P24)."""
    tb = oracle_tables(N, L_BOX, 16, 4, 0)
    f = inputs.random_field(3, N, seed=40 + N, signed=False).to(cuda_device)
    for P in sorted({N, N + 2, 3 * N // 2 - 3}):
        if P < N:
            continue
        col = B.Collision(N, L_BOX, 16, 4, 0, pad=P)
        assert col.info["P"] == P and col.info["path"] == B.FKS_PATH_GENERIC
        Q = col.collision_batch(f).cpu().numpy()
        ref = np.stack([o.collision_direct(x, tb, P=P) for x in f.cpu().numpy()])
        assert rel_err_per_cell(Q, ref).max() <= TOL_Q, P


def test_collision_aliased_N32_P32(cuda_device):
    cfg = CONFIGS["c2"]
    f = inputs.make_f(cfg, device=cuda_device, cells=[0, 300])
    col = B.Collision(cfg.N, cfg.L, cfg.M, cfg.M_r, cfg.kernel, pad=32)
    Q = col.collision_batch(f).cpu().numpy()
    ref = oracle_Q(f.cpu().numpy(), cfg_tables("c2"), P=32)
    assert rel_err_per_cell(Q, ref).max() <= TOL_Q


# ---------------- variable hard spheres ----------------------------------------

@pytest.mark.parametrize("alpha,C", [(0.5, 0.0), (0.3, 0.1), (1.0, 0.25)])
def test_tables_vhs(cuda_device, alpha, C):
    col = B.Collision(12, L_BOX, 16, 8, 2, vhs_alpha=alpha, vhs_C=C)
    ref = oracle_tables(12, L_BOX, 16, 8, 2, alpha=alpha, C_alpha=C or o.VHS_C_DEFAULT)
    a, b, _, _ = B.fks_get_tables(col.h, 12, ref.w.size)
    assert np.abs(a - ref.a).max() <= TOL_TABLE * np.abs(ref.a).max()
    assert np.abs(b - ref.b).max() <= TOL_TABLE * np.abs(ref.b).max()


@pytest.mark.parametrize("N", [6, 8])
def test_collision_vhs_vs_direct_sum(cuda_device, N):
    f = inputs.random_field(3, N, seed=70 + N, signed=False).to(cuda_device)
    col = B.Collision(N, L_BOX, 16, 4, 2, vhs_alpha=0.5)
    Q = col.collision_batch(f).cpu().numpy()
    tb = oracle_tables(N, L_BOX, 16, 4, 2, alpha=0.5)
    ref = np.stack([o.collision_direct(x, tb) for x in f.cpu().numpy()])
    assert rel_err_per_cell(Q, ref).max() <= TOL_Q


def test_collision_vhs_fast_path_c2(cuda_device):
    cfg = CONFIGS["c2"]
    f = inputs.make_f(cfg, device=cuda_device, cells=[3])
    col = B.Collision(cfg.N, cfg.L, cfg.M, 2, 2, vhs_alpha=0.5)
    assert col.info["path"] == B.FKS_PATH_FAST and col.info["T"] == cfg.M * 2
    Q = col.collision_batch(f).cpu().numpy()
    ref = oracle_Q(f.cpu().numpy(), oracle_tables(cfg.N, cfg.L, cfg.M, 2, 2, alpha=0.5))
    assert rel_err_per_cell(Q, ref).max() <= TOL_Q


def test_vhs_argument_checks(cuda_device):
    with pytest.raises(B.FksError):
        B.Collision(8, L_BOX, 16, 4, 2, vhs_alpha=1.5)
    with pytest.raises(B.FksError):
        B.Collision(8, L_BOX, 16, 0, 2, vhs_alpha=0.5)


def test_collision_bkw_report(cuda_device):
    """c1 (BKW, N = 24): Q vs the analytic ∂f/∂t.  Resolution-limited (~0.2-0.5, P14): reported,
    gated only loosely; the 1e-6 BKW pin is the oracle's N = 64 test."""
    cfg = CONFIGS["c1"]
    f = inputs.make_f(cfg, device=cuda_device)[:4]
    Q = make(cfg).collision_batch(f).cpu().numpy()
    Ks = inputs.cell_params(cfg)[:4, 0, 0]
    v3 = o.velocity_grid3(cfg.N, cfg.L)
    for q, K in zip(Q, Ks):
        ex = o.bkw_dfdt(v3, K)
        assert np.abs(q - ex).max() / np.abs(ex).max() < 1.0


# ---------------- edge cases ---------------------------------------------------------------------------

def test_edge_cases(cuda_device):
    col = B.Collision(8, L_BOX, 16, 16, 0)
    f = torch.rand(4, 8, 8, 8, dtype=torch.float64, device=cuda_device)
    Q = torch.full_like(f, 7.0)
    B.fks_collision_batch(col.h, f, Q, 0)                      # n_cells = 0: no-op
    torch.cuda.synchronize()
    assert (Q == 7.0).all()
    with pytest.raises(B.FksError) as ei:
        B.fks_collision_batch(col.h, f, f, 4)                   # overlap
    assert ei.value.status == B.FKS_ERR_INVALID
    with pytest.raises(B.FksError) as ei:
        B.fks_collision_batch(col.h, f.cpu(), Q, 4)             # host pointer
    assert ei.value.status == B.FKS_ERR_INVALID
    with pytest.raises(B.FksError) as ei:
        B.fks_step(col.h, f, Q, 0.1)                            # before transport setup
    assert ei.value.status == B.FKS_ERR_STATE
    # one cell, ragged counts
    for n in (1, 3):
        Q = col.collision_batch(f[:n].contiguous())
        ref = oracle_Q(f[:n].cpu().numpy(), oracle_tables(8, L_BOX, 16, 16, 0))
        assert rel_err_per_cell(Q.cpu().numpy(), ref).max() <= TOL_Q
    B.fks_sync(col.h)


def test_chunking_matches_unchunked(cuda_device):
    cfg = CONFIGS["c0"]
    f = inputs.make_f(cfg, device=cuda_device)
    q1 = B.Collision(16, L_BOX, 16, 16, 0).collision_batch(f)
    q2 = B.Collision(16, L_BOX, 16, 16, 0, max_cells_in_flight=3).collision_batch(f)
    assert torch.equal(q1, q2)


@pytest.mark.parametrize("n, chunk, sub", [(30, 7, None), (25, 12, None), (13, 12, None), (40, 16, "3"), (30, 12, "5")])
def test_pipelined_chunks_match_unchunked(cuda_device, monkeypatch, n, chunk, sub):
    """N = 32 batches of more than one workspace chunk run through the two-slot stream pipeline (the transforms of
    chunks k - 1 and k + 1 beside the term loop of chunk k, fast32.cu fast_collision_pipelined): bit-identical to
    one chunk and to the same chunking run sequentially (FKS_NO_PIPELINE=1 at init), for ragged last chunks,
    two chunks and many; collision batch and Euler step with the fused transport gather; with the side-stream
    transforms launched over sub-ranges of `sub` cells (FKS_PIPE_SUB; ragged last sub-range)."""
    if sub is not None:
        monkeypatch.setenv("FKS_PIPE_SUB", sub)
    cfg = CONFIGS["c3"]
    f = inputs.make_f(cfg, device=cuda_device, cells=list(range(n)))
    whole = make(cfg)
    piped = make(cfg, max_cells_in_flight=chunk)
    monkeypatch.setenv("FKS_NO_PIPELINE", "1")
    seq = make(cfg, max_cells_in_flight=chunk)
    monkeypatch.delenv("FKS_NO_PIPELINE")
    q = [c.collision_batch(f) for c in (whole, piped, seq)]
    assert torch.equal(q[0], q[1]) and torch.equal(q[0], q[2])
    shape = (n, 1, 1)
    outs = []
    for c in (whole, piped, seq):
        c.transport_setup(shape, 1, 1)
        out = torch.empty_like(f)
        c.step(f, out, 0.05)
        outs.append(out)
    torch.cuda.synchronize()
    assert torch.equal(outs[0], outs[1]) and torch.equal(outs[0], outs[2])


# ---------------- transport and the step ---------------------------------------------------------------

def test_transport_bit_exact(cuda_device):
    N, shape = 8, (5, 4, 3)
    n = 60
    f = torch.rand(n, N, N, N, dtype=torch.float64, device=cuda_device)
    col = B.Collision(N, L_BOX, 16, 16, 0)
    col.transport_setup(shape, 7, 3)
    cell = o.GenericCell(N=N, c_num=7, c_den=3)
    ref = f.cpu().numpy()
    cur = f
    for _ in range(4):
        out = torch.empty_like(cur)
        col.transport_step(cur, out)
        d = cell.advance()
        assert np.array_equal(col.last_shift(), d)
        ref = o.transport(ref, shape, d)
        assert np.array_equal(out.cpu().numpy(), ref)
        cur = out


def test_step_homogeneous_c0(cuda_device):
    cfg = CONFIGS["c0"]
    f = inputs.make_f(cfg, device=cuda_device)
    col = make(cfg)
    col.transport_setup(cfg.shape, 0, 1)
    out = torch.empty_like(f)
    s = cfg.coll_scale
    col.step(f, out, s)
    fh = f.cpu().numpy()
    Q = oracle_Q(fh, cfg_tables("c0"))
    got = out.cpu().numpy()
    dq = (got - fh) / s
    assert rel_err_per_cell(dq, Q).max() <= 1e-9
    assert np.abs(got.sum() - fh.sum()) / np.abs(fh).sum() <= 1e-12      # mass per step (A24)


def test_step_with_transport(cuda_device):
    N, shape = 16, (4, 3, 2)
    cfg = CONFIGS["c0"]
    n = 24
    f = inputs.random_field(n, N, seed=3).to(cuda_device) * 0.01 + inputs.make_f(cfg, device=cuda_device)[:1]
    col = B.Collision(N, L_BOX, 16, 16, 0)
    col.transport_setup(shape, 1, 2)
    cell = o.GenericCell(N=N, c_num=1, c_den=2)
    tb = cfg_tables("c0")
    cur = f
    ref = f.cpu().numpy()
    s = 0.01
    for _ in range(2):
        out = torch.empty_like(cur)
        col.step(cur, out, s)
        ref = o.fks_step(ref, shape, cell, tb, s)
        got = out.cpu().numpy()
        dq_ref = ref - o.transport(cur.cpu().numpy(), shape, col.last_shift())
        dq = got - o.transport(cur.cpu().numpy(), shape, col.last_shift())
        assert rel_err_per_cell(dq, dq_ref).max() <= 1e-9
        cur = out
        ref = got  # continue from the GPU state so both see identical inputs


# ---------------- full-size configs on sampled cells ------------------------------------------------------

@pytest.mark.parametrize("name", ["c2", "c3"])
def test_collision_config_sampled(cuda_device, name):
    cfg = CONFIGS[name]
    f = inputs.make_f(cfg, device=cuda_device)
    col = make(cfg)
    Q = col.collision_batch(f)
    torch.cuda.synchronize()
    cells = inputs.sample_cells(cfg, 4)
    fh = f[cells].cpu().numpy()
    ref = oracle_Q(fh, cfg_tables(name))
    assert rel_err_per_cell(Q[cells].cpu().numpy(), ref).max() <= TOL_Q
    del f, Q


# ---------------- fast path (N = 32 fused kernel) -----------------------------------------------------------

@pytest.mark.parametrize("name", ["c2", "c4"])
def test_fast_path_vs_oracle(cuda_device, name):
    cfg = CONFIGS[name]
    col = make(cfg, path=B.FKS_PATH_FAST)
    assert B.fks_get_path(col.h) == B.FKS_PATH_FAST
    cells = [0, 1, 2, cfg.n_cells // 2 + 3, cfg.n_cells - 1]
    f = inputs.make_f(cfg, device=cuda_device, cells=cells)
    Q = col.collision_batch(f).cpu().numpy()
    ref = oracle_Q(f.cpu().numpy(), cfg_tables(name))
    assert rel_err_per_cell(Q, ref).max() <= TOL_Q


def test_fast_path_random_and_ragged(cuda_device):
    cfg = CONFIGS["c2"]
    col = make(cfg, path=B.FKS_PATH_FAST)
    f = inputs.random_field(7, 32, seed=11, signed=True).to(cuda_device)
    Q = col.collision_batch(f).cpu().numpy()
    ref = oracle_Q(f.cpu().numpy(), cfg_tables("c2"))
    assert rel_err_per_cell(Q, ref).max() <= TOL_Q
    # generic and fast paths agree on the same input (different arithmetic order only)
    qg = make(cfg, path=B.FKS_PATH_GENERIC).collision_batch(f).cpu().numpy()
    assert rel_err_per_cell(Q, qg).max() <= TOL_Q


def test_fast_path_project_mass(cuda_device):
    """project_mass (A24: Q^_0 := 0) on the N = 32 fast path: the zero mode is cleared in the back transform's first
    kernel (kx = 0 plane of the x-transformed G); against the oracle with project_mass, and Σ Q = 0 to rounding."""
    cfg = CONFIGS["c2"]
    col = make(cfg, path=B.FKS_PATH_FAST, project_mass=1)
    f = inputs.make_f(cfg, device=cuda_device, cells=[0, 5, 300, 511])
    Q = col.collision_batch(f).cpu().numpy()
    ref = oracle_Q(f.cpu().numpy(), cfg_tables("c2"), project_mass=True)
    assert rel_err_per_cell(Q, ref).max() <= TOL_Q
    assert np.abs(Q.reshape(4, -1).sum(1)).max() <= 1e-13 * np.abs(Q).max() * Q[0].size


def test_fast_path_mass(cuda_device):
    cfg = CONFIGS["c4"]
    f = inputs.make_f(cfg, device=cuda_device, cells=list(range(16)))
    col = make(cfg, path=B.FKS_PATH_FAST)
    Q = col.collision_batch(f).cpu().numpy()
    tb = cfg_tables("c4")
    fh = f.cpu().numpy()
    loss = np.stack([np.abs(o.loss_part(x, tb)).sum() for x in fh])
    assert (np.abs(Q.reshape(16, -1).sum(1)) / loss).max() <= 1e-11


def test_c4_full_box_step_sampled(cuda_device):
    """c4 at full size (48^3 cells x 32^3, 29 GB per copy, M = 64, c = 1/8, Kn = 0.01): two fks_step on the
    device; after each, sampled cells are checked against the oracle applied to the transported GPU state
    (exact gather of the previous state with the oracle's own shifts), and mass is conserved to 1e-12."""
    cfg = CONFIGS["c4"]
    f = inputs.make_f(cfg, device=cuda_device)
    g = torch.empty_like(f)
    col = make(cfg)
    col.transport_setup(cfg.shape, cfg.cfl_num, cfg.cfl_den)
    cell = o.GenericCell(N=cfg.N, c_num=cfg.cfl_num, c_den=cfg.cfl_den)
    tb = cfg_tables("c4")
    s = cfg.coll_scale
    cells = inputs.sample_cells(cfg, 3, seed=4)
    cur, nxt = f, g
    for step in range(2):
        m0 = cur.sum(dtype=torch.float64).item()
        col.step(cur, nxt, s)
        torch.cuda.synchronize()
        d = cell.advance()
        assert np.array_equal(col.last_shift(), d)
        flat = cur.view(cur.shape[0], -1)
        for j in cells:
            src = torch.as_tensor(o.source_cells(int(j), cfg.shape, d).reshape(-1), device=cuda_device)
            idx = torch.arange(cfg.N ** 3, device=cuda_device)
            fstar = flat[src, idx].view(cfg.N, cfg.N, cfg.N).cpu().numpy()
            ref = o.euler(fstar, o.collision_fast(fstar, tb), s)
            got = nxt[int(j)].cpu().numpy()
            dq_ref = ref - fstar                       # = s * Q_oracle(f*)
            assert np.abs((got - fstar) - dq_ref).max() <= TOL_Q * np.abs(dq_ref).max() + 1e-15
        m1 = nxt.sum(dtype=torch.float64).item()
        assert abs(m1 - m0) / abs(m0) <= 1e-12
        cur, nxt = nxt, cur
    del f, g


# ---------------- host-buffer step: slab-pipelined copies must not change a single bit ----------------------

@pytest.mark.parametrize("name,shape,cfl", [("c2", (16, 2, 1), (1, 1)), ("c2", (12, 1, 2), (3, 1)), ("c0", (5, 2, 1), (1, 2))])
def test_step_host_matches_device(cuda_device, name, shape, cfl):
    """fks_step_host (pinned host buffers, 3-stream slab pipeline with a periodic halo of max|delta_x| planes)
    equals fks_step on device buffers bit for bit, over two consecutive steps (the generic cell advances)."""
    cfg = CONFIGS[name]
    n = shape[0] * shape[1] * shape[2]
    f = inputs.make_f(cfg, device=cuda_device, cells=[i % cfg.n_cells for i in range(n)])
    dev = make(cfg)
    host = make(cfg)
    dev.transport_setup(shape, *cfl)
    host.transport_setup(shape, *cfl)
    a, b = f.clone(), torch.empty_like(f)
    ha = torch.empty(f.shape, dtype=torch.float64, pin_memory=True)
    hb = torch.empty_like(ha, pin_memory=True)
    ha.copy_(f)
    for _ in range(2):
        dev.step(a, b, 0.01)
        B.fks_step_host(host.h, ha, hb, 0.01)
        a, b = b, a
        ha, hb = hb, ha
    torch.cuda.synchronize()
    assert torch.equal(a.cpu(), ha)


@pytest.mark.parametrize("name,shape,cfl,slabs", [("c0", (4, 16, 2), (1, 1), "4"), ("c0", (6, 16, 1), (3, 2), "6"),
                                                   ("c2", (4, 16, 1), (1, 1), "4"), ("c2", (64, 1, 1), (1, 1), "4"),
                                                   ("c2", (48, 1, 1), (3, 1), "3")])
def test_step_host_split_slabs(cuda_device, monkeypatch, name, shape, cfl, slabs):
    """fks_step_host with one-plane slabs whose first and last plane are cut into 4 row blocks (each copied and
    computed as soon as the rows it reads have landed, y-halo of max|delta_y| rows, periodic in y), and with
    multi-plane slabs whose first and last slab give up their outer quarter (>= max|delta_x| planes) as a piece of
    its own (c2-like 1-D boxes, CFL 1 and 3): bit-identical to fks_step over two steps, on the small-N path (c0)
    and the N = 32 fast path (c2 cells, fused gather, chunk pipeline)."""
    monkeypatch.setenv("FKS_HOST_SLABS", slabs)
    test_step_host_matches_device(cuda_device, name, shape, cfl)


def test_step_host_pageable(cuda_device):
    """Pageable host memory takes the same path (copies become synchronous) and gives the same bits."""
    cfg = CONFIGS["c2"]
    shape = (8, 1, 1)
    f = inputs.make_f(cfg, device=cuda_device, cells=list(range(8)))
    dev, host = make(cfg), make(cfg)
    dev.transport_setup(shape, 1, 1)
    host.transport_setup(shape, 1, 1)
    out = torch.empty_like(f)
    dev.step(f, out, 0.02)
    hin = f.cpu().contiguous()
    hout = torch.empty_like(hin)
    B.fks_step_host(host.h, hin, hout, 0.02)
    torch.cuda.synchronize()
    assert torch.equal(out.cpu(), hout)


@pytest.mark.parametrize("name,n", [("c0", 8), ("c2", 1536)])
def test_collision_batch_host_matches_device(cuda_device, name, n):
    """fks_collision_batch_host (pinned host buffers, chunks pipelined over three streams) equals the
    device-resident batch bit for bit (cells are independent; each chunk runs the same kernels)."""
    cfg = CONFIGS[name]
    f = inputs.make_f(cfg, device=cuda_device, cells=[c % cfg.n_cells for c in range(n)])
    col = make(cfg)
    Qd = col.collision_batch(f).cpu()
    fh = f.cpu().pin_memory()
    Qh = torch.empty_like(fh).pin_memory()
    B.fks_collision_batch_host(col.h, fh, Qh, n)
    assert torch.equal(Qh, Qd)
    fp = f.cpu()  # pageable
    Qp = torch.empty_like(fp)
    B.fks_collision_batch_host(col.h, fp, Qp, n)
    assert torch.equal(Qp, Qd)


# ---------------- small-N fast path (N = 16, 24; csrc/small.cu) edge cases ------------------------------------------

def test_small_path_single_cell_and_many_terms(cuda_device):
    """One cell (3 units on a 148-CTA grid) and many terms: Maxwell molecules with 16 radial nodes and 16 directions
    at N = 16 (T + 1 = 257, 16 term chunks summed in order) against the oracle."""
    N = 16
    col = B.Collision(N, L_BOX, 16, 16, 1)
    assert B.fks_get_path(col.h) == B.FKS_PATH_FAST
    f = inputs.random_field(1, N, seed=71, signed=False).to(cuda_device)
    Q = col.collision_batch(f).cpu().numpy()
    ref = oracle_Q(f.cpu().numpy(), oracle_tables(N, L_BOX, 16, 16, 1))
    assert rel_err_per_cell(Q, ref).max() <= TOL_Q


def test_small_path_more_units_than_ctas(cuda_device):
    """c1 velocity grid (N = 24) with 150 cells: 150 x 3 x 16 units over the persistent grid (every CTA runs many
    units, G zeroed per unit); sampled cells against the oracle, and chunking (max_cells_in_flight) is bit-exact."""
    cfg = CONFIGS["c1"]
    f = inputs.random_field(150, cfg.N, seed=5, signed=False).to(cuda_device)
    col = B.Collision(cfg.N, cfg.L, cfg.M, cfg.M_r, cfg.kernel)
    Q = col.collision_batch(f)
    q2 = B.Collision(cfg.N, cfg.L, cfg.M, cfg.M_r, cfg.kernel, max_cells_in_flight=37).collision_batch(f)
    assert torch.equal(Q, q2)
    idx = [0, 1, 77, 149]
    ref = oracle_Q(f[idx].cpu().numpy(), cfg_tables("c1"))
    assert rel_err_per_cell(Q[idx].cpu().numpy(), ref).max() <= TOL_Q


@pytest.mark.parametrize("N,kernel,kw", [(32, 1, {}), (24, 2, {"vhs_alpha": 0.5}), (16, 2, {"vhs_alpha": 0.25}),
                                         (32, 0, {"quad_rule": 1})])
def test_fast_paths_other_kernels_and_rules(cuda_device, N, kernel, kw):
    """Both fast paths are table-driven: Maxwell molecules on the N = 32 kernel, VHS on the small-N kernel (N = 24,
    16) and the paper's rectangle quadrature rule on N = 32, each against the oracle (few directions and radial
    nodes so that the oracle stays fast)."""
    f = inputs.random_field(2, N, seed=90 + N + kernel, signed=False).to(cuda_device)
    col = B.Collision(N, L_BOX, 4, 2, kernel, **kw)
    assert col.info["path"] == B.FKS_PATH_FAST
    Q = col.collision_batch(f).cpu().numpy()
    okw = {}
    if "vhs_alpha" in kw:
        okw["alpha"] = kw["vhs_alpha"]
    if "quad_rule" in kw:
        okw["rule"] = kw["quad_rule"]
    ref = oracle_Q(f.cpu().numpy(), oracle_tables(N, L_BOX, 4, 2, kernel, **okw))
    assert rel_err_per_cell(Q, ref).max() <= TOL_Q
