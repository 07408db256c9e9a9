"""GPU parity of the macroscopic moments and the BGK operator / step against the
CPU oracle, through the C ABI, on the same seeded inputs.

Tolerances (derived in DESIGN.md §6): moments per component ≤ 1e-13 · Σ_k |φ(v_k)| |f_k| Δv³ (summation order
only); BGK per cell ≤ 1e-12 · ν · max(max|E|, max|f|) (moments' rounding amplified by the exponent |v−u|²/2T and
the separable product of three exponentials); transport part bit-exact.
"""
import numpy as np
import pytest
import torch

from oracle import fks_oracle as o
from paper_1701_01608_b200 import binding as B
from paper_1701_01608_b200 import inputs
from paper_1701_01608_b200.configs import CONFIGS, L_BOX

pytestmark = pytest.mark.gpu

TOL_U = 1e-13
TOL_BGK = 1e-12


def _phi_abs_scale(f, N, L):
    """Σ_k |φ_a(v_k)| |f_k| Δv³ per cell and component: the scale of the summation rounding."""
    phi = np.abs(o.collision_invariants(N, L))
    fa = np.abs(f.reshape(-1, N, N, N))
    return np.stack([[np.sum(phi[a] * fc) for a in range(5)] for fc in fa]) * (2 * L / N) ** 3


def _check_moments(f_host, U, W, N, L):
    Uo = o.moments(f_host.reshape(-1, N, N, N), N, L).reshape(-1, 5)
    scale = _phi_abs_scale(f_host, N, L)
    assert np.all(np.abs(U - Uo) <= TOL_U * scale + 1e-300), np.abs(U - Uo).max()
    Wo = o.primitive(Uo)
    ok = Uo[:, 0] > 0
    assert np.allclose(W[ok], Wo[ok], rtol=1e-11, atol=1e-13)


def _random_two_maxwellian(n, N, L, seed):
    rng = np.random.default_rng(seed)
    v3 = o.velocity_grid3(N, L)
    f = np.zeros((n, N, N, N))
    for c in range(n):
        for _ in range(2):
            f[c] += o.maxwellian(v3, rng.uniform(0.5, 1.5), rng.uniform(-1, 1, 3), rng.uniform(0.6, 1.5))
    return f


def _check_bgk(Q, Qo, f, nu):
    n = f.shape[0]
    E = Qo / nu + f
    scale = nu * np.maximum(np.abs(E).reshape(n, -1).max(1), np.abs(f).reshape(n, -1).max(1))
    err = np.abs(Q - Qo).reshape(n, -1).max(1)
    assert np.all(err <= TOL_BGK * scale), (err / scale).max()


@pytest.mark.parametrize("N,n", [(4, 3), (6, 5), (16, 9), (24, 4), (32, 6), (48, 2), (64, 1)])
def test_moments_random(cuda_device, N, n):
    # N = 6: ragged tail (216 points, one CTA); 24: 2-CTA clusters; 48: 7 CTAs of 128 KB; 64: 16-CTA cluster
    col = B.Collision(N, L_BOX, 16, 16, 0)
    f = _random_two_maxwellian(n, N, L_BOX, 100 + N)
    fd = torch.as_tensor(f, device=cuda_device)
    U, W = col.moments(fd)
    torch.cuda.synchronize()
    _check_moments(f, U.cpu().numpy(), W.cpu().numpy(), N, L_BOX)


@pytest.mark.parametrize("name", ["c0", "c2"])
def test_moments_config(cuda_device, name):
    cfg = CONFIGS[name]
    cells = list(range(min(cfg.n_cells, 64)))
    f = inputs.make_f(cfg, device=cuda_device, cells=cells)
    col = B.Collision(cfg.N, cfg.L, cfg.M, cfg.M_r, cfg.kernel)
    U, W = col.moments(f)
    torch.cuda.synchronize()
    _check_moments(f.cpu().numpy(), U.cpu().numpy(), W.cpu().numpy(), cfg.N, cfg.L)


@pytest.mark.parametrize("N,n", [(6, 4), (16, 8), (24, 3), (32, 5), (48, 1)])
def test_bgk_batch_random(cuda_device, N, n):
    nu = 10.0  # τ = 0.1
    col = B.Collision(N, L_BOX, 16, 16, 0)
    f = _random_two_maxwellian(n, N, L_BOX, 200 + N)
    Q = col.bgk_batch(torch.as_tensor(f, device=cuda_device), nu)
    torch.cuda.synchronize()
    _check_bgk(Q.cpu().numpy(), o.bgk(f, N, L_BOX, nu), f, nu)


def test_bgk_edge_cases(cuda_device):
    N, Lb, nu = 8, 4.0, 3.0
    col = B.Collision(N, Lb, 16, 16, 0)
    f = np.zeros((4, N, N, N))
    f[1, 4, 4, 4] = 1.0                       # one particle at v = 0: T = 0 exactly -> E = 0
    f[2] = -1.0                               # rho < 0 -> E = 0
    f[3] = _random_two_maxwellian(1, N, Lb, 3)[0]
    Q = col.bgk_batch(torch.as_tensor(f, device=cuda_device), nu).cpu().numpy()
    assert np.array_equal(Q[0], np.zeros((N, N, N)))
    assert np.array_equal(Q[1], -nu * f[1]) and np.array_equal(Q[2], -nu * f[2])
    _check_bgk(Q[3:], o.bgk(f[3:], N, Lb, nu), f[3:], nu)
    # n_cells = 0 is a no-op; U and W both NULL is an error
    B.fks_bgk_batch(col.h, torch.zeros(1, N, N, N, device=cuda_device, dtype=torch.float64),
                    torch.zeros(1, N, N, N, device=cuda_device, dtype=torch.float64), nu, 0)
    with pytest.raises(B.FksError):
        B.fks_moments(col.h, torch.zeros(1, N, N, N, device=cuda_device, dtype=torch.float64), None, None, 1)
    # a misaligned (8-byte offset) input takes the element-wise staging path and gives the same numbers
    buf = torch.zeros(4 * N ** 3 + 1, dtype=torch.float64, device=cuda_device)
    fm = buf[1:].view(4, N, N, N)
    fm.copy_(torch.as_tensor(f, device=cuda_device))
    Qm = col.bgk_batch(fm, nu).cpu().numpy()
    assert np.array_equal(Qm, Q)


@pytest.mark.parametrize("name,shape,cfl", [("c0", (2, 2, 2), (1, 1)), ("c2", (16, 1, 1), (3, 2)),
                                            ("c2", (4, 3, 2), (1, 1))])
def test_bgk_step_with_transport(cuda_device, name, shape, cfl):
    cfg = CONFIGS[name]
    n = shape[0] * shape[1] * shape[2]
    f = inputs.make_f(cfg, device=cuda_device, cells=list(range(n)))
    col = B.Collision(cfg.N, cfg.L, cfg.M, cfg.M_r, cfg.kernel)
    col.transport_setup(shape, *cfl)
    cell = o.GenericCell(cfg.N, *cfl)     # advanced by o.bgk_step
    shadow = o.GenericCell(cfg.N, *cfl)   # the same bookkeeping, for the transported f* of each step
    nu_dt = 0.3
    fh = f.cpu().numpy()
    out = torch.empty_like(f)
    U = torch.empty((n, 5), dtype=torch.float64, device=cuda_device)
    W = torch.empty_like(U)
    for step in range(2):
        col.bgk_step(f, out, nu_dt, U, W)
        torch.cuda.synchronize()
        ref = o.bgk_step(fh, shape, cell, nu_dt, cfg.L)
        delta = shadow.advance()
        assert np.array_equal(col.last_shift(), delta)
        fs = o.transport(fh, shape, delta)
        _check_moments(fs, U.cpu().numpy(), W.cpu().numpy(), cfg.N, cfg.L)
        _check_bgk((out.cpu().numpy() - fs) / nu_dt, (ref - fs) / nu_dt, fs, 1.0)
        fh = ref
        f, out = out, f


def test_bgk_step_identity_matches_batch(cuda_device):
    # cfl_num = 0: transport is the identity and the step is f + νΔt·Q_BGK(f) with Q from fks_bgk_batch
    cfg = CONFIGS["c2"]
    f = inputs.make_f(cfg, device=cuda_device, cells=list(range(8)))
    col = B.Collision(cfg.N, cfg.L, cfg.M, cfg.M_r, cfg.kernel)
    col.transport_setup((8, 1, 1), 0, 1)
    out = torch.empty_like(f)
    col.bgk_step(f, out, 0.25)
    Q = col.bgk_batch(f, 1.0)
    torch.cuda.synchronize()
    d = (out - f - 0.25 * Q).abs().max().item()
    assert d <= 1e-15 * f.abs().max().item()


def test_bgk_step_c3_full_size_sampled(cuda_device):
    # the launch configuration bench.py --workload bgk times: the whole c3 box (32^3 cells x 32^3), sampled cells
    cfg = CONFIGS["c3"]
    f = inputs.make_f(cfg, device=cuda_device)
    out = torch.empty_like(f)
    n = cfg.n_cells
    U = torch.empty((n, 5), dtype=torch.float64, device=cuda_device)
    col = B.Collision(cfg.N, cfg.L, cfg.M, cfg.M_r, cfg.kernel)
    col.transport_setup(cfg.shape, cfg.cfl_num, cfg.cfl_den)
    nu_dt = 10.0 * cfg.cfl_num / cfg.cfl_den / cfg.shape[0] / cfg.L  # ν = 10, Δt = c·Δx/L
    col.bgk_step(f, out, nu_dt, U, None)
    torch.cuda.synchronize()
    delta = col.last_shift().astype(np.int64)
    N3 = cfg.N ** 3
    flat = f.view(n, N3)
    for j in [0, 1, 777, 16383, 20000, n - 1]:
        src = torch.as_tensor(o.source_cells(j, cfg.shape, delta).reshape(-1), device=cuda_device)
        fs = flat[src, torch.arange(N3, device=cuda_device)].cpu().numpy().reshape(1, cfg.N, cfg.N, cfg.N)
        ref = fs + nu_dt * (o.local_maxwellian(fs, cfg.N, cfg.L) - fs)
        got = out[j:j + 1].cpu().numpy()
        _check_bgk((got - fs) / nu_dt, (ref - fs) / nu_dt, fs, 1.0)
        Uo = o.moments(fs[0], cfg.N, cfg.L)
        assert np.all(np.abs(U[j].cpu().numpy() - Uo) <= TOL_U * _phi_abs_scale(fs, cfg.N, cfg.L)[0])
    # mass over the periodic box: transport permutes, relaxation changes it only by the quadrature error of E
    m_in, m_out = f.sum().item(), out.sum().item()
    assert abs(m_out - m_in) <= 1e-6 * abs(m_in)


def test_abi_rejects_invalid_arguments(cuda_device):
    """Validation errors of the moments / BGK / slab entry points return before any launch (fks.h conventions)."""
    import ctypes
    lib = B.load_library()
    N = 8
    col = B.Collision(N, 4.0, 16, 16, 0)
    f = torch.rand(3, N, N, N, dtype=torch.float64, device=cuda_device)
    g = torch.empty_like(f)
    U = torch.empty(3, 5, dtype=torch.float64, device=cuda_device)
    h = col.h
    ST = lambda fn, *a: fn(*a)  # noqa: E731
    inv, state = B.FKS_ERR_INVALID, B.FKS_ERR_STATE
    # NULL handle
    assert ST(lib.fks_moments, None, f.data_ptr(), U.data_ptr(), None, 3, None) == inv
    assert ST(lib.fks_bgk_batch, None, f.data_ptr(), g.data_ptr(), 1.0, 3, None) == inv
    # moments: both outputs NULL, negative count, host pointer, output overlapping the input
    assert ST(lib.fks_moments, h, f.data_ptr(), None, None, 3, None) == inv
    assert ST(lib.fks_moments, h, f.data_ptr(), U.data_ptr(), None, -1, None) == inv
    fh = torch.zeros(3, N, N, N, dtype=torch.float64)
    assert ST(lib.fks_moments, h, fh.data_ptr(), U.data_ptr(), None, 3, None) == inv
    assert ST(lib.fks_moments, h, f.data_ptr(), f.data_ptr(), None, 3, None) == inv
    # BGK operator: overlap, non-finite nu
    assert ST(lib.fks_bgk_batch, h, f.data_ptr(), f.data_ptr(), 1.0, 3, None) == inv
    assert ST(lib.fks_bgk_batch, h, f.data_ptr(), g.data_ptr(), float("nan"), 3, None) == inv
    # BGK step before any transport setup; slab calls on a single-domain handle
    assert ST(lib.fks_bgk_step, h, f.data_ptr(), g.data_ptr(), 0.1, None, None, None) == state
    H = ctypes.c_int()
    assert ST(lib.fks_slab_halo, h, ctypes.byref(H)) == state
    col.transport_setup((3, 1, 1), 1, 1)
    assert ST(lib.fks_bgk_step, h, f.data_ptr(), f.data_ptr(), 0.1, None, None, None) == inv
    planes = (ctypes.c_void_p * 8)()
    assert ST(lib.fks_step_slab, h, planes, g.data_ptr(), 0.01, None) == state
    # slab setup: invalid ranges; then the single-domain step is refused and a NULL plane is rejected
    assert ST(lib.fks_transport_setup_slab, h, 4, 1, 1, -1, 2, 1, 1) == inv
    assert ST(lib.fks_transport_setup_slab, h, 4, 1, 1, 0, 0, 1, 1) == inv
    assert ST(lib.fks_transport_setup_slab, h, 4, 1, 1, 0, 2, 1, 1) == B.FKS_OK
    assert ST(lib.fks_bgk_step, h, f.data_ptr(), g.data_ptr(), 0.1, None, None, None) == state
    assert ST(lib.fks_step_slab, h, None, g.data_ptr(), 0.01, None) == inv
    assert ST(lib.fks_step_slab, h, planes, g.data_ptr(), 0.01, None) == inv  # NULL entries
    # the handle still works after all the rejected calls
    col.transport_setup((3, 1, 1), 1, 1)
    col.bgk_step(f, g, 0.1)
    B.fks_sync(h)


# ---------------- NEXT-1: moments fused into the fks_step epilogue (fks_step_moments) ------------------------------

@pytest.mark.parametrize("N,shape,cfl,path", [(32, (4, 3, 2), (1, 1), B.FKS_PATH_AUTO),     # fast path, fused gather
                                               (32, (2, 2, 2), (0, 1), B.FKS_PATH_AUTO),     # fast path, no transport
                                               (24, (3, 2, 2), (1, 2), B.FKS_PATH_AUTO),     # small-N path
                                               (16, (3, 2, 1), (2, 1), B.FKS_PATH_GENERIC)])  # generic path
def test_step_moments(cuda_device, N, shape, cfl, path):
    """fks_step_moments: f_out bit-identical to fks_step's (two handles, same inputs and generic-cell history, two
    consecutive steps), U and W of f_out against the oracle's moments of the same f_out (Eq. DM_update P:464-493:
    the per-step moments of the new state) and against fks_moments(f_out)."""
    n = int(np.prod(shape))
    f = torch.as_tensor(_random_two_maxwellian(n, N, L_BOX, 300 + N), device=cuda_device)
    a = B.Collision(N, L_BOX, 16, 16, 0, path=path)
    b = B.Collision(N, L_BOX, 16, 16, 0, path=path)
    a.transport_setup(shape, *cfl)
    b.transport_setup(shape, *cfl)
    s = 0.05
    cur = f
    for _ in range(2):
        out_a, out_b = torch.empty_like(cur), torch.empty_like(cur)
        a.step(cur, out_a, s)
        U, W = b.step_moments(cur, out_b, s)
        torch.cuda.synchronize()
        assert torch.equal(out_a, out_b)
        fo = out_b.cpu().numpy()
        _check_moments(fo, U.cpu().numpy(), W.cpu().numpy(), N, L_BOX)
        Um, Wm = b.moments(out_b)
        torch.cuda.synchronize()
        assert np.all(np.abs(U.cpu().numpy() - Um.cpu().numpy()) <= TOL_U * _phi_abs_scale(fo, N, L_BOX))
        cur = out_b


def test_step_moments_c3_bench_cells(cuda_device):
    """At the bench configuration's velocity grid (c3: N = 32, M = 32, CFL 1, fused gather) on a 4 x 4 x 2 box:
    the moments of the new state, and the collision's conservation (mass of every cell's increment ~ 0, so the box
    mass in U equals the transported input's mass)."""
    cfg = CONFIGS["c3"]
    shape = (4, 4, 2)
    f = inputs.make_f(cfg, device=cuda_device, cells=list(range(32)))
    col = B.Collision(cfg.N, cfg.L, cfg.M, cfg.M_r, cfg.kernel)
    col.transport_setup(shape, cfg.cfl_num, cfg.cfl_den)
    out = torch.empty_like(f)
    U, W = col.step_moments(f, out, cfg.coll_scale)
    torch.cuda.synchronize()
    fo = out.cpu().numpy()
    _check_moments(fo, U.cpu().numpy(), W.cpu().numpy(), cfg.N, cfg.L)
    Uin = o.moments(f.cpu().numpy(), cfg.N, cfg.L)
    assert abs(U[:, 0].sum().item() - Uin[:, 0].sum()) <= 1e-12 * Uin[:, 0].sum()


def test_step_moments_argument_checks(cuda_device):
    col = B.Collision(16, L_BOX, 16, 16, 0)
    col.transport_setup((2, 1, 1), 1, 1)
    f = torch.rand(2, 16, 16, 16, dtype=torch.float64, device=cuda_device)
    out = torch.empty_like(f)
    with pytest.raises(B.FksError) as ei:
        B.fks_step_moments(col.h, f, out, 0.1, None, None)
    assert ei.value.status == B.FKS_ERR_INVALID
    with pytest.raises(B.FksError) as ei:   # U overlapping f_out
        B.fks_step_moments(col.h, f, out, 0.1, out, None)
    assert ei.value.status == B.FKS_ERR_INVALID


@pytest.mark.parametrize("sub", [None, "3"])
def test_step_moments_chunked(cuda_device, monkeypatch, sub):
    """fks_step_moments when the step runs in several workspace chunks (max_cells_in_flight): the moment rows of
    every chunk land at their cells' offsets (fast path, fused gather; chunk pipeline, also with its side-stream
    transforms over sub-ranges of 3 cells, FKS_PIPE_SUB)."""
    if sub is not None:
        monkeypatch.setenv("FKS_PIPE_SUB", sub)
    N, shape = 32, (5, 2, 2)
    n = int(np.prod(shape))
    f = torch.as_tensor(_random_two_maxwellian(n, N, L_BOX, 404), device=cuda_device)
    a = B.Collision(N, L_BOX, 16, 16, 0)
    b = B.Collision(N, L_BOX, 16, 16, 0, max_cells_in_flight=7)
    for col in (a, b):
        col.transport_setup(shape, 1, 1)
    oa, ob = torch.empty_like(f), torch.empty_like(f)
    Ua, Wa = a.step_moments(f, oa, 0.05)
    Ub, Wb = b.step_moments(f, ob, 0.05)
    torch.cuda.synchronize()
    assert torch.equal(oa, ob)
    fo = ob.cpu().numpy()
    _check_moments(fo, Ub.cpu().numpy(), Wb.cpu().numpy(), N, L_BOX)
    assert np.abs(Ua.cpu().numpy() - Ub.cpu().numpy()).max() <= TOL_U * _phi_abs_scale(fo, N, L_BOX).max()
