"""Pins of the plain C++17 CPU oracle (oracle/cpp/fks_oracle.cpp via oracle/cpp_oracle.py), BJ.north_star's
"plain, slow CPU implementation in C++".

Two kinds of checks, as for the numpy oracle:
  * external pins of the C++ code itself — textbook quadrature values, closed forms of the defining integrals,
    the brute-force O(N^6) double sum against the fast form (both evaluated by the C++ code), mass conservation,
    bilinearity, exact translation equivariance, spectral decay of Q(M, M), spectral convergence to the BKW
    ∂f/∂t, and the direction of the transport shift;
  * a cross-check against the independently written numpy oracle (itself pinned in test_oracle_pins*.py) to
    1e-13 on tables, collision (fast, direct, aliased), transport and the full step, for all three kernels.
The C++ library is compiled here by g++ (no CUDA); it shares no code with paper_1701_01608_b200/.
"""
import math

import numpy as np
import pytest
from scipy import integrate

from oracle import cpp_oracle as c
from oracle import fks_oracle as o

L = 13.242640687119286           # (3+√2)R/2 with R = 6
R = 6.0


@pytest.fixture(scope="module", autouse=True)
def _built():
    c.build()


def _two_maxwellian(N, seed):
    v3 = o.velocity_grid3(N, L)
    rng = np.random.default_rng(seed)
    f = np.zeros((N, N, N))
    for _ in range(2):
        f += o.maxwellian(v3, rng.uniform(0.5, 1.5), rng.uniform(-1, 1, 3), rng.uniform(0.5, 1.5))
    f[np.linalg.norm(v3, axis=-1) > R] = 0
    return f


# ---------------- quadratures -------------------------------------------------------------

def test_cpp_gauss_legendre_textbook():
    x, w = c.gauss_legendre(3)
    assert np.allclose(x, [-math.sqrt(0.6), 0, math.sqrt(0.6)], atol=1e-15)
    assert np.allclose(w, [5 / 9, 8 / 9, 5 / 9], atol=1e-15)
    for n in (2, 5, 16, 64):
        x, w = c.gauss_legendre(n)
        for k in range(2 * n):
            exact = 2.0 / (k + 1) if k % 2 == 0 else 0.0
            assert abs(np.sum(w * x ** k) - exact) < 2e-14, (n, k)
    x, w = c.gauss_legendre(16, 0.0, R)
    assert abs(np.sum(w * x ** 3) - R ** 4 / 4) < 1e-12 * R ** 4


@pytest.mark.parametrize("nt,nf", [(4, 4), (8, 4), (8, 8)])
def test_cpp_direction_rules(nt, nf):
    e, w = c.directions(nt, nf)
    assert abs(np.sum(w) - 2 * math.pi) < 1e-13
    assert np.allclose(np.linalg.norm(e, axis=1), 1.0, atol=1e-15)
    assert np.allclose(np.einsum("d,da,db->ab", w, e, e), (2 * math.pi / 3) * np.eye(3), atol=1e-13)
    # paper rectangle rule: closed forms of Σw e_z² and Σw e_x² (see test_P2_paper_rule_second_moments)
    e, w = c.directions(nt, nf, c.QUAD_PAPER_RECT)
    c1, c3 = 1 / math.tan(math.pi / (2 * nt)), 1 / math.tan(3 * math.pi / (2 * nt))
    m = np.einsum("d,da,db->ab", w, e, e)
    assert abs(np.sum(w) - (math.pi ** 2 / nt) * c1) < 1e-12
    assert abs(m[2, 2] - math.pi ** 2 / (4 * nt) * (c1 + c3)) < 1e-12
    assert abs(m[0, 0] - math.pi ** 2 / (8 * nt) * (3 * c1 - c3)) < 1e-12


@pytest.mark.parametrize("s", [0.0, 0.3, 1.7, 6.6])
def test_cpp_phi_psi_against_quadrature(s):
    # φ_R(s) = 2∫_0^R ρ cos(ρ s) dρ (A1);  ψ_R(τ) = ∫_0^π φ_R(τ cos θ) dθ (A2)
    ref, _ = integrate.quad(lambda r: 2 * r * math.cos(r * s), 0, R, epsabs=1e-14, epsrel=1e-14, limit=400)
    assert abs(c.phi_R(np.array([s]), R)[0] - ref) <= 1e-13 * R * R
    inner = lambda th: integrate.quad(lambda r: 2 * r * math.cos(r * s * math.cos(th)), 0, R,
                                      epsabs=1e-14, epsrel=1e-14, limit=400)[0]
    ref, _ = integrate.quad(inner, 0, math.pi, epsabs=1e-13, epsrel=1e-14, limit=400)
    assert abs(c.psi_R(np.array([s]), R)[0] - ref) <= 1e-12 * math.pi * R * R


# ---------------- the collision operator ---------------------------------------------------------------

@pytest.mark.parametrize("N", [4, 6, 8])
@pytest.mark.parametrize("kernel", [c.KERNEL_HARD_SPHERES, c.KERNEL_MAXWELL])
def test_cpp_fast_equals_direct(N, kernel):
    """Eq. CF1 evaluated two ways by the C++ oracle: the zero-padded convolution form
     equals the brute-force double sum for every exact padding P ≥ 3N/2 − 2 (A10)."""
    tb = c.build_tables(N, L, M=16, M_r=4, kernel=kernel)
    rng = np.random.default_rng([1701, N, kernel, 7])
    f = np.ascontiguousarray(2 * rng.random((2, N, N, N)) - 1)
    Qd = c.collision_direct(f, tb)
    scale = np.abs(Qd).max()
    for P in (3 * N // 2, 2 * N, 3 * N // 2 - 2):
        assert np.abs(c.collision_batch(f, tb, P=P) - Qd).max() <= 1e-12 * scale, P
    if N > 4:   # P = N aliases: a different operator (A10)
        assert np.abs(c.collision_batch(f, tb, P=N) - Qd).max() > 1e-6 * scale
        # ... equal to the aliased double sum (pairs l + m = k mod P)
        assert np.abs(c.collision_batch(f, tb, P=N) - c.collision_direct(f, tb, P=N)).max() <= 1e-12 * scale


def test_cpp_mass_realness_bilinearity_translation():
    N = 16
    tb = c.build_tables(N, L, M=16)
    f = np.stack([_two_maxwellian(N, s) for s in range(3)])
    Q, mi = c.collision_batch(f, tb, return_imag=True)
    for i in range(3):
        ql = c.loss_part(f[i], tb)
        assert abs(Q[i].sum()) / np.abs(ql).sum() < 1e-11            # Σ_j Q_j = N³ Q̂_0 = 0 (App. A4)
        assert mi[i] <= 1e-13 * np.abs(Q[i]).max()
    Qp = c.collision_batch(f, tb, project_mass=True)
    assert max(abs(Qp[i].sum()) for i in range(3)) < 1e-14 * np.abs(f).sum()
    assert np.abs(c.collision_batch(3 * f[:1], tb) - 9 * Q[:1]).max() <= 1e-14 * 9 * np.abs(Q[0]).max()
    assert np.abs(c.collision_batch(np.zeros_like(f[:1]), tb)).max() == 0.0
    g = np.ascontiguousarray(np.roll(f[:1], (2, -3, 5), axis=(1, 2, 3)))
    assert np.abs(c.collision_batch(g, tb)[0] - np.roll(Q[0], (2, -3, 5), axis=(0, 1, 2))).max() \
        <= 1e-13 * np.abs(Q[0]).max()


def test_cpp_threads_do_not_change_results():
    N = 8
    tb = c.build_tables(N, L, M=16)
    f = np.random.default_rng(11).random((7, N, N, N))
    assert np.array_equal(c.collision_batch(f, tb, threads=1), c.collision_batch(f, tb, threads=4))


def test_cpp_equilibrium_spectral_decay():
    """Q(M, M) → 0 spectrally for a Maxwellian truncated to the ball of radius R."""
    ratios = []
    for N in (16, 24, 32):
        tb = c.build_tables(N, L, M=16)
        v3 = o.velocity_grid3(N, L)
        f = o.maxwellian(v3, 1.0, (0.3, -0.2, 0.1), 1.0)
        f[np.linalg.norm(v3, axis=-1) > R] = 0
        Q = c.collision_batch(f[None], tb)[0]
        ratios.append(np.abs(Q).max() / np.abs(c.loss_part(f, tb)).max())
    assert ratios[0] > ratios[1] > ratios[2]
    assert ratios[2] < 2e-3


def test_cpp_bkw_spectral_convergence():
    """BKW (Maxwell molecules): Q(f_K) → ∂f/∂t of the closed form as N grows (App. A6); the 1e-6 level needs
    N = 64 (pinned for the numpy oracle, test_P14_bkw_N64_1e6), to which this oracle is cross-checked below."""
    errs = []
    for N in (16, 24, 32):
        v3 = o.velocity_grid3(N, L)
        K = 0.7
        f = o.bkw(v3, K)
        f[np.linalg.norm(v3, axis=-1) > R] = 0
        tb = c.build_tables(N, L, M=4, M_r=8, kernel=c.KERNEL_MAXWELL)
        ex = o.bkw_dfdt(v3, K)
        errs.append(np.abs(c.collision_batch(f[None], tb)[0] - ex).max() / np.abs(ex).max())
    assert errs[0] > errs[1] > errs[2] and errs[2] < 0.1, errs       # measured 0.76, 0.18, 0.079 (2x2 angles)


def test_cpp_transport_direction():
    """f(t+dt, x) = f(t, x − v dt): a particle with v dt = (+1, 0, −1) cells moves that way."""
    N, shape = 8, (5, 3, 4)
    nx, ny, nz = shape
    k = (3 * N // 4, N // 2, N // 4)                     # v = (L/2, 0, −L/2) on v_k = −L + 2Lk/N (A13)
    f = np.zeros((nx * ny * nz, N, N, N))
    f[0][k] = 1.0
    cell = c.GenericCell(N=N, c_num=2, c_den=1)          # dt = 2 dx / L
    cur = f
    for n in range(1, 6):
        cur = c.transport(cur, shape, cell.advance())
        assert np.argwhere(cur[:, k[0], k[1], k[2]] == 1.0).ravel().tolist() == [(n % nx) * ny * nz + (-n) % nz]
        assert cur.sum() == 1.0


# ---------------- cross-check against the numpy oracle ---------------------------------------------------

@pytest.mark.parametrize("kernel", [c.KERNEL_HARD_SPHERES, c.KERNEL_MAXWELL, c.KERNEL_VHS])
def test_cpp_vs_numpy_tables_and_collision(kernel):
    N = 16
    kw = dict(M=16, kernel=kernel)
    tn, tc = o.build_tables(N, L, **kw), c.build_tables(N, L, **kw)
    assert tn.a.shape == tc.a.shape
    assert np.abs(tn.a - tc.a).max() <= 1e-13 * np.abs(tn.a).max()
    assert np.abs(tn.b - tc.b).max() <= 1e-13 * np.abs(tn.b).max()
    f = np.stack([_two_maxwellian(N, 20 + s) for s in range(2)])
    Qc = c.collision_batch(f, tc)
    for i in range(2):
        Qn = o.collision_fast(f[i], tn)
        assert np.abs(Qc[i] - Qn).max() <= 1e-13 * np.abs(Qn).max()


def test_cpp_vs_numpy_variants():
    """Paper quadrature rule, cutoff ratio, VHS exponent, aliased P and the direct sum agree to 1e-13."""
    N = 8
    f = np.random.default_rng(3).random((N, N, N))
    for kw in (dict(rule=o.QUAD_PAPER_RECT), dict(cutoff_ratio=1.5), dict(kernel=o.KERNEL_VHS, alpha=0.3)):
        tn, tc = o.build_tables(N, L, M=16, **kw), c.build_tables(N, L, M=16, **kw)
        Qn = o.collision_fast(f, tn)
        assert np.abs(c.collision_batch(f[None], tc)[0] - Qn).max() <= 1e-13 * np.abs(Qn).max(), kw
    tn, tc = o.build_tables(N, L, M=16), c.build_tables(N, L, M=16)
    for P in (N, N + 2):
        Qn = o.collision_fast(f, tn, P=P)
        assert np.abs(c.collision_batch(f[None], tc, P=P)[0] - Qn).max() <= 1e-13 * np.abs(Qn).max(), P
    Qn = o.collision_direct(f, tn)
    assert np.abs(c.collision_direct(f, tc) - Qn).max() <= 1e-13 * np.abs(Qn).max()


def test_cpp_vs_numpy_transport_and_step():
    N, shape = 8, (3, 2, 2)
    n = 12
    rng = np.random.default_rng(9)
    f = rng.random((n, N, N, N))
    tn, tc = o.build_tables(N, L, M=16), c.build_tables(N, L, M=16)
    cn, cc = o.GenericCell(N=N, c_num=3, c_den=2), c.GenericCell(N=N, c_num=3, c_den=2)
    for _ in range(3):
        dn, dc = cn.advance(), cc.advance()
        assert np.array_equal(dn, dc)
        assert np.array_equal(o.transport(f, shape, dn), c.transport(f, shape, dc))
    fn = o.fks_step(f, shape, cn, tn, 0.05)
    fc = c.fks_step(f, shape, cc, tc, 0.05)
    assert np.abs(fn - fc).max() <= 1e-13 * np.abs(fn).max()
