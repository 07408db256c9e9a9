"""Pins of the oracle's macroscopic moments and BGK operator (DESIGN.md §6 P18-P23).

Closed forms (moments of a Maxwellian), the paper's own alternative formula for the moments after transport
(Eq. DM_update), and invariants of the BGK operator (vanishing at equilibrium, conservation, entropy decay).
"""
import math

import numpy as np

from oracle import fks_oracle as o

L = 13.242640687119286  # (3+√2)R/2 with R = 6 (A8)


def _alias_tol(N, T):
    """Error bound of the node sum for Gaussian moments up to |v|²: the first aliased Fourier mode of
    e^{-v²/2T} on the node spacing h = 2L/N is e^{-2π²T/h²}, times (2π/h)² for the |v|² weight (×10 margin)."""
    h = 2 * L / N
    return max(1e-13, 10 * (2 * math.pi / h) ** 2 * math.exp(-2 * math.pi ** 2 * T / h ** 2))


def _closed_form_U(rho, u, T):
    """(ρ, ρu, E) of ρ(2πT)^{-3/2}e^{-|v-u|²/2T}: E = ρ|u|²/2 + 3ρT/2."""
    u = np.asarray(u, dtype=np.float64)
    return np.array([rho, *(rho * u), 0.5 * rho * (u @ u) + 1.5 * rho * T])


def test_P18_moments_of_maxwellian_closed_form():
    # the trapezoid rule on [-L, L)^3 is spectrally accurate for a Gaussian well inside the box:
    # error ~ exp(-2π²T/h²) ≈ 3e-13 at N = 32 (h = 2L/N); ≈ 8e-8 at N = 24
    v3 = o.velocity_grid3(32, L)
    for rho, u, T in [(1.0, (0, 0, 0), 1.0), (1.3, (0.3, -0.2, 0.45), 1.1), (0.125, (-0.7, 0.1, 0.25), 0.8)]:
        U = o.moments(o.maxwellian(v3, rho, u, T), 32, L)
        ex = _closed_form_U(rho, u, T)
        assert np.abs(U - ex).max() <= _alias_tol(32, T) * np.abs(ex).max(), (U, ex)
    v3 = o.velocity_grid3(24, L)
    U = o.moments(o.maxwellian(v3, 1.0, (0.2, 0.3, -0.1), 1.2), 24, L)
    ex = _closed_form_U(1.0, (0.2, 0.3, -0.1), 1.2)
    assert np.abs(U - ex).max() <= _alias_tol(24, 1.2) * np.abs(ex).max()
    # linearity over a batch: two cells of a two-Maxwellian mixture
    v3 = o.velocity_grid3(32, L)
    f = np.stack([o.maxwellian(v3, 1.0, (0.5, 0, 0), 1.0) + o.maxwellian(v3, 0.5, (-0.5, 0.2, 0), 0.7),
                  o.maxwellian(v3, 2.0, (0, 0, 0.3), 1.4)])
    U = o.moments(f, 32, L)
    ex = np.stack([_closed_form_U(1.0, (0.5, 0, 0), 1.0) + _closed_form_U(0.5, (-0.5, 0.2, 0), 0.7),
                   _closed_form_U(2.0, (0, 0, 0.3), 1.4)])
    assert U.shape == (2, 5) and np.abs(U - ex).max() <= _alias_tol(32, 0.7) * np.abs(ex).max()


def test_P19_primitive_of_closed_form():
    for rho, u, T in [(1.0, (0, 0, 0), 1.0), (0.3, (1.5, -2.0, 0.25), 4.0), (7.0, (0.01, 0.02, -0.03), 0.05)]:
        W = o.primitive(_closed_form_U(rho, u, T))
        assert np.allclose(W, [rho, *u, T], rtol=1e-14, atol=1e-15)


def test_P20_DM_update_equals_moments_of_transported_f():
    # the paper's incremental formula (particles leaving / entering, Eq. DM_update) must give the
    # moments of the transported distribution (transport is a per-velocity permutation of cells)
    rng = np.random.default_rng(20)
    N, shape = 6, (3, 2, 2)
    Lb = 3.0
    f = rng.random((12, N, N, N))
    cell = o.GenericCell(N, 3, 2)  # CFL 3/2: shifts of 0, ±1, ±2 cells
    for _ in range(2):
        delta = cell.advance()
        U1 = o.moments_update(o.moments(f, N, Lb), f, shape, delta, N, Lb)
        fs = o.transport(f, shape, delta)
        U2 = o.moments(fs, N, Lb)
        assert np.abs(U1 - U2).max() <= 1e-13 * np.abs(U2).max()
        # total (ρ, ρu, E) over the periodic box is invariant under transport
        assert np.allclose(U2.sum(axis=0), o.moments(f, N, Lb).sum(axis=0), rtol=1e-13, atol=1e-13)
        f = fs


def test_P21_bgk_vanishes_at_equilibrium():
    v3 = o.velocity_grid3(32, L)
    nu = 10.0  # τ = 0.1 of the paper's Sod runs
    for rho, u, T in [(1.0, (0, 0, 0), 5.0 / 5), (0.125, (0.3, 0, -0.1), 0.8), (1.0, (0.1, 0.2, 0.3), 1.5)]:
        M = o.maxwellian(v3, rho, u, T)
        assert np.abs(o.bgk(M, 32, L, nu)).max() <= _alias_tol(32, T) * nu * M.max()


def test_P22_bgk_conserves_mass_momentum_energy():
    v3 = o.velocity_grid3(32, L)
    f = o.maxwellian(v3, 1.0, (0.8, 0, 0), 0.9) + o.maxwellian(v3, 0.6, (-0.6, 0.3, 0.1), 1.2)
    nu = 10.0
    Uq = o.moments(o.bgk(f, 32, L, nu), 32, L)
    Uf = o.moments(f, 32, L)
    assert np.abs(Uq).max() <= _alias_tol(32, 0.9) * nu * np.abs(Uf).max()
    # and it is far from equilibrium, so the test is not vacuous
    assert np.abs(o.bgk(f, 32, L, nu)).max() > 1e-2 * nu * f.max()


def test_P23_bgk_relaxation_decreases_entropy_and_keeps_positivity():
    v3 = o.velocity_grid3(32, L)
    f = o.maxwellian(v3, 1.0, (1.0, 0, 0), 1.0) + o.maxwellian(v3, 1.0, (-1.0, 0, 0), 1.0)
    f = np.where(f > 1e-300, f, 1e-300)
    H = lambda g: float(np.sum(g * np.log(g)))  # noqa: E731  Boltzmann H functional (discrete)
    cell = o.GenericCell(32, 0, 1)  # identity transport: a space-homogeneous relaxation
    g = f[None]
    Hs = [H(g[0])]
    for _ in range(3):
        g = o.bgk_step(g, (1, 1, 1), cell, 0.5, L)
        assert g.min() > 0  # convex combination of f* > 0 and E > 0 for 0 < νΔt ≤ 1
        Hs.append(H(g[0]))
    assert all(b < a for a, b in zip(Hs, Hs[1:]))
    # νΔt = 1 relaxes in one step onto the Maxwellian with the same (ρ, u, T): closed form of the moments
    g1 = o.bgk_step(f[None], (1, 1, 1), o.GenericCell(32, 0, 1), 1.0, L)[0]
    W = o.primitive(o.moments(g1, 32, L))
    # mixing ±u0: ρ = 2, u = 0, (3/2)ρT = Σ(ρ_i u0²/2 + 3ρ_i T0/2)  =>  T = T0 + u0²/3
    assert np.allclose(W, [2.0, 0, 0, 0, 1.0 + 1.0 / 3.0], rtol=_alias_tol(32, 1.0), atol=_alias_tol(32, 1.0))


def test_bgk_degenerate_cells():
    # reading A26: no Maxwellian for ρ ≤ 0 or T ≤ 0 -> E = 0, so Q_BGK = -ν f
    N = 8
    z = np.zeros((N, N, N))
    assert np.array_equal(o.bgk(z, N, 4.0, 3.0), z)
    spike = np.zeros((N, N, N))
    spike[4, 4, 4] = 1.0  # a single particle at v = 0: ρ > 0, T = 0
    assert np.array_equal(o.bgk(spike, N, 4.0, 3.0), -3.0 * spike)
    neg = -np.ones((N, N, N))  # ρ < 0
    assert np.array_equal(o.bgk(neg, N, 4.0, 2.0), -2.0 * neg)
