"""Pins of the variable-hard-sphere kernel tables (DESIGN.md §6 P25-P26; reading A30):
B = C_α|u|^α through the radial split with B~(ρ, ρ') = 4C_α(ρ²+ρ'²)^{(α−1)/2}.  The two ends of the family
are the independently written kernels (α = 0: Maxwell molecules; α = 1, C = 1/4: the closed-form hard-sphere
tables), and the loss rate of a Maxwellian has a closed form for every α."""
import math

import numpy as np
import pytest
from scipy import special

from oracle import fks_oracle as o

L = 13.242640687119286
R = 6.0


def test_P25_vhs_alpha0_is_maxwell_molecules():
    mm = o.build_tables(12, L, M=16, M_r=8, kernel=o.KERNEL_MAXWELL)
    v0 = o.build_tables(12, L, M=16, M_r=8, kernel=o.KERNEL_VHS, alpha=0.0)
    assert np.array_equal(mm.a, v0.a)
    assert np.abs(mm.b - v0.b).max() <= 1e-14 * np.abs(mm.b).max()


def test_P25_vhs_alpha1_is_hard_spheres():
    # B~ = 4 C_1 = 1: the radial split of the closed-form φ_R, ψ_R (A1, A2); Gauss-Legendre in ρ is exact enough
    # that the collision operators agree to rounding
    N = 12
    hs = o.build_tables(N, L, M=16, kernel=o.KERNEL_HARD_SPHERES)
    v1 = o.build_tables(N, L, M=16, M_r=16, kernel=o.KERNEL_VHS, alpha=1.0, C_alpha=0.25)
    assert np.abs(hs.b[0] - v1.b[0]).max() <= 1e-13 * np.abs(hs.b[0]).max()  # B̂_F(m, m)
    f = np.random.default_rng(3).random((N, N, N))
    qh, qv = o.collision_fast(f, hs), o.collision_fast(f, v1)
    assert np.abs(qh - qv).max() <= 1e-11 * np.abs(qh).max()


@pytest.mark.parametrize("alpha", [0.25, 0.5, 0.75])
def test_P26_vhs_loss_rate_closed_form(alpha):
    # ν = ∫ f(v*) ∫_{S²} B dω dv* at v = u for a Maxwellian (ρ, T): 4π C_α ρ E|W|^α, W ~ N(0, T I₃),
    # E|W|^α = (2T)^{α/2} Γ((3+α)/2)/Γ(3/2); α = 1, C = 1/4 gives ρ√(8πT) (P13), α = 0 gives ρ
    N, T = 24, 1.0
    tb = o.build_tables(N, L, M=64, M_r=16, kernel=o.KERNEL_VHS, alpha=alpha)
    v3 = o.velocity_grid3(N, L)
    f = o.maxwellian(v3, 1.0, (0, 0, 0), T)
    f[np.linalg.norm(v3, axis=-1) > R] = 0
    i = N // 2
    nu = o.loss_part(f, tb)[i, i, i] / f[i, i, i]
    ex = 4 * math.pi * o.VHS_C_DEFAULT * (2 * T) ** (alpha / 2) * special.gamma((3 + alpha) / 2) / special.gamma(1.5)
    assert abs(nu / ex - 1) < 1e-3, (nu, ex)
    assert abs(4 * math.pi * 0.25 * (2 * T) ** 0.5 * special.gamma(2) / special.gamma(1.5) - math.sqrt(8 * math.pi * T)) < 1e-14
