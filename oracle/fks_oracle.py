"""CPU ORACLE for the FKS fast-spectral Boltzmann hot path (arXiv 1701.01608) — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` / ``--impl reference``
leg may import or call this module.  The product path (``paper_1701_01608_b200``) never imports it and
shares no code with it: this file has its own grid, its own quadrature, its own weight tables (scipy
Bessel functions, numpy Gauss-Legendre) and its own naive per-axis DFTs (explicit DFT matrices, no FFT).

Everything is fp64, plain and slow, written in the paper's order and notation.  Citations:
``P:n`` = line n of PAPER.md (Appendix A "Boltzmann collision operator" is P:1469-1632; the FKS scheme is
§2.1), ``A<n>`` = the readings of garbled / silent passages listed in DESIGN.md §3 (taken from
SURVEY.md §8(c)).

What is computed:

  f̂_l   = N^-3 Σ_j f_j e^{-2πi l·j/N},  l ∈ K'^3, K' = {-(N/2-1)..N/2-1}          (A9, A14)
  Q̂_k   = Σ_{l,m∈K', l+m=k} β̂(l,m) f̂_l f̂_m,  β̂(l,m) = Σ_{t=0}^{T} a_t(l) b_t(m)        (Eq. CF1)
  Q_j   = Σ_{k∈K'} Q̂_k e^{2πi k·j/N}

with the separated ("A convolutions") Carleman weights a_t, b_t of P:1589-1632 and the loss term t = 0
(a_0 = 1, b_0 = -Σ_{t≥1} a_t b_t = -B̂_F(m,m)).  ``collision_fast`` evaluates this with zero-padded
(P = 3N/2) pruned transforms — the paper's convolution algorithm; ``collision_direct`` is the double sum.

Pinned by tests/test_oracle_pins.py (P1-P16 of DESIGN.md §6).  No function here is "parity unpinned".
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
from scipy import special

# ---------------------------------------------------------------------------------------------------
# Geometry
# ---------------------------------------------------------------------------------------------------

#: λ = 2/(3+√2): support radius R = λ·T for the periodised box [-T,T]^3.
LAMBDA = 2.0 / (3.0 + math.sqrt(2.0))

KERNEL_HARD_SPHERES = 0  # B~ ≡ 1 (A4)
KERNEL_MAXWELL = 1       # B~ = (1/π)(|x|²+|y|²)^{-1/2} (Eq. Btilde_pl with α=0; A5)
KERNEL_VHS = 2           # B = C_α|u|^α, 0 ≤ α ≤ 1: B~ = 4C_α(|x|²+|y|²)^{-(1-α)/2} (A30)
VHS_C_DEFAULT = 1.0 / (4.0 * math.pi)  # C_α default: α = 0 is the Maxwell-molecule normalisation (A5)

QUAD_GL_UNIFORM = 0      # Gauss-Legendre in cos θ × uniform φ on the half sphere (A11, A12)
QUAD_PAPER_RECT = 1      # (θ_p, φ_q) = (pπ/A1, qπ/A2), weight π²/(A1A2)·sin θ_p (A2)


def support_radius(L: float) -> float:
    """R = λL: f is supported in B_R and the box is [-L, L)^3 with L = (3+√2)R/2 (A8)."""
    return LAMBDA * L


def kprime(N: int) -> np.ndarray:
    """Retained modes per axis, K' = {-(N/2-1), ..., N/2-1}; the Nyquist mode is dropped (A9)."""
    if N % 2 or N < 4:
        raise ValueError("N must be even and >= 4")
    return np.arange(-(N // 2 - 1), N // 2)


def velocity_nodes(N: int, L: float) -> np.ndarray:
    """Node-centred velocity grid v_j = -L + j·2L/N, j = 0..N-1 (A13)."""
    return -L + np.arange(N) * (2.0 * L / N)


def wavenumbers(N: int, L: float) -> np.ndarray:
    """ξ_l = (π/L)·l for l ∈ K' (the physical frequency of mode l on the box [-L, L))."""
    return (math.pi / L) * kprime(N)


# ---------------------------------------------------------------------------------------------------
# Quadratures (readings A2, A6, A11, A12)
# ---------------------------------------------------------------------------------------------------

def gauss_legendre(n: int, a: float = -1.0, b: float = 1.0):
    """n-point Gauss-Legendre nodes/weights on [a, b] (library routine numpy.polynomial.legendre)."""
    x, w = np.polynomial.legendre.leggauss(n)
    return 0.5 * (b - a) * x + 0.5 * (b + a), 0.5 * (b - a) * w


def split_angles(M: int):
    """M directions → (n_θ, n_φ) = (2^⌈log2(M)/2⌉, M/n_θ): 16→(4,4), 32→(8,4), 64→(8,8) (A12)."""
    n_theta = 2 ** math.ceil(math.log2(M) / 2)
    if M % n_theta:
        n_theta = M
    return n_theta, M // n_theta


def directions(n_theta: int, n_phi: int, rule: int = QUAD_GL_UNIFORM):
    """Unit directions e_d on the half sphere and weights w_d (Σ_d w_d ≈ 2π, the half-sphere area).

    GL rule (default, A11): μ_p = cos θ_p Gauss-Legendre on [-1, 1], φ_q = qπ/n_φ, w = W_p·π/n_φ.
    Paper rule (with the sin θ of the spherical measure outside ψ, A2):
    θ_p = pπ/n_θ, φ_q = qπ/n_φ, w = π²/(n_θ n_φ)·sin θ_p.
    Order: d = p·n_φ + q.
    """
    if rule == QUAD_GL_UNIFORM:
        mu, W = gauss_legendre(n_theta)
        st = np.sqrt(1.0 - mu * mu)
        wt = W * (math.pi / n_phi)
    elif rule == QUAD_PAPER_RECT:
        th = np.arange(n_theta) * (math.pi / n_theta)
        mu, st = np.cos(th), np.sin(th)
        wt = (math.pi ** 2 / (n_theta * n_phi)) * st
    else:
        raise ValueError("unknown quadrature rule")
    ph = np.arange(n_phi) * (math.pi / n_phi)
    e = np.empty((n_theta * n_phi, 3))
    w = np.empty(n_theta * n_phi)
    for p in range(n_theta):
        for q in range(n_phi):
            d = p * n_phi + q
            e[d] = (st[p] * math.cos(ph[q]), st[p] * math.sin(ph[q]), mu[p])
            w[d] = wt[p]
    return e, w


# ---------------------------------------------------------------------------------------------------
# Separated Carleman weights (readings A1-A7)
# ---------------------------------------------------------------------------------------------------

def phi_R(s, R: float):
    """φ_R(s) = ∫_{-R}^{R} |ρ| e^{iρs} dρ = 2R²[sin(Rs)/(Rs) − 2 sin²(Rs/2)/(Rs)²], φ_R(0) = R²  (A1)."""
    s = np.asarray(s, dtype=np.float64)
    x = R * s
    out = np.empty_like(x)
    z = x == 0.0
    xs = np.where(z, 1.0, x)
    out[...] = 2.0 * R * R * (np.sin(xs) / xs - 2.0 * np.sin(0.5 * xs) ** 2 / (xs * xs))
    out[z] = R * R
    return out


def psi_R(tau, R: float):
    """ψ_R(τ) = ∫_0^π φ_R(τ cos θ) dθ = 2πR·J₁(Rτ)/τ, ψ_R(0) = πR²  (A2)."""
    tau = np.asarray(tau, dtype=np.float64)
    z = tau == 0.0
    ts = np.where(z, 1.0, tau)
    out = 2.0 * math.pi * R * special.j1(R * ts) / ts
    out[z] = math.pi * R * R
    return out


@dataclass
class Tables:
    """Weight tables a_t(l), b_t(l) on K'^3, t = 0..T (t = 0 is the loss term).

    HS (B~ ≡ 1, separable): t = 1 + d,   a_t = w_d φ_R(ξ_l·e_d),  b_t = ψ_R(|ξ_l − (ξ_l·e_d)e_d|).
    MM (non-separable, radial split A6):  t = 1 + d·M_r + i,
        a_t = w_d·2W_iρ_i·cos(ρ_i ξ_l·e_d),  b_t = 2 Σ_j W_jρ_j (ρ_i²+ρ_j²)^{-1/2} J₀(ρ_j |Π_{e_d⊥} ξ_l|).
    Loss: a_0 = 1, b_0 = −Σ_{t≥1} a_t b_t  (so β̂(l,m) = B̂_F(l,m) − B̂_F(m,m)).
    """
    N: int
    L: float
    R: float
    kernel: int
    e: np.ndarray
    w: np.ndarray
    M_r: int
    a: np.ndarray = field(repr=False)  # (T+1, K', K', K')
    b: np.ndarray = field(repr=False)

    @property
    def T(self) -> int:
        return self.a.shape[0] - 1


def _xi_grid(N: int, L: float):
    xi = wavenumbers(N, L)
    X, Y, Z = np.meshgrid(xi, xi, xi, indexing="ij")
    return np.stack([X, Y, Z], axis=-1)  # (K',K',K',3)


def iter_terms(N: int, L: float, M: int = 16, M_r: int = 16, kernel: int = KERNEL_HARD_SPHERES,
               n_theta: int = 0, n_phi: int = 0, rule: int = QUAD_GL_UNIFORM, cutoff_ratio: float = 1.0,
               alpha: float = 0.5, C_alpha: float = VHS_C_DEFAULT):
    """Yield (a_t, b_t) for t = 1..T in order — step by step as in DESIGN.md §2.2
    (P:1612-1632 with readings A1-A7, A11, A12).  HS: t = 1 + d.  MM and VHS: t = 1 + d·M_r + i.

    VHS (A30): the same radial split as MM with B~(ρ_i, ρ_j) = 4C_α(ρ_i²+ρ_j²)^{(α−1)/2}, i.e.
    b_t = 2π Σ_j W_jρ_j B~(ρ_i, ρ_j) J₀(ρ_j τ)  (MM: 4C_0 = 1/π gives the factor 2 above)."""
    R = support_radius(L)
    Rc = R * (cutoff_ratio if cutoff_ratio > 0 else 1.0)  # Carleman cutoff x, y ∈ B_Rc (A7)
    if n_theta <= 0 or n_phi <= 0:
        n_theta, n_phi = split_angles(M)
    e, w = directions(n_theta, n_phi, rule)
    xi = _xi_grid(N, L)
    xi2 = np.sum(xi * xi, axis=-1)
    if kernel == KERNEL_HARD_SPHERES:
        for d in range(e.shape[0]):
            s = xi @ e[d]                                   # ξ_l · e_d
            tau = np.sqrt(np.maximum(xi2 - s * s, 0.0))     # |Π_{e_d⊥} ξ_l|
            yield w[d] * phi_R(s, Rc), psi_R(tau, Rc)
    elif kernel == KERNEL_MAXWELL:
        rho, Wr = gauss_legendre(M_r, 0.0, Rc)
        Bt = 1.0 / np.sqrt(rho[:, None] ** 2 + rho[None, :] ** 2)  # π·B~(ρ_i, ρ_j)
        for d in range(e.shape[0]):
            s = xi @ e[d]
            tau = np.sqrt(np.maximum(xi2 - s * s, 0.0))
            J0 = special.j0(rho[:, None, None, None] * tau[None])      # (M_r, K'^3)
            for i in range(M_r):
                yield (w[d] * 2.0 * Wr[i] * rho[i] * np.cos(rho[i] * s),
                       2.0 * np.tensordot(Wr * rho * Bt[i], J0, axes=(0, 0)))
    elif kernel == KERNEL_VHS:
        if not 0.0 <= alpha <= 1.0:
            raise ValueError("VHS needs 0 <= alpha <= 1")
        rho, Wr = gauss_legendre(M_r, 0.0, Rc)
        Bt = 4.0 * C_alpha * (rho[:, None] ** 2 + rho[None, :] ** 2) ** ((alpha - 1.0) / 2.0)  # B~(ρ_i, ρ_j)
        for d in range(e.shape[0]):
            s = xi @ e[d]
            tau = np.sqrt(np.maximum(xi2 - s * s, 0.0))
            J0 = special.j0(rho[:, None, None, None] * tau[None])
            for i in range(M_r):
                yield (w[d] * 2.0 * Wr[i] * rho[i] * np.cos(rho[i] * s),
                       2.0 * math.pi * np.tensordot(Wr * rho * Bt[i], J0, axes=(0, 0)))
    else:
        raise ValueError("unknown kernel")


def build_tables(N: int, L: float, M: int = 16, M_r: int = 16, kernel: int = KERNEL_HARD_SPHERES,
                 n_theta: int = 0, n_phi: int = 0, rule: int = QUAD_GL_UNIFORM,
                 cutoff_ratio: float = 1.0, alpha: float = 0.5, C_alpha: float = VHS_C_DEFAULT) -> Tables:
    """Materialise all terms, then the loss term t = 0: a_0 = 1, b_0 = −Σ_{t≥1} a_t b_t."""
    if n_theta <= 0 or n_phi <= 0:
        n_theta, n_phi = split_angles(M)
    e, w = directions(n_theta, n_phi, rule)
    terms = list(iter_terms(N, L, M, M_r, kernel, n_theta, n_phi, rule, cutoff_ratio, alpha, C_alpha))
    a = np.stack([t[0] for t in terms])
    b = np.stack([t[1] for t in terms])
    a0 = np.ones((1,) + a.shape[1:])
    b0 = -np.sum(a * b, axis=0, keepdims=True)
    return Tables(N=N, L=L, R=support_radius(L) * (cutoff_ratio if cutoff_ratio > 0 else 1.0),
                  kernel=kernel, e=e, w=w, M_r=M_r,
                  a=np.concatenate([a0, a]), b=np.concatenate([b0, b]))


def collision_fast_streamed(f: np.ndarray, term_args: dict, P: int | None = None) -> np.ndarray:
    """Same as ``collision_fast`` but regenerates the terms instead of storing (T+1)·K'^3 tables
    (needed for the N = 64 Maxwell-molecule BKW pin: 1025 terms × 63^3 × 2 fp64 = 4 GB)."""
    N = f.shape[-1]
    P = P or default_pad(N)
    fh = forward_modes(f)
    G = np.zeros((P, P, P), dtype=np.complex128)
    b0 = np.zeros(fh.shape)
    for a_t, b_t in iter_terms(N, **term_args):
        b0 -= a_t * b_t
        G += padded_inverse(a_t * fh, P) * padded_inverse(b_t * fh, P)
    G += padded_inverse(fh, P) * padded_inverse(b0 * fh, P)      # loss term t = 0 (a_0 = 1)
    return inverse_modes(padded_forward(G, N), N).real


def B_F(tables: Tables, l_idx, m_idx) -> float:
    """B̂_F(l, m) ≈ Σ_{t≥1} a_t(l) b_t(m) for index triples into K'^3."""
    a, b = tables.a, tables.b
    return float(np.sum(a[1:, l_idx[0], l_idx[1], l_idx[2]] * b[1:, m_idx[0], m_idx[1], m_idx[2]]))


# ---------------------------------------------------------------------------------------------------
# Naive per-axis DFTs (explicit DFT matrices; A10, A14)
# ---------------------------------------------------------------------------------------------------

def _along(M: np.ndarray, x: np.ndarray, axis: int) -> np.ndarray:
    """y[..., i, ...] = Σ_j M[i, j] x[..., j, ...] along `axis` (one matrix product per axis)."""
    return np.moveaxis(np.tensordot(M, x, axes=(1, axis)), 0, axis)


# Extended precision (x87 80-bit long double) is available for conditioning studies: near-equilibrium cells
# have Q ~ 1e-3 of the gain/loss terms that cancel to form it.
_PI_LD = np.longdouble("3.14159265358979323846264338327950288")


def _cdtype(ext: bool):
    return np.clongdouble if ext else np.complex128


def _expmat(rows, cols, M, sign, ext):
    """exp(sign·2πi·rows⊗cols/M) as a dense matrix (rows, cols: integer vectors)."""
    if ext:
        arg = np.outer(rows.astype(np.longdouble), cols.astype(np.longdouble)) * (2 * _PI_LD / np.longdouble(M))
        return np.cos(arg) + (1j if sign > 0 else -1j) * np.sin(arg)
    return np.exp(sign * 2j * math.pi * np.outer(rows, cols) / M)


def forward_modes(f: np.ndarray, ext: bool = False) -> np.ndarray:
    """f̂_l = N^-3 Σ_j f_j e^{-2πi l·j/N} for l ∈ K'^3 (P:1507 discretised; A14).  f: (N, N, N) real."""
    N = f.shape[-1]
    F = _expmat(kprime(N), np.arange(N), N, -1, ext)
    x = f.astype(_cdtype(ext))
    for ax in range(3):
        x = _along(F, x, ax)
    return x / N ** 3


def inverse_modes(Qh: np.ndarray, N: int) -> np.ndarray:
    """Q_j = Σ_{k∈K'} Q̂_k e^{2πi k·j/N}, j ∈ [0,N)^3 (complex; the imaginary part is round-off, A15)."""
    E = _expmat(np.arange(N), kprime(N), N, +1, Qh.dtype == np.clongdouble)
    x = Qh
    for ax in range(3):
        x = _along(E, x, ax)
    return x


def padded_inverse(Z: np.ndarray, P: int) -> np.ndarray:
    """z(p) = Σ_{l∈K'^3} Z(l) e^{2πi l·p/P}, p ∈ [0,P)^3: trig polynomial sampled on the padded grid."""
    K = kprime(Z.shape[-1] + 1)
    E = _expmat(np.arange(P), K, P, +1, Z.dtype == np.clongdouble)
    x = Z
    for ax in range(3):
        x = _along(E, x, ax)
    return x


def padded_forward(G: np.ndarray, N: int) -> np.ndarray:
    """Ĝ_k = P^-3 Σ_p G(p) e^{-2πi k·p/P} restricted to k ∈ K'^3 (Galerkin projection)."""
    P = G.shape[-1]
    ext = G.dtype in (np.clongdouble, np.longdouble)
    F = _expmat(kprime(N), np.arange(P), P, -1, ext)
    x = G.astype(_cdtype(ext))
    for ax in range(3):
        x = _along(F, x, ax)
    return x / P ** 3


def default_pad(N: int) -> int:
    """P = 3N/2: the smallest convenient size ≥ 3N/2 − 2 that makes the product exact on K' (A10)."""
    return 3 * N // 2


# ---------------------------------------------------------------------------------------------------
# Collision operator Q(f, f) — two evaluations of the same definition
# ---------------------------------------------------------------------------------------------------

def collision_fast(f: np.ndarray, tables: Tables, P: int | None = None, project_mass: bool = False,
                   return_diag: bool = False, ext: bool = False):
    """Fast spectral Q for ONE cell, the paper's convolution algorithm:

    1. f̂ = forward_modes(f)
    2. for t = 0..T:  A_t(p) = Σ_l a_t(l) f̂_l e^{2πi l·p/P},  B_t(p) = Σ_m b_t(m) f̂_m e^{2πi m·p/P}
                      G(p) += A_t(p)·B_t(p)           — "a discrete sum of A convolutions"
    3. Q̂_k = P^-3 Σ_p G(p) e^{-2πi k·p/P}, k ∈ K'   — exact for P ≥ 3N/2 − 2 (A10)
    4. optional (A24): Q̂_0 := 0
    5. Q_j = Σ_k Q̂_k e^{2πi k·j/N}; return Re Q (and max|Im Q| as a diagnostic, A15).
    ext=True evaluates every step in x87 extended precision (tables stay the fp64 values), for conditioning studies.
    """
    N = f.shape[-1]
    P = P or default_pad(N)
    fh = forward_modes(f, ext)
    G = np.zeros((P, P, P), dtype=_cdtype(ext))
    a_tab = tables.a.astype(np.longdouble) if ext else tables.a
    b_tab = tables.b.astype(np.longdouble) if ext else tables.b
    for t in range(tables.a.shape[0]):
        A = padded_inverse(a_tab[t] * fh, P)
        B = padded_inverse(b_tab[t] * fh, P)
        G += A * B
    Qh = padded_forward(G, N)
    c = N // 2 - 1
    q0 = Qh[c, c, c]
    if project_mass:
        Qh[c, c, c] = 0.0
    Q = inverse_modes(Qh, N)
    if ext:
        Q = Q.astype(np.complex128)
    if return_diag:
        return Q.real, {"max_imag": float(np.max(np.abs(Q.imag))), "Qhat0": complex(q0), "fhat": fh, "Qhat": Qh}
    return Q.real


def beta_matrix(tables: Tables) -> np.ndarray:
    """β̂(l, m) = Σ_{t=0}^{T} a_t(l) b_t(m) = B̂_F(l,m) − B̂_F(m,m) as a dense (K'^3 × K'^3) matrix."""
    n = tables.a[0].size
    return tables.a.reshape(-1, n).T @ tables.b.reshape(-1, n)


def collision_direct(f: np.ndarray, tables: Tables, project_mass: bool = False, P: int | None = None) -> np.ndarray:
    """Direct O(N^6) Galerkin double sum Q̂_k = Σ_{l+m=k} β̂(l,m) f̂_l f̂_m (Eq. CF1).

    With P given (N ≤ P < 3N/2 − 2): the aliased collocation operator of a P-point product grid (SURVEY §8(f)
    NEXT-4 (ii); P = N is the classical collocation spectral method), Q̂_k = Σ_{l+m ≡ k (mod P)} β̂(l,m) f̂_l f̂_m
    per axis — the pair (l, m) contributes to the k ∈ K' congruent to l + m, if any.  P ≥ 3N/2 − 2 gives back
    the exact sum.  Guarded to N ≤ 24 (the β̂ matrix has (N−1)^6 entries)."""
    N = f.shape[-1]
    if N > 24:
        raise ValueError("direct sum guarded to N <= 24")
    K = kprime(N)
    n1 = K.size
    fh = forward_modes(f)
    beta = beta_matrix(tables).reshape((n1,) * 6)
    Qh = np.zeros((n1, n1, n1), dtype=np.complex128)
    c = N // 2 - 1
    if P is not None:
        # aliased: every (l, m) pair, target k = ((l + m + c) mod P) − c when that lies in K'
        if P < N:
            raise ValueError("P >= N")
        s = K[:, None] + K[None, :]                       # l + m per axis
        kk = np.mod(s + c, P) - c
        valid = np.abs(kk) <= c
        tgt = kk + c                                      # index of k
        for ix in range(n1):
            for iy in range(n1):
                for iz in range(n1):
                    vx, vy, vz = valid[ix], valid[iy], valid[iz]
                    mx, my, mz = np.nonzero(vx)[0], np.nonzero(vy)[0], np.nonzero(vz)[0]
                    b = beta[ix, iy, iz][np.ix_(mx, my, mz)]
                    contrib = fh[ix, iy, iz] * b * fh[np.ix_(mx, my, mz)]
                    np.add.at(Qh, np.ix_(tgt[ix, mx], tgt[iy, my], tgt[iz, mz]), contrib)
        if project_mass:
            Qh[c, c, c] = 0.0
        return inverse_modes(Qh, N).real
    # index i ↔ mode K[i] = i - c;  k = l + m ∈ K' ⟺ 0 ≤ il + im − c < n1
    for ix in range(n1):
        for iy in range(n1):
            for iz in range(n1):
                # m ranges over K' with k = l + m ∈ K'
                mx = np.arange(max(0, c - ix), min(n1, n1 + c - ix))
                my = np.arange(max(0, c - iy), min(n1, n1 + c - iy))
                mz = np.arange(max(0, c - iz), min(n1, n1 + c - iz))
                b = beta[ix, iy, iz][np.ix_(mx, my, mz)]
                contrib = fh[ix, iy, iz] * b * fh[np.ix_(mx, my, mz)]
                Qh[np.ix_(mx + ix - c, my + iy - c, mz + iz - c)] += contrib
    if project_mass:
        Qh[c, c, c] = 0.0
    return inverse_modes(Qh, N).real


def collision_batch(f: np.ndarray, tables: Tables, P: int | None = None, project_mass: bool = False):
    """Q for every cell of f[n_cells, N, N, N] (cells are independent)."""
    return np.stack([collision_fast(fc, tables, P, project_mass) for fc in f]) if len(f) else np.zeros_like(f)


def loss_part(f: np.ndarray, tables: Tables) -> np.ndarray:
    """Q_loss(v) = f(v)·Σ_m B̂_F(m,m) f̂_m e^{iξ_m·v} (the loss term alone, positive), used to normalise
    parity and mass metrics (A23, A24).  = −(t=0 term of the fast sum)."""
    N = f.shape[-1]
    fh = forward_modes(f)
    nu = inverse_modes(-tables.b[0] * fh, N).real
    return f * nu


# ---------------------------------------------------------------------------------------------------
# FKS transport (exact shift of the generic cell; reading A16)
# ---------------------------------------------------------------------------------------------------

@dataclass
class GenericCell:
    """Integer offsets of the N particles per axis inside the generic cell.

    Units: 1/(N·c_den) cell.  A particle with velocity index k moves (2k − N)·c_num units per step,
    where c = c_num/c_den = Δt·L/Δx is the CFL number (A16).  Offsets live in [−½, ½) cell.
    """
    N: int
    c_num: int
    c_den: int
    offsets: np.ndarray = None  # (3, N) int64

    def __post_init__(self):
        if self.offsets is None:
            self.offsets = np.zeros((3, self.N), dtype=np.int64)

    def advance(self) -> np.ndarray:
        """Move every particle by v_k Δt; return δ[3, N] = whole cells crossed (A16)."""
        N, unit = self.N, self.N * self.c_den
        k = np.arange(N, dtype=np.int64)
        disp = (2 * k - N) * self.c_num
        delta = np.empty((3, N), dtype=np.int64)
        for a in range(3):
            o = self.offsets[a] + disp
            d = np.floor_divide(o + unit // 2, unit)
            self.offsets[a] = o - d * unit
            delta[a] = d
        return delta


def transport(f: np.ndarray, shape, delta: np.ndarray) -> np.ndarray:
    """f*_{j,k} = f_{(j − δ(k)) mod n, k} on a periodic (nx, ny, nz) cell grid.

    f: (nx·ny·nz, N, N, N), cell index (jx·ny + jy)·nz + jz.  One np.roll per velocity."""
    nx, ny, nz = shape
    N = f.shape[-1]
    g = f.reshape(nx, ny, nz, N, N, N)
    out = np.empty_like(g)
    for kx in range(N):
        for ky in range(N):
            for kz in range(N):
                out[:, :, :, kx, ky, kz] = np.roll(g[:, :, :, kx, ky, kz],
                                                   (int(delta[0, kx]), int(delta[1, ky]), int(delta[2, kz])),
                                                   axis=(0, 1, 2))
    return out.reshape(f.shape)


def source_cells(j: int, shape, delta: np.ndarray) -> np.ndarray:
    """For one destination cell j, the source cell index of every velocity k: (j − δ(k)) mod n."""
    nx, ny, nz = shape
    N = delta.shape[1]
    jx, jy, jz = j // (ny * nz), (j // nz) % ny, j % nz
    sx = (jx - delta[0]) % nx
    sy = (jy - delta[1]) % ny
    sz = (jz - delta[2]) % nz
    return (sx[:, None, None] * ny + sy[None, :, None]) * nz + sz[None, None, :]  # (N, N, N)


def euler(f_star: np.ndarray, Q: np.ndarray, s: float) -> np.ndarray:
    """f^{n+1} = f* + s·Q(f*), s = Δt/Kn (Eq. disc_relax; A18)."""
    return f_star + s * Q


def fks_step(f: np.ndarray, shape, cell: GenericCell, tables: Tables, s: float, P: int | None = None,
             project_mass: bool = False) -> np.ndarray:
    """One FKS step: transport → collision → explicit Euler (A17)."""
    delta = cell.advance()
    fs = transport(f, shape, delta)
    return np.stack([euler(fc, collision_fast(fc, tables, P, project_mass), s) for fc in fs])


# ---------------------------------------------------------------------------------------------------
# Closed forms used by the pins (not part of the method)
# ---------------------------------------------------------------------------------------------------

def maxwellian(v3: np.ndarray, rho: float, u, T: float) -> np.ndarray:
    """M[f] = ρ(2πT)^{-3/2} exp(−|v−u|²/2T); v3: (..., 3)."""
    d = v3 - np.asarray(u, dtype=np.float64)
    return rho * (2 * math.pi * T) ** -1.5 * np.exp(-np.sum(d * d, axis=-1) / (2 * T))


def bkw(v3: np.ndarray, K: float) -> np.ndarray:
    """BKW solution f_K = (2πK)^{-3/2} e^{-|v|²/2K}[(5K−3)/(2K) + (1−K)|v|²/(2K²)] (DESIGN.md §6 P14)."""
    r2 = np.sum(v3 * v3, axis=-1)
    return (2 * math.pi * K) ** -1.5 * np.exp(-r2 / (2 * K)) * ((5 * K - 3) / (2 * K) + (1 - K) * r2 / (2 * K * K))


def bkw_dfdt(v3: np.ndarray, K: float) -> np.ndarray:
    """∂_t f_K = K'(t)·∂_K f_K with K' = (1−K)/6 for Maxwell molecules with ∫B dω = 1 (A5)."""
    r2 = np.sum(v3 * v3, axis=-1)
    g = (5 * K - 3) / (2 * K) + (1 - K) * r2 / (2 * K * K)
    dg = 3.0 / (2 * K * K) + r2 * (-1.0 / K ** 3 + 1.0 / (2 * K * K))
    M = (2 * math.pi * K) ** -1.5 * np.exp(-r2 / (2 * K))
    dlnM = -1.5 / K + r2 / (2 * K * K)
    return (1 - K) / 6.0 * M * (dlnM * g + dg)


def velocity_grid3(N: int, L: float) -> np.ndarray:
    v = velocity_nodes(N, L)
    X, Y, Z = np.meshgrid(v, v, v, indexing="ij")
    return np.stack([X, Y, Z], axis=-1)


# ---------------------------------------------------------------------------------------------------
# Macroscopic moments (ToConservative / ToPrimitive) and the BGK operator
# ---------------------------------------------------------------------------------------------------

def collision_invariants(N: int, L: float) -> np.ndarray:
    """φ(v_k) = (1, v_x, v_y, v_z, |v|²/2) at every node: shape (5, N, N, N)."""
    v3 = velocity_grid3(N, L)
    return np.stack([np.ones(v3.shape[:-1]), v3[..., 0], v3[..., 1], v3[..., 2], 0.5 * np.sum(v3 * v3, axis=-1)])


def moments(f: np.ndarray, N: int, L: float) -> np.ndarray:
    """ToConservative: U_j = Σ_k φ(v_k) f_{j,k} (Δv)³ = (ρ, ρu_x, ρu_y, ρu_z, E) per cell.

    f: (n_cells, N, N, N) or (N, N, N); Δv = 2L/N.  Returns (n_cells, 5) or (5,)."""
    h3 = (2.0 * L / N) ** 3
    phi = collision_invariants(N, L)
    fc = f.reshape(-1, N, N, N)
    U = np.array([[np.sum(phi[a] * fc[c]) * h3 for a in range(5)] for c in range(fc.shape[0])])
    return U if f.ndim > 3 else U[0]


def moments_update(U_prev: np.ndarray, f_prev: np.ndarray, shape, delta: np.ndarray, N: int, L: float) -> np.ndarray:
    """Eq. DM_update: U_j^{n+1} = U_j^n + Σ_{k moved} (m_{j−δ(k),k} − m_{j,k}) φ(v_k) (Δv)³.

    Only the particles that change cell contribute (δ(k) ≠ 0); written as the paper's sum over particles."""
    h3 = (2.0 * L / N) ** 3
    phi = collision_invariants(N, L)
    U = np.array(U_prev, dtype=np.float64, copy=True)
    n = f_prev.shape[0]
    for j in range(n):
        src = source_cells(j, shape, delta)
        for kx in range(N):
            for ky in range(N):
                for kz in range(N):
                    if delta[0, kx] == 0 and delta[1, ky] == 0 and delta[2, kz] == 0:
                        continue
                    dm = f_prev[src[kx, ky, kz], kx, ky, kz] - f_prev[j, kx, ky, kz]
                    U[j] += dm * phi[:, kx, ky, kz] * h3
    return U


def primitive(U: np.ndarray) -> np.ndarray:
    """ToPrimitive: (ρ, u, T) from (ρ, ρu, E) with (3/2)ρT = E − ρ|u|²/2.  Shape (..., 5)."""
    U = np.asarray(U, dtype=np.float64)
    rho = U[..., 0]
    with np.errstate(divide="ignore", invalid="ignore"):
        u = U[..., 1:4] / rho[..., None]
        T = (U[..., 4] - 0.5 * rho * np.sum(u * u, axis=-1)) / (1.5 * rho)
    return np.concatenate([rho[..., None], u, T[..., None]], axis=-1)


def local_maxwellian(f: np.ndarray, N: int, L: float) -> np.ndarray:
    """E_{j,k} = M[f_j](v_k): the Maxwellian with the cell's (ρ, u, T) sampled at the nodes (P:179-183,
    P:397-410).  Reading A26: a cell with ρ ≤ 0 or T ≤ 0 (no Maxwellian exists) gets E = 0."""
    fc = f.reshape(-1, N, N, N)
    W = primitive(moments(fc, N, L).reshape(-1, 5))
    v3 = velocity_grid3(N, L)
    E = np.zeros_like(fc)
    for c in range(fc.shape[0]):
        rho, u, T = W[c, 0], W[c, 1:4], W[c, 4]
        if rho > 0 and T > 0:
            E[c] = maxwellian(v3, rho, u, T)
    return E.reshape(f.shape)


def bgk(f: np.ndarray, N: int, L: float, nu: float) -> np.ndarray:
    """Q_BGK(f) = ν (M[f] − f) per cell."""
    return nu * (local_maxwellian(f, N, L) - f)


def bgk_step(f: np.ndarray, shape, cell: GenericCell, nu_dt: float, L: float) -> np.ndarray:
    """One FKS step with the BGK operator: transport, then explicit Euler f^{n+1} = f* + Δt ν (E − f*)
    (Eq. disc_relax; A17).  nu_dt = ν Δt."""
    N = f.shape[-1]
    delta = cell.advance()
    fs = transport(f, shape, delta)
    return fs + nu_dt * (local_maxwellian(fs, N, L) - fs)
