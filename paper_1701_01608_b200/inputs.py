"""Seeded synthetic inputs shaped like the paper's runs — shared by tests, bench and smoke.

This module holds none of the method's arithmetic (no transforms, tables, collision or transport): it only
draws per-cell parameters with numpy (`default_rng([1701, cfg_id])`, cells in order, Maxwellian 1 then 2)
and evaluates Maxwellian / BKW initial data on the velocity grid with torch on any device.  Every f is
set to 0 for |v| > R, the method's compact-support assumption (A20).
"""
from __future__ import annotations

import math

import numpy as np
import torch

from .configs import Config, CONFIGS, R_SUPPORT


def cfg_id(cfg: Config) -> int:
    return int(cfg.name[1:]) if cfg.name[1:].isdigit() else 99


def velocity_axis(N: int, L: float, device="cpu") -> torch.Tensor:
    """v_j = −L + j·2L/N (node-centred, A13)."""
    return -L + torch.arange(N, dtype=torch.float64, device=device) * (2.0 * L / N)


def cell_params(cfg: Config, seed: int | None = None) -> np.ndarray:
    """Per-cell Maxwellian parameters, shape (n_cells, n_max, 5) = (ρ, ux, uy, uz, T) per Maxwellian
    (ρ = 0 for unused slots), or (n_cells, 1, 1) = K for the BKW recipe."""
    key = [1701, cfg_id(cfg)] if seed is None else [1701, cfg_id(cfg), seed]
    rng = np.random.default_rng(key)
    n = cfg.n_cells
    if cfg.init == "two_maxwellian":          # BJ.configs[0] / [4]
        U = rng.random((n, 2, 5))            # == per cell, per Maxwellian: ρ, ux, uy, uz, T drawn in order
        p = np.empty((n, 2, 5))
        p[..., 0] = 0.5 + U[..., 0]          # ρ ~ U(0.5, 1.5)
        p[..., 1:4] = -1.0 + 2.0 * U[..., 1:4]  # u ~ U(−1, 1)^3
        p[..., 4] = 0.5 + U[..., 4]          # T ~ U(0.5, 1.5)
        return p
    if cfg.init == "bkw":                     # BJ.configs[1]
        return rng.uniform(0.5, 0.9, (n, 1, 1))
    if cfg.init == "shock_slab":              # BJ.configs[2]
        p = np.zeros((n, 1, 5))
        du = 1e-3 * rng.uniform(-1.0, 1.0, (n, 3))
        for c in range(n):
            left = c < n // 2
            p[c, 0] = (1.0 if left else 0.125, du[c, 0], du[c, 1], du[c, 2], 1.0 if left else 0.8)
        return p
    if cfg.init == "periodic_box":            # BJ.configs[3], reading A22
        ph = rng.uniform(0.0, 1.0, 3)
        nx, ny, nz = cfg.shape
        p = np.zeros((n, 1, 5))
        for jx in range(nx):
            x = (jx + 0.5) / nx
            for jy in range(ny):
                y = (jy + 0.5) / ny
                for jz in range(nz):
                    z = (jz + 0.5) / nz
                    c = (jx * ny + jy) * nz + jz
                    rho = 1.0 + 0.2 * math.sin(2 * math.pi * x) * math.cos(2 * math.pi * y)
                    u = 0.1 * np.array([math.sin(2 * math.pi * (y + ph[0])), math.sin(2 * math.pi * (z + ph[1])),
                                        math.sin(2 * math.pi * (x + ph[2]))])
                    p[c, 0] = (rho, u[0], u[1], u[2], 1.0)
        return p
    raise ValueError(cfg.init)


def fill(cfg: Config, out: torch.Tensor, params: np.ndarray, cells=None, chunk: int = 2048) -> torch.Tensor:
    """Evaluate the initial data of `params` (rows = `cells`, default all) into out[len(cells), N, N, N]."""
    N, L = cfg.N, cfg.L
    dev = out.device
    v = velocity_axis(N, L, dev)
    vx, vy, vz = v.view(N, 1, 1), v.view(1, N, 1), v.view(1, 1, N)
    inside = ((vx * vx + vy * vy + vz * vz) <= R_SUPPORT * R_SUPPORT).to(torch.float64)
    rows = np.arange(params.shape[0]) if cells is None else np.asarray(cells)
    for c0 in range(0, len(rows), chunk):
        idx = rows[c0:c0 + chunk]
        pr = torch.as_tensor(params[idx], dtype=torch.float64, device=dev)
        n = len(idx)
        if cfg.init == "bkw":
            K = pr[:, 0, 0].view(n, 1, 1, 1)
            r2 = (vx * vx + vy * vy + vz * vz).unsqueeze(0)
            f = (2 * math.pi * K) ** -1.5 * torch.exp(-r2 / (2 * K)) * ((5 * K - 3) / (2 * K) + (1 - K) * r2 / (2 * K * K))
        else:
            f = torch.zeros((n, N, N, N), dtype=torch.float64, device=dev)
            for a in range(pr.shape[1]):
                rho, ux, uy, uz, T = (pr[:, a, i].view(n, 1, 1, 1) for i in range(5))
                d2 = (vx - ux) ** 2 + (vy - uy) ** 2 + (vz - uz) ** 2
                f += rho * (2 * math.pi * T) ** -1.5 * torch.exp(-d2 / (2 * T))
        out[c0:c0 + n] = f * inside
    return out


def make_f(cfg: Config, device="cpu", cells=None, seed: int | None = None) -> torch.Tensor:
    """f[n, N, N, N] fp64 for the config (all cells, or the listed cell indices) on `device`."""
    params = cell_params(cfg, seed)
    n = cfg.n_cells if cells is None else len(cells)
    out = torch.empty((n, cfg.N, cfg.N, cfg.N), dtype=torch.float64, device=device)
    return fill(cfg, out, params, cells)


def random_field(n_cells: int, N: int, seed: int, signed: bool = False, device="cpu") -> torch.Tensor:
    """Unstructured random fields for algebraic parity cases (uniform [0,1) or [−1,1))."""
    g = np.random.default_rng([1701, 1000 + seed]).random((n_cells, N, N, N))
    if signed:
        g = 2 * g - 1
    return torch.as_tensor(g, dtype=torch.float64, device=device)


def sample_cells(cfg: Config, n: int, seed: int = 0) -> np.ndarray:
    """A seeded, sorted sample of cell indices (always includes the first and last cell)."""
    total = cfg.n_cells
    if n >= total:
        return np.arange(total)
    rng = np.random.default_rng([1701, 77, cfg_id(cfg), seed])
    pick = set(rng.choice(total, size=n, replace=False).tolist())
    pick.update({0, total - 1})
    return np.array(sorted(pick))


__all__ = ["CONFIGS", "cell_params", "fill", "make_f", "random_field", "sample_cells", "velocity_axis"]
