"""Shared helpers for the parity tests: oracle tables per config (cached), per-cell error metrics."""
from __future__ import annotations

import functools

import numpy as np

from oracle import fks_oracle as o
from paper_1701_01608_b200.configs import CONFIGS

TOL_Q = 1e-10       # BJ.north_star: relative L∞ per cell (A23)
TOL_TABLE = 1e-13   # DESIGN.md P17


@functools.lru_cache(maxsize=None)
def oracle_tables(N, L, M, M_r, kernel, n_theta=0, n_phi=0, rule=0, cutoff_ratio=1.0, alpha=0.5,
                  C_alpha=o.VHS_C_DEFAULT):
    return o.build_tables(N, L, M=M, M_r=M_r, kernel=kernel, n_theta=n_theta, n_phi=n_phi, rule=rule,
                          cutoff_ratio=cutoff_ratio, alpha=alpha, C_alpha=C_alpha)


def cfg_tables(name):
    c = CONFIGS[name]
    return oracle_tables(c.N, c.L, c.M, c.M_r, c.kernel)


def rel_err_per_cell(q_gpu: np.ndarray, q_ref: np.ndarray) -> np.ndarray:
    """e_c = ‖Q_gpu − Q_ora‖∞ / ‖Q_ora‖∞ for each cell c (A23)."""
    n = q_ref.shape[0]
    d = np.abs(q_gpu.reshape(n, -1) - q_ref.reshape(n, -1)).max(axis=1)
    s = np.abs(q_ref.reshape(n, -1)).max(axis=1)
    return d / np.maximum(s, 1e-300)


def oracle_Q(f: np.ndarray, tables, P=None, project_mass=False) -> np.ndarray:
    return np.stack([o.collision_fast(fc, tables, P, project_mass) for fc in f])
