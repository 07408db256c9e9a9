"""The five workloads of BASELINE.json `configs` (c0..c4), with the readings of DESIGN.md §3 (A8, A12, A19, A21, A22).

Pure data: no arithmetic of the method lives here.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, asdict

KERNEL_HARD_SPHERES = 0
KERNEL_MAXWELL = 1

R_SUPPORT = 6.0                                   # BJ.configs[0]: R = 6
L_BOX = (3.0 + math.sqrt(2.0)) * R_SUPPORT / 2.0  # T = (3+√2)R/2 = 13.2426407 (A8)


@dataclass(frozen=True)
class Config:
    name: str
    N: int                 # velocity points per axis
    M: int                 # angular directions (half sphere)
    M_r: int               # radial Gauss-Legendre nodes (Maxwell molecules) / self-check (HS)
    kernel: int
    shape: tuple           # spatial cells (nx, ny, nz); n_cells = nx·ny·nz
    init: str              # input recipe
    cfl_num: int           # CFL c = Δt·L/Δx as a rational (A16, A19)
    cfl_den: int
    Kn: float              # Knudsen number: s = Δt/Kn (A18)
    dt_homog: float = 0.01  # homogeneous configs: s = 0.01 (A19)
    L: float = L_BOX
    steps: int = 1

    @property
    def n_cells(self) -> int:
        return self.shape[0] * self.shape[1] * self.shape[2]

    @property
    def dx(self) -> float:
        return 1.0 / max(self.shape)        # unit box [0,1)^d, Δx = 1/n (A21)

    @property
    def dt(self) -> float:
        if self.cfl_num == 0:
            return self.dt_homog
        return (self.cfl_num / self.cfl_den) * self.dx / self.L

    @property
    def coll_scale(self) -> float:
        """s = Δt/Kn multiplying Q in the Euler update (A18)."""
        return self.dt / self.Kn

    def as_dict(self):
        d = asdict(self)
        d["n_cells"] = self.n_cells
        return d


CONFIGS = {
    "c0": Config("c0", 16, 16, 16, KERNEL_HARD_SPHERES, (8, 1, 1), "two_maxwellian", 0, 1, 1.0),
    "c1": Config("c1", 24, 16, 16, KERNEL_MAXWELL, (64, 1, 1), "bkw", 0, 1, 1.0),
    "c2": Config("c2", 32, 32, 16, KERNEL_HARD_SPHERES, (512, 1, 1), "shock_slab", 1, 1, 1.0),
    "c3": Config("c3", 32, 32, 16, KERNEL_HARD_SPHERES, (32, 32, 32), "periodic_box", 1, 1, 1.0),
    "c4": Config("c4", 32, 64, 16, KERNEL_HARD_SPHERES, (48, 48, 48), "two_maxwellian", 1, 8, 0.01, steps=10),
}
