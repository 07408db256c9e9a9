"""ctypes front end of the plain C++17 CPU oracle (oracle/cpp/fks_oracle.cpp) — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__`` (build + smoke) and ``bench.py``'s ``cpu_baseline`` / ``--impl reference``
leg may import this module.  It exposes the same functions as ``oracle.fks_oracle`` (the numpy oracle) with the
same array layouts, so that the pins of tests/test_oracle_pins*.py can be run against both, and the two
oracles can be cross-checked against each other.  The arithmetic lives in C++; this file only marshals arrays.
"""
from __future__ import annotations

import ctypes as C
import math
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "cpp", "fks_oracle.cpp")
LIB = os.path.join(HERE, "cpp", "libfks_oracle.so")
CXX = os.environ.get("CXX", "g++")
FLAGS = ["-O2", "-std=c++17", "-fPIC", "-shared", "-pthread", "-Wall", "-Wextra"]

LAMBDA = 2.0 / (3.0 + math.sqrt(2.0))
KERNEL_HARD_SPHERES, KERNEL_MAXWELL, KERNEL_VHS = 0, 1, 2
QUAD_GL_UNIFORM, QUAD_PAPER_RECT = 0, 1
VHS_C_DEFAULT = 1.0 / (4.0 * math.pi)


def build(force: bool = False) -> str:
    """Compile libfks_oracle.so in-tree with the host C++ compiler (no CUDA involved)."""
    if not force and os.path.exists(LIB) and os.path.getmtime(LIB) >= os.path.getmtime(SRC):
        return LIB
    r = subprocess.run([CXX] + FLAGS + [SRC, "-o", LIB], capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("C++ oracle build failed:\n" + r.stderr[-4000:])
    return LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        d, i, ll, vp = C.c_double, C.c_int, C.c_longlong, C.c_void_p
        sig = {
            "fkso_n_terms": ([i, d, i, i, i, i, i], i),
            "fkso_gauss_legendre": ([i, d, d, vp, vp], i),
            "fkso_directions": ([i, i, i, vp, vp], i),
            "fkso_phi_psi": ([vp, ll, d, vp, vp], None),
            "fkso_tables": ([i, d, i, i, i, i, i, i, d, d, d, vp, vp], i),
            "fkso_forward_modes": ([i, vp, vp, vp], None),
            "fkso_collision_fast": ([i, i, i, vp, vp, i, vp, vp, vp, ll, i], i),
            "fkso_collision_direct": ([i, i, vp, vp, i, i, vp, vp, ll, i], i),
            "fkso_loss_part": ([i, vp, vp, vp], None),
            "fkso_generic_cell_advance": ([i, ll, ll, vp, vp], None),
            "fkso_transport": ([vp, vp, i, i, i, i, vp], None),
            "fkso_step": ([i, i, i, vp, vp, vp, vp, i, i, i, ll, ll, vp, d, i, vp], i),
        }
        for name, (args, res) in sig.items():
            fn = getattr(_lib, name)
            fn.argtypes, fn.restype = args, res
    return _lib


def _p(x: np.ndarray):
    assert x.flags.c_contiguous
    return x.ctypes.data_as(C.c_void_p)


def default_threads() -> int:
    return len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)


def support_radius(L: float) -> float:
    return LAMBDA * L


def kprime(N: int) -> np.ndarray:
    return np.arange(-(N // 2 - 1), N // 2)


def split_angles(M: int):
    n_theta = 2 ** math.ceil(math.log2(M) / 2)
    if M % n_theta:
        n_theta = M
    return n_theta, M // n_theta


def gauss_legendre(n: int, a: float = -1.0, b: float = 1.0):
    x, w = np.empty(n), np.empty(n)
    lib().fkso_gauss_legendre(n, a, b, _p(x), _p(w))
    return x, w


def directions(n_theta: int, n_phi: int, rule: int = QUAD_GL_UNIFORM):
    e, w = np.empty((n_theta * n_phi, 3)), np.empty(n_theta * n_phi)
    lib().fkso_directions(n_theta, n_phi, rule, _p(e), _p(w))
    return e, w


def _phi_psi(s, R):
    s = np.ascontiguousarray(np.asarray(s, dtype=np.float64))
    phi, psi = np.empty_like(s), np.empty_like(s)
    lib().fkso_phi_psi(_p(s), s.size, R, _p(phi), _p(psi))
    return phi, psi


def phi_R(s, R: float):
    return _phi_psi(s, R)[0]


def psi_R(tau, R: float):
    return _phi_psi(tau, R)[1]


@dataclass
class Tables:
    N: int
    L: float
    R: float
    kernel: int
    e: np.ndarray
    w: np.ndarray
    M_r: int
    a: np.ndarray = field(repr=False)
    b: np.ndarray = field(repr=False)

    @property
    def T(self) -> int:
        return self.a.shape[0] - 1


def build_tables(N: int, L: float, M: int = 16, M_r: int = 16, kernel: int = KERNEL_HARD_SPHERES,
                 n_theta: int = 0, n_phi: int = 0, rule: int = QUAD_GL_UNIFORM, cutoff_ratio: float = 1.0,
                 alpha: float = 0.5, C_alpha: float = VHS_C_DEFAULT) -> Tables:
    if n_theta <= 0 or n_phi <= 0:
        n_theta, n_phi = split_angles(M)
    T = lib().fkso_n_terms(N, L, M, M_r, kernel, n_theta, n_phi)
    K = N - 1
    a = np.empty((T + 1, K, K, K))
    b = np.empty_like(a)
    if lib().fkso_tables(N, L, M, M_r, kernel, n_theta, n_phi, rule, cutoff_ratio, alpha, C_alpha, _p(a), _p(b)):
        raise ValueError("bad table arguments")
    e, w = directions(n_theta, n_phi, rule)
    return Tables(N=N, L=L, R=support_radius(L) * (cutoff_ratio if cutoff_ratio > 0 else 1.0), kernel=kernel,
                  e=e, w=w, M_r=M_r, a=a, b=b)


def default_pad(N: int) -> int:
    return 3 * N // 2


def forward_modes(f: np.ndarray) -> np.ndarray:
    N = f.shape[-1]
    f = np.ascontiguousarray(f, dtype=np.float64)
    re, im = np.empty((N - 1,) * 3), np.empty((N - 1,) * 3)
    lib().fkso_forward_modes(N, _p(f), _p(re), _p(im))
    return re + 1j * im


def collision_batch(f: np.ndarray, tables: Tables, P: int | None = None, project_mass: bool = False,
                    threads: int | None = None, return_imag: bool = False):
    f = np.ascontiguousarray(f, dtype=np.float64)
    N = f.shape[-1]
    n = f.shape[0]
    P = P or default_pad(N)
    Q = np.empty_like(f)
    mi = np.empty(max(n, 1))
    rc = lib().fkso_collision_fast(N, P, tables.a.shape[0], _p(tables.a), _p(tables.b), int(project_mass), _p(f),
                                   _p(Q), _p(mi), n, threads or default_threads())
    if rc:
        raise ValueError("bad collision arguments")
    return (Q, mi[:n]) if return_imag else Q


def collision_fast(f: np.ndarray, tables: Tables, P: int | None = None, project_mass: bool = False,
                   return_diag: bool = False):
    Q, mi = collision_batch(f[None], tables, P, project_mass, threads=1, return_imag=True)
    if return_diag:
        return Q[0], {"max_imag": float(mi[0])}
    return Q[0]


def collision_direct(f: np.ndarray, tables: Tables, project_mass: bool = False, P: int | None = None,
                     threads: int | None = None) -> np.ndarray:
    f = np.ascontiguousarray(f, dtype=np.float64)
    batch = f.ndim == 4
    fb = f if batch else f[None]
    N = fb.shape[-1]
    Q = np.empty_like(fb)
    rc = lib().fkso_collision_direct(N, tables.a.shape[0], _p(tables.a), _p(tables.b), int(project_mass),
                                     int(P or 0), _p(fb), _p(Q), fb.shape[0], threads or default_threads())
    if rc:
        raise ValueError("direct sum guarded to N <= 24")
    return Q if batch else Q[0]


def loss_part(f: np.ndarray, tables: Tables) -> np.ndarray:
    f = np.ascontiguousarray(f, dtype=np.float64)
    out = np.empty_like(f)
    b0 = np.ascontiguousarray(tables.b[0])
    lib().fkso_loss_part(f.shape[-1], _p(b0), _p(f), _p(out))
    return out


@dataclass
class GenericCell:
    N: int
    c_num: int
    c_den: int
    offsets: np.ndarray = None

    def __post_init__(self):
        if self.offsets is None:
            self.offsets = np.zeros((3, self.N), dtype=np.int64)

    def advance(self) -> np.ndarray:
        delta = np.empty((3, self.N), dtype=np.int64)
        lib().fkso_generic_cell_advance(self.N, self.c_num, self.c_den, _p(self.offsets), _p(delta))
        return delta


def transport(f: np.ndarray, shape, delta: np.ndarray) -> np.ndarray:
    f = np.ascontiguousarray(f, dtype=np.float64)
    d = np.ascontiguousarray(delta, dtype=np.int64)
    out = np.empty_like(f)
    lib().fkso_transport(_p(f), _p(out), shape[0], shape[1], shape[2], f.shape[-1], _p(d))
    return out


def euler(f_star: np.ndarray, Q: np.ndarray, s: float) -> np.ndarray:
    return f_star + s * Q


def fks_step(f: np.ndarray, shape, cell: GenericCell, tables: Tables, s: float, P: int | None = None,
             threads: int | None = None) -> np.ndarray:
    f = np.ascontiguousarray(f, dtype=np.float64)
    N = f.shape[-1]
    out = np.empty_like(f)
    rc = lib().fkso_step(N, P or default_pad(N), tables.a.shape[0], _p(tables.a), _p(tables.b), _p(f), _p(out),
                         shape[0], shape[1], shape[2], cell.c_num, cell.c_den, _p(cell.offsets), s,
                         threads or default_threads(), None)
    if rc:
        raise ValueError("bad step arguments")
    return out
