"""ctypes binding of libfks (include/fks.h): argument marshalling only — every step of the path runs in the
library's sm_100a kernels.  PyTorch tensors are accepted for device memory and streams (plumbing).

There is no fallback: if libfks.so is missing or a call fails, an exception is raised.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libfks.so")

FKS_OK, FKS_ERR_INVALID, FKS_ERR_UNSUPPORTED, FKS_ERR_NOMEM, FKS_ERR_CUDA, FKS_ERR_STATE = range(6)
FKS_KERNEL_HARD_SPHERES, FKS_KERNEL_MAXWELL, FKS_KERNEL_VHS = 0, 1, 2
FKS_QUAD_GL_UNIFORM, FKS_QUAD_PAPER_RECT = 0, 1
FKS_PATH_AUTO, FKS_PATH_GENERIC, FKS_PATH_FAST = 0, 1, 2

STATUS_NAMES = {0: "FKS_OK", 1: "FKS_ERR_INVALID", 2: "FKS_ERR_UNSUPPORTED", 3: "FKS_ERR_NOMEM",
                4: "FKS_ERR_CUDA", 5: "FKS_ERR_STATE"}

#: every symbol include/fks.h declares (checked by tests/test_abi.py)
EXPORTS = ["fks_collision_init", "fks_collision_init_ex", "fks_collision_batch", "fks_collision_batch_host",
           "fks_transport_setup", "fks_transport_step", "fks_step", "fks_step_host", "fks_get_info", "fks_get_path",
           "fks_get_fast_layout",
           "fks_get_tables", "fks_get_last_shift", "fks_profile", "fks_profile_read", "fks_debug_timestamps", "fks_launch_count",
           "fks_sync", "fks_destroy", "fks_last_error", "fks_moments", "fks_bgk_batch", "fks_bgk_step",
           "fks_transport_setup_slab", "fks_slab_halo", "fks_slab_plane_count", "fks_transport_step_slab",
           "fks_step_slab", "fks_step_moments", "fks_step_slab_range", "fks_small_schedule"]


class fks_params(C.Structure):
    _fields_ = [("N", C.c_int), ("L", C.c_double), ("M_angles", C.c_int), ("M_radial", C.c_int),
                ("kernel", C.c_int), ("n_theta", C.c_int), ("n_phi", C.c_int), ("quad_rule", C.c_int),
                ("pad", C.c_int), ("cutoff_ratio", C.c_double), ("project_mass", C.c_int),
                ("max_cells_in_flight", C.c_longlong), ("path", C.c_int), ("vhs_alpha", C.c_double),
                ("vhs_C", C.c_double)]


class FksError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


_lib = None


def load_library(path: str = None):
    """Load libfks.so (built in-tree by paper_1701_01608_b200/build.py).  Raises if it is missing."""
    global _lib
    if _lib is not None:
        return _lib
    path = path or os.environ.get("FKS_LIB") or LIB_PATH
    if not os.path.exists(path):
        raise RuntimeError(f"libfks.so not found at {path}: run __graft_entry__.build() "
                           "(there is no CPU fallback)")
    lib = C.CDLL(path)
    vp, ll, d, i = C.c_void_p, C.c_longlong, C.c_double, C.c_int
    pp = C.POINTER(C.c_void_p)
    dp = C.POINTER(C.c_double)
    sig = {
        "fks_collision_init": ([pp, i, d, i, i, i], i),
        "fks_collision_init_ex": ([pp, C.POINTER(fks_params)], i),
        "fks_collision_batch": ([vp, vp, vp, ll, vp], i),
        "fks_collision_batch_host": ([vp, vp, vp, ll], i),
        "fks_transport_setup": ([vp, i, i, i, ll, ll], i),
        "fks_transport_step": ([vp, vp, vp, vp], i),
        "fks_step": ([vp, vp, vp, d, vp], i),
        "fks_step_host": ([vp, vp, vp, d], i),
        "fks_moments": ([vp, vp, vp, vp, ll, vp], i),
        "fks_step_moments": ([vp, vp, vp, d, vp, vp, vp], i),
        "fks_small_schedule": ([i, C.POINTER(i), C.POINTER(i), C.POINTER(i), C.POINTER(i), vp, vp], i),
        "fks_transport_setup_slab": ([vp, i, i, i, i, i, ll, ll], i),
        "fks_slab_halo": ([vp, C.POINTER(i)], i),
        "fks_slab_plane_count": ([vp, C.POINTER(i)], i),
        "fks_transport_step_slab": ([vp, vp, vp, vp], i),
        "fks_step_slab": ([vp, vp, vp, d, vp], i),
        "fks_step_slab_range": ([vp, vp, vp, d, i, i, i, vp], i),
        "fks_bgk_batch": ([vp, vp, vp, d, ll, vp], i),
        "fks_bgk_step": ([vp, vp, vp, d, vp, vp, vp], i),
        "fks_get_info": ([vp, C.POINTER(i), C.POINTER(i), dp, dp], i),
        "fks_get_path": ([vp], i),
        "fks_get_fast_layout": ([vp, C.POINTER(i), C.POINTER(i)], i),
        "fks_get_tables": ([vp, vp, vp, vp, vp], i),
        "fks_get_last_shift": ([vp, vp], i),
        "fks_profile": ([vp, i], i),
        "fks_profile_read": ([vp, dp, C.POINTER(ll)], i),
        "fks_debug_timestamps": ([vp, vp, ll], ll),
        "fks_launch_count": ([vp], ll),
        "fks_sync": ([vp, vp], i),
        "fks_destroy": ([vp], None),
        "fks_last_error": ([], C.c_char_p),
    }
    for name, (args, res) in sig.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    _lib = lib
    return lib


def _check(st: int):
    if st != FKS_OK:
        raise FksError(st, load_library().fks_last_error().decode())


def _ptr(x):
    """Device/host address of a torch tensor (or an int / None)."""
    if x is None:
        return None
    if isinstance(x, int):
        return x
    return x.data_ptr()


def _stream(stream):
    if stream is None:
        import torch
        if torch.cuda.is_available():
            return torch.cuda.current_stream().cuda_stream
        return None
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream


# ---- C-ABI mirrors (same names) ---------------------------------------------------------------------

def fks_collision_init(N: int, L: float, M_angles: int, M_radial: int, kernel: int) -> int:
    h = C.c_void_p()
    _check(load_library().fks_collision_init(C.byref(h), N, L, M_angles, M_radial, kernel))
    return h.value


def fks_collision_init_ex(**kw) -> int:
    p = fks_params()
    for k, v in kw.items():
        setattr(p, k, v)
    h = C.c_void_p()
    _check(load_library().fks_collision_init_ex(C.byref(h), C.byref(p)))
    return h.value


def fks_collision_batch(h: int, f, Q, n_cells: int | None = None, stream=None):
    n = f.shape[0] if n_cells is None else n_cells
    _check(load_library().fks_collision_batch(h, _ptr(f), _ptr(Q), n, _stream(stream)))


def fks_collision_batch_host(h: int, f_host, Q_host, n_cells: int | None = None):
    n = f_host.shape[0] if n_cells is None else n_cells
    _check(load_library().fks_collision_batch_host(h, _ptr(f_host), _ptr(Q_host), n))


def fks_transport_setup(h: int, nx: int, ny: int, nz: int, cfl_num: int, cfl_den: int):
    _check(load_library().fks_transport_setup(h, nx, ny, nz, cfl_num, cfl_den))


def fks_transport_step(h: int, f_in, f_out, stream=None):
    _check(load_library().fks_transport_step(h, _ptr(f_in), _ptr(f_out), _stream(stream)))


def fks_step(h: int, f_in, f_out, coll_scale: float, stream=None):
    _check(load_library().fks_step(h, _ptr(f_in), _ptr(f_out), coll_scale, _stream(stream)))


def fks_step_moments(h: int, f_in, f_out, coll_scale: float, U=None, W=None, stream=None):
    _check(load_library().fks_step_moments(h, _ptr(f_in), _ptr(f_out), coll_scale, _ptr(U), _ptr(W), _stream(stream)))


def fks_small_schedule(N: int):
    """Test-only: the small-N kernel's per-phase schedule {warps, nzs, nys, nxs, cnt[4][16], items[4][16][12]}."""
    import numpy as np
    w, z, y, x = C.c_int(), C.c_int(), C.c_int(), C.c_int()
    cnt = np.zeros((4, 16), dtype=np.uint8)
    items = np.zeros((4, 16, 12), dtype=np.uint8)
    rc = load_library().fks_small_schedule(N, C.byref(w), C.byref(z), C.byref(y), C.byref(x),
                                           cnt.ctypes.data_as(C.c_void_p), items.ctypes.data_as(C.c_void_p))
    if rc != 0:
        raise FksError(1, f"no small-N schedule for N = {N}")
    return {"warps": w.value, "nzs": z.value, "nys": y.value, "nxs": x.value, "cnt": cnt, "items": items}


def fks_step_host(h: int, f_in_host, f_out_host, coll_scale: float):
    _check(load_library().fks_step_host(h, _ptr(f_in_host), _ptr(f_out_host), coll_scale))


def fks_transport_setup_slab(h: int, nx_global: int, ny: int, nz: int, x0: int, nx_local: int, cfl_num: int,
                             cfl_den: int):
    _check(load_library().fks_transport_setup_slab(h, nx_global, ny, nz, x0, nx_local, cfl_num, cfl_den))


def fks_slab_halo(h: int) -> int:
    H = C.c_int()
    _check(load_library().fks_slab_halo(h, C.byref(H)))
    return H.value


def fks_slab_plane_count(h: int) -> int:
    n = C.c_int()
    _check(load_library().fks_slab_plane_count(h, C.byref(n)))
    return n.value


def _plane_array(h: int, planes):
    """HOST array of device pointers (ints or tensors) for the _slab calls; the C side reads exactly
    fks_slab_plane_count(h) entries, so the length is checked here."""
    want = fks_slab_plane_count(h)
    if len(planes) != want:
        raise FksError(1, f"planes has {len(planes)} entries, the slab needs nx_local + 2*halo = {want}")
    arr = (C.c_void_p * len(planes))()
    for i, p in enumerate(planes):
        arr[i] = _ptr(p)
    return arr


def fks_transport_step_slab(h: int, planes, f_out, stream=None):
    _check(load_library().fks_transport_step_slab(h, _plane_array(h, planes), _ptr(f_out), _stream(stream)))


def fks_step_slab(h: int, planes, f_out, coll_scale: float, stream=None):
    _check(load_library().fks_step_slab(h, _plane_array(h, planes), _ptr(f_out), coll_scale, _stream(stream)))


def fks_step_slab_range(h: int, planes, f_out, coll_scale: float, lx0: int, lx1: int, advance: bool, stream=None):
    _check(load_library().fks_step_slab_range(h, _plane_array(h, planes), _ptr(f_out), coll_scale, lx0, lx1,
                                              1 if advance else 0, _stream(stream)))


def fks_moments(h: int, f, U=None, W=None, n_cells: int | None = None, stream=None):
    n = f.shape[0] if n_cells is None else n_cells
    _check(load_library().fks_moments(h, _ptr(f), _ptr(U), _ptr(W), n, _stream(stream)))


def fks_bgk_batch(h: int, f, Q, nu: float, n_cells: int | None = None, stream=None):
    n = f.shape[0] if n_cells is None else n_cells
    _check(load_library().fks_bgk_batch(h, _ptr(f), _ptr(Q), nu, n, _stream(stream)))


def fks_bgk_step(h: int, f_in, f_out, nu_dt: float, U=None, W=None, stream=None):
    _check(load_library().fks_bgk_step(h, _ptr(f_in), _ptr(f_out), nu_dt, _ptr(U), _ptr(W), _stream(stream)))


def fks_get_info(h: int) -> dict:
    P, T = C.c_int(), C.c_int()
    R, lam = C.c_double(), C.c_double()
    _check(load_library().fks_get_info(h, C.byref(P), C.byref(T), C.byref(R), C.byref(lam)))
    return {"P": P.value, "T": T.value, "R": R.value, "lambda": lam.value}


def fks_get_path(h: int) -> int:
    return int(load_library().fks_get_path(h))


def fks_get_fast_layout(h: int) -> dict:
    a, b = C.c_int(), C.c_int()
    _check(load_library().fks_get_fast_layout(h, C.byref(a), C.byref(b)))
    return {"ctas_per_cell": a.value, "concurrent_cells": b.value}


def fks_get_tables(h: int, N: int, n_dirs: int):
    import numpy as np
    info = fks_get_info(h)
    K = N - 1
    a = np.empty((info["T"] + 1, K, K, K))
    b = np.empty_like(a)
    dirs = np.empty((n_dirs, 3))
    w = np.empty(n_dirs)
    _check(load_library().fks_get_tables(h, a.ctypes.data, b.ctypes.data, dirs.ctypes.data, w.ctypes.data))
    return a, b, dirs, w


def fks_get_last_shift(h: int, N: int):
    import numpy as np
    d = np.empty((3, N), dtype=np.int32)
    _check(load_library().fks_get_last_shift(h, d.ctypes.data))
    return d


def fks_profile(h: int, enable: bool = True):
    _check(load_library().fks_profile(h, 1 if enable else 0))


def fks_profile_read(h: int):
    """Per-phase (transport, forward, term loop, back) summed event milliseconds and launch counts."""
    ms = (C.c_double * 4)()
    cnt = (C.c_longlong * 4)()
    _check(load_library().fks_profile_read(h, ms, cnt))
    return list(ms), list(cnt)


def fks_debug_timestamps(h: int, n: int = 65536):
    import numpy as np
    buf = np.zeros(n, dtype=np.int64)
    got = load_library().fks_debug_timestamps(h, buf.ctypes.data, n)
    return buf[:got]


def fks_launch_count(h: int) -> int:
    return int(load_library().fks_launch_count(h))


def fks_sync(h: int, stream=None):
    _check(load_library().fks_sync(h, _stream(stream)))


def fks_destroy(h: int):
    if h:
        load_library().fks_destroy(h)


def fks_last_error() -> str:
    return load_library().fks_last_error().decode()


class Collision:
    """Owning wrapper around an fks_ctx handle (same operations as the C ABI)."""

    def __init__(self, N: int, L: float, M_angles: int = 16, M_radial: int = 16, kernel: int = 0, **kw):
        self.N = N
        self.h = fks_collision_init_ex(N=N, L=L, M_angles=M_angles, M_radial=M_radial, kernel=kernel, **kw)
        self.info = fks_get_info(self.h)
        self.info["path"] = fks_get_path(self.h)
        self.info.update(fks_get_fast_layout(self.h))

    def collision_batch(self, f, Q=None, stream=None):
        import torch
        Q = torch.empty_like(f) if Q is None else Q
        fks_collision_batch(self.h, f, Q, f.shape[0], stream)
        return Q

    def transport_setup(self, shape, cfl_num: int, cfl_den: int = 1):
        fks_transport_setup(self.h, shape[0], shape[1], shape[2], cfl_num, cfl_den)

    def transport_step(self, f_in, f_out, stream=None):
        fks_transport_step(self.h, f_in, f_out, stream)

    def step(self, f_in, f_out, coll_scale: float, stream=None):
        fks_step(self.h, f_in, f_out, coll_scale, stream)

    def step_moments(self, f_in, f_out, coll_scale: float, stream=None):
        """fks_step plus the moments (U, W) of f_out, [n_cells][5] each (fused into the step's last kernel)."""
        import torch
        U = torch.empty((f_out.shape[0], 5), dtype=torch.float64, device=f_out.device)
        W = torch.empty_like(U)
        fks_step_moments(self.h, f_in, f_out, coll_scale, U, W, stream)
        return U, W

    def moments(self, f, stream=None):
        """(U, W): conservative (ρ, ρu, E) and primitive (ρ, u, T) moments per cell, [n_cells][5] each."""
        import torch
        U = torch.empty((f.shape[0], 5), dtype=torch.float64, device=f.device)
        W = torch.empty_like(U)
        fks_moments(self.h, f, U, W, f.shape[0], stream)
        return U, W

    def bgk_batch(self, f, nu: float, Q=None, stream=None):
        import torch
        Q = torch.empty_like(f) if Q is None else Q
        fks_bgk_batch(self.h, f, Q, nu, f.shape[0], stream)
        return Q

    def bgk_step(self, f_in, f_out, nu_dt: float, U=None, W=None, stream=None):
        fks_bgk_step(self.h, f_in, f_out, nu_dt, U, W, stream)

    def last_shift(self):
        return fks_get_last_shift(self.h, self.N)

    def launches(self) -> int:
        return fks_launch_count(self.h)

    def close(self):
        if self.h:
            fks_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
