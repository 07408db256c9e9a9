"""CPU checks of the boundary: libfks.so builds for sm_100a, loads, and exports every symbol fks.h declares;
without a GPU every compute entry fails loudly (there is no CPU fallback)."""
import ctypes
import os
import re
import subprocess

import pytest

from paper_1701_01608_b200 import binding, build

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    build.build()
    return binding.load_library()


def header_symbols():
    src = open(os.path.join(ROOT, "include", "fks.h")).read()
    return sorted(set(re.findall(r"\b(fks_[a-z_]+)\s*\(", src)))


def test_header_and_binding_agree():
    assert header_symbols() == sorted(binding.EXPORTS)


def test_library_exports_every_symbol(lib):
    for name in header_symbols():
        assert hasattr(lib, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", build.LIB], capture_output=True, text=True).stdout
    for name in header_symbols():
        assert re.search(rf"\bT {name}\b", out), name


def test_sm100a_code_present(lib):
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", build.LIB], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_fails_loudly_without_gpu(lib):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    h = ctypes.c_void_p()
    st = lib.fks_collision_init(ctypes.byref(h), 16, 13.24, 16, 16, 0)
    assert st == binding.FKS_ERR_CUDA and h.value is None
    assert lib.fks_last_error()
    with pytest.raises(binding.FksError):
        binding.Collision(16, 13.24)


def test_argument_validation_without_gpu(lib):
    h = ctypes.c_void_p()
    assert lib.fks_collision_init(ctypes.byref(h), 15, 13.24, 16, 16, 0) == binding.FKS_ERR_UNSUPPORTED
    assert lib.fks_collision_init(ctypes.byref(h), 130, 13.24, 16, 16, 0) == binding.FKS_ERR_UNSUPPORTED
    assert lib.fks_collision_init(ctypes.byref(h), 16, -1.0, 16, 16, 0) == binding.FKS_ERR_INVALID
    assert lib.fks_collision_init(ctypes.byref(h), 16, 13.24, 0, 16, 0) == binding.FKS_ERR_INVALID
    assert lib.fks_collision_init(ctypes.byref(h), 16, 13.24, 16, 0, 1) == binding.FKS_ERR_INVALID
    assert lib.fks_collision_init(ctypes.byref(h), 16, 13.24, 16, 16, 7) == binding.FKS_ERR_UNSUPPORTED
    assert lib.fks_collision_batch(None, None, None, 1, None) == binding.FKS_ERR_INVALID
    assert lib.fks_step(None, None, None, 0.1, None) == binding.FKS_ERR_INVALID


def test_cutoff_ratio_range_without_gpu(lib):
    """R_c / R below 1 would truncate the Carleman integral (A7): rejected before any device work; 0 is the
    default sentinel and [1, (1+sqrt2)/sqrt2] is accepted (FKS_ERR_CUDA here only because there is no GPU)."""
    import torch

    def init(ratio):
        p = binding.fks_params(N=16, L=13.24, M_angles=16, M_radial=16, kernel=0, cutoff_ratio=ratio)
        h = ctypes.c_void_p()
        return lib.fks_collision_init_ex(ctypes.byref(h), ctypes.byref(p))
    for bad in (0.5, 0.999, -1.0, 1.8):
        assert init(bad) == binding.FKS_ERR_INVALID, bad
    if not torch.cuda.is_available():
        for good in (0.0, 1.0, 1.5):
            assert init(good) == binding.FKS_ERR_CUDA, good


def test_product_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_1701_01608_b200")
    for dirpath, _, files in os.walk(pkg):
        for fn in files:
            if fn.endswith((".py", ".cu", ".cuh", ".cpp", ".h")):
                txt = open(os.path.join(dirpath, fn)).read()
                assert not re.search(r"^\s*(from|import)\s+oracle", txt, re.M), fn
                assert "fks_oracle" not in txt, fn


@pytest.mark.parametrize("N", [16, 24])
def test_small_schedule_host_logic(N):
    """The small-N kernel's static schedule (built on the host, no device): every slot of every phase appears
    exactly once; X slots run on a warp of their TMEM lane quarter (slot % 4 == warp % 4), whose G block they
    own across terms; phase A = Z + X, B = Y, C and D = X + Y; the makespan (Z = 2 units) is within one unit of
    the balanced bound."""
    sc = binding.fks_small_schedule(N)
    W, nzs, nys, nxs = sc["warps"], sc["nzs"], sc["nys"], sc["nxs"]
    for ph in range(4):
        seen = []
        load = []
        for w in range(W):
            items = [int(x) for x in sc["items"][ph, w, :sc["cnt"][ph, w]]]
            seen += items
            load.append(sum(2 if it >> 5 == 0 else 1 for it in items))
            for it in items:
                if it >> 5 == 2:
                    assert (it & 31) % 4 == w % 4, (ph, w, it)
        want = ({(0 << 5) | s for s in range(nzs)} if ph == 0 else set()) | \
               ({(1 << 5) | s for s in range(nys)} if ph != 0 else set()) | \
               ({(2 << 5) | s for s in range(nxs)} if ph != 1 else set())
        assert sorted(seen) == sorted(want), ph
        assert max(load) <= -(-sum(load) // W) + 1, (ph, load)
    assert sc["cnt"][:, W:].sum() == 0
