"""paper_1701_01608_b200 — B200-native hot path of the Fast Kinetic Scheme (arXiv 1701.01608).

libfks.so (csrc/, sm_100a) + a thin ctypes binding with the C-ABI names (binding.py).  Seeded synthetic
inputs live in inputs.py, the five workloads in configs.py.  Nothing here imports the CPU oracle.
"""
from .binding import *  # noqa: F401,F403
from .binding import Collision, FksError, load_library  # noqa: F401
from .configs import CONFIGS, Config  # noqa: F401
