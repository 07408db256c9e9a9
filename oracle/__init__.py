"""CPU oracle — TEST INFRASTRUCTURE ONLY (see fks_oracle.py header).  Never imported by the product path."""
from .fks_oracle import *  # noqa: F401,F403
from . import fks_oracle  # noqa: F401
