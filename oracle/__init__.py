"""CPU fp64 oracle package (TEST INFRASTRUCTURE ONLY; see oracle.py / moe_oracle.h)."""
from .oracle import *  # noqa: F401,F403
from .oracle import build, lib, max_rel_diff  # noqa: F401
