"""VecAttention fp64 CPU oracle -- TEST INFRASTRUCTURE ONLY (see oracle.py header)."""
from .oracle import *  # noqa: F401,F403
from .oracle import build  # noqa: F401
