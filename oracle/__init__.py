"""CPU oracle package (TEST INFRASTRUCTURE ONLY; see oracle/oracle.py)."""
from .oracle import *  # noqa: F401,F403
from .oracle import build, lib, np_sum  # noqa: F401
