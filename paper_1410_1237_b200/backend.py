"""Kernel backend seam (mirror of PL/backend.py) -- CUDA only.

The reference chooses between a compiled OpenMP module and a pure-Python twin
(PL/backend.py:13-70).  This build has exactly one backend, the sm_100a CUDA
library, and no CPU fallback: ``name()`` is "cuda", ``has_compiled()`` is
True, ``use("compiled" | "auto" | "cuda")`` keeps it and ``use("python")``
raises ValueError.  ``active()`` returns a module-like object exposing the
reference's four kernel signatures (PL/_kernels.pyx:21-195) over numpy
arrays, for kernel-granular parity tests; the engine itself calls the device
API directly and never round-trips through numpy.
"""

from __future__ import annotations

import logging
import os

from . import _kernels_cuda as _cuda

log = logging.getLogger(__name__)

_NAMES = {"cuda", "compiled", "auto"}


def _initial():
    requested = os.environ.get("PARLOUVAIN_BACKEND", "auto").strip().lower()
    if requested not in _NAMES:
        raise ImportError(
            f"PARLOUVAIN_BACKEND={requested!r}: this build runs only the CUDA backend "
            "(no CPU fallback)")
    return _cuda


_active = _initial()


def active():
    """The kernel module currently in use (always the CUDA one)."""
    return _active


def name() -> str:
    return "cuda"


def has_compiled() -> bool:
    return True


def use(which: str):
    """Select a backend; only the CUDA backend exists.  Returns the old name."""
    key = which.strip().lower()
    if key not in _NAMES:
        raise ValueError(f"backend {which!r} is not available: this build has no CPU fallback")
    return name()
