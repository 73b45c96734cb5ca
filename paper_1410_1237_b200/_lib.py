"""ctypes binding of libplv.so (the C ABI declared in include/plv.h).

There is no CPU fallback: if the library is missing or no sm_100 device is
visible, every entry point raises.  Status codes map onto the reference's
exception classes (PL/errors.py): PLV_EWEIGHT -> GraphParseError, PLV_ERANGE /
PLV_EINVAL / PLV_EDUP -> ValueError, otherwise RuntimeError.
"""

from __future__ import annotations

import ctypes
import os

from .errors import EdgelessGraphError, GraphParseError

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, f"libplv_{os.environ['PLV_VARIANT']}.so"
                        if os.environ.get("PLV_VARIANT") else "libplv.so")

PLV_OK = 0
PLV_EINVAL = -1
PLV_EWEIGHT = -2
PLV_ERANGE = -3
PLV_ECUDA = -4
PLV_ENODEV = -5
PLV_EDUP = -6

F_INDEPENDENT = 1
F_INTEGRAL = 2
F_IDENTITY = 4

STEP_DECIDE = 0
STEP_APPLY = 1
STEP_FINISH = 2
STEP_LIVE = 3
NCCL_ID_BYTES = 128
INGEST_HOST = 1

_P = ctypes.c_void_p
_I64 = ctypes.c_int64
_U64 = ctypes.c_uint64
_D = ctypes.c_double
_INT = ctypes.c_int

# name -> argtypes (all return int status unless listed in _RESTYPE)
_SIGS = {
    "plv_abi_version": [],
    "plv_last_error": [],
    "plv_device_ok": [],
    "plv_launch_count": [],
    "plv_debug_trace": [ctypes.c_int],
    "plv_debug_trace_read": [ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p],
    "plv_sum": [_P, _I64, _P, _P],
    "plv_modularity": [_P, _P, _I64, _D, _P, _P],
    "plv_csr_build": [_P, _P, _P, _I64, _I64, _P, _P, _P, _P, _P, _P, _P, _P],
    "plv_csr_from_sorted": [_P, _P, _P, _I64, _I64, _P, _P, _P, _P, _P, _P, _P, _P],
    "plv_edge_records": [_P, _P, _P, _I64, _P, _P, _P, _P, _P],
    "plv_vf_records": [_P, _P, _P, _P, _I64, _P, _P, _P, _P, _P, _P],
    "plv_color": [_P, _P, _I64, _I64, _P, _P, _P],
    "plv_color_assign": [_P, _P, _P, _I64, _P, _P, _P],
    "plv_color_conflicts": [_P, _P, _P, _I64, _P, _P, _P],
    "plv_color_classes": [_P, _I64, _I64, _P, _P, _P],
    "plv_decide": [_P, _P, _P, _P, _P, _P, _I64, _P, _P, _P, _D, _P, _P, _P, _P, _P, _P],
    "plv_decide_ex": [_P, _P, _P, _P, _P, _P, _I64, _P, _P, _P, _D, _INT, _P, _P, _P, _P, _P,
                      _P],
    "plv_apply": [_P, _P, _P, _P, _P, _I64, _P, _I64, _P, _P, _P, _P, _INT, _P, _P, _P, _P, _P,
                  _P],
    "plv_phase_create": [_P, _P, _P, _P, _P, _I64, _D, _INT, _P, _P, _P, _I64, _P, _P, _P, _P,
                         _INT, _P, _P],
    "plv_phase_create_part": [_P, _P, _P, _P, _P, _I64, _D, _INT, _P, _P, _P, _I64, _P, _P, _P,
                              _P, _I64, _I64, _P, _P, _P, _P, _P, _P, _P, _P],
    "plv_phase_create_part2": [_P, _P, _P, _P, _P, _I64, _D, _INT, _P, _P, _P, _I64, _P, _P,
                               _P, _P, _I64, _I64, _P, _P, _P, _P, _P, _P, _P, _P, _P],
    "plv_phase_step": [_P, _I64, _INT, _P, _P, _P],
    "plv_phase_slices": [_P, _P, _P],
    "plv_nccl_unique_id": [_P],
    "plv_nccl_comm_init": [_I64, _I64, _P, _P],
    "plv_nccl_comm_destroy": [_P],
    "plv_phase_iterate": [_P, _P, _P, _P, _P],
    "plv_phase_run": [_P, _D, _I64, _P, _P, _P, _P, _P],
    "plv_phase_decide_ms": [_P, _P],
    "plv_phase_graph_kernels": [_P, _P],
    "plv_phase_ahead_stats": [_P, _P],
    "plv_phase_destroy": [_P],
    "plv_rebuild_records": [_P, _P, _P, _I64, _P, _P, _P, _P, _P, _P, _P],
    "plv_compose": [_P, _P, _P, _I64, _P, _P],
    "plv_parse_edge_list": [_P, _I64, _P, _P, _P, _I64, _P, _P],
    "plv_parse_mm": [_P, _I64, _I64, _INT, _P, _P, _P, _I64, _P, _P],
    "plv_parse_metis": [_P, _I64, _I64, _I64, _INT, _P, _P, _P, _I64, _P, _P],
    "plv_format_assignment": [_P, _INT, _I64, _P, _I64, _P, _P],
    "plv_pair_counts": [_P, _P, _I64, _P, _P],
    "plv_gen_rmat": [_U64, _INT, _I64, _D, _D, _D, _D, _D, _P, _P, _P, _I64, _P, _P],
    "plv_gen_sbm": [_U64, _I64, _I64, _D, _D, _P, _P, _P, _I64, _P, _P],
    "plv_gen_grid": [_U64, _I64, _D, _I64, _D, _P, _P, _P, _I64, _P, _P],
    "plv_gen_chung_lu": [_U64, _P, _I64, _I64, _P, _P, _P, _I64, _P, _P],
    "plv_gen_rmat_range": [_U64, _INT, _I64, _D, _D, _D, _D, _D, _I64, _I64, _P, _P, _P, _I64,
                           _P, _P],
    "plv_route_records": [_P, _P, _P, _I64, _P, _INT, _P, _P, _P, _I64, _P, _P],
    "plv_part_own_rows": [_P, _P, _P, _I64, _I64, _I64, _P, _P, _P, _P, _P, _P],
    "plv_part_vf_only": [_P, _P, _P, _P, _I64, _I64, _I64, _P, _P],
    "plv_part_vf_map": [_P, _I64, _P, _P, _P, _P, _P],
    "plv_part_vf_records": [_P, _P, _P, _I64, _I64, _I64, _P, _P, _P, _P, _P, _P, _P, _P, _P,
                            _P, _P],
    "plv_scatter_i32": [_P, _P, ctypes.c_int32, _I64, _P, _P],
    "plv_select_rejected": [_P, _P, _I64, _P, _P, _P],
    "plv_renumber": [_P, _I64, _P, _P, _P],
    "plv_part_rebuild_records": [_P, _P, _P, _I64, _I64, _I64, _P, _P, _P, _P, _P, _P, _P],
}
_RESTYPE = {"plv_last_error": ctypes.c_char_p, "plv_launch_count": ctypes.c_ulonglong}

_LIB = None


class _Lib:
    def __init__(self, handle):
        self._h = handle
        for name, args in _SIGS.items():
            fn = getattr(handle, name)
            fn.argtypes = args
            fn.restype = _RESTYPE.get(name, ctypes.c_int)
            setattr(self, name[4:], fn)


def lib() -> _Lib:
    """Load libplv.so (raises if it was not built: there is no fallback)."""
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"{LIB_PATH} is missing: build it with `python -m paper_1410_1237_b200.build` "
                "(this package has no CPU fallback)")
        _LIB = _Lib(ctypes.CDLL(LIB_PATH))
    return _LIB


def exported_symbols() -> list[str]:
    return sorted(_SIGS)


def check(rc: int, what: str = ""):
    if rc == PLV_OK:
        return
    msg = lib().last_error()
    msg = msg.decode() if msg else what
    if rc == PLV_EWEIGHT:
        raise GraphParseError(msg)
    if rc in (PLV_ERANGE, PLV_EINVAL, PLV_EDUP):
        if "edgeless" in msg:
            raise EdgelessGraphError(msg)
        raise ValueError(msg)
    raise RuntimeError(f"libplv error {rc} in {what}: {msg}")


def ptr(t) -> int | None:
    """Raw device pointer of a torch tensor (None -> NULL)."""
    if t is None:
        return None
    return t.data_ptr()


def stream() -> int:
    import torch
    return torch.cuda.current_stream().cuda_stream


def device():
    """The CUDA device every tensor of this package lives on (fails loudly)."""
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("paper_1410_1237_b200 needs a CUDA (sm_100) device; "
                           "there is no CPU fallback")
    return torch.device("cuda", torch.cuda.current_device())


def i64_host(n: int = 1):
    return (ctypes.c_int64 * n)()


def f64_host(n: int = 1):
    return (ctypes.c_double * n)()


def hp(arr) -> int:
    """Address of a host ctypes buffer, for `_h` arguments."""
    return ctypes.addressof(arr)
