"""The reference's kernel seam (PL/_kernels.pyx) over numpy arrays, on device.

Each call uploads its numpy arguments, runs the CUDA kernel through libplv's
C ABI and writes the outputs back into the caller's numpy buffers, with the
reference's argument order, dtypes (int64 / float64 / uint8) and in-place
semantics.  Used by ``backend.active()`` for kernel-granular parity tests.
"""

from __future__ import annotations

import numpy as np

from . import _lib

COMPILED = True


def _dev(a, dtype, keep):
    """Upload `a`; the tensor is appended to `keep` so that it outlives the
    (asynchronous) kernel that reads it."""
    import torch
    t = torch.from_numpy(np.array(a, dtype=dtype, copy=True)).to(_lib.device())
    keep.append(t)
    return _lib.ptr(t)


def decide_moves(offsets, neighbors, weights, kdeg, labels, subset, snap_assign, snap_atot,
                 snap_sizes, m, max_degree, workers, out_targets, out_moved):
    """PL/_kernels.pyx:21-101 on device (exact ordered folds)."""
    keep = []
    import torch
    ns = len(subset)
    dev = _lib.device()
    n = len(kdeg)
    lab = np.asarray(labels)
    ident = len(lab) == n and np.array_equal(lab, np.arange(n))
    tg = torch.empty(max(ns, 1), dtype=torch.int32, device=dev)
    mv = torch.empty(max(ns, 1), dtype=torch.uint8, device=dev)
    eo = torch.empty(max(ns, 1), dtype=torch.float64, device=dev)
    eb = torch.empty(max(ns, 1), dtype=torch.float64, device=dev)
    _lib.check(_lib.lib().decide(
        _dev(offsets, np.int64, keep), _dev(neighbors, np.int32, keep),
        _dev(weights, np.float64, keep), _dev(kdeg, np.float64, keep),
        None if ident else _dev(lab, np.int32, keep), _dev(subset, np.int32, keep), ns,
        _dev(snap_assign, np.int32, keep), _dev(snap_atot, np.float64, keep),
        _dev(snap_sizes, np.int32, keep), float(m), _lib.ptr(tg), _lib.ptr(mv),
        _lib.ptr(eo), _lib.ptr(eb), None, _lib.stream()), "decide_moves")
    out_targets[:ns] = tg[:ns].cpu().numpy()
    out_moved[:ns] = mv[:ns].cpu().numpy()


def apply_moves(offsets, neighbors, weights, kdeg, selfw, subset, targets, moved, assign,
                a_tot, w_int, sizes):
    """PL/_kernels.pyx:104-145 on device; mutates assign/a_tot/w_int/sizes."""
    keep = []
    ns = len(subset)
    n = len(kdeg)
    sub = np.asarray(subset, dtype=np.int64)
    flags = _lib.F_IDENTITY if (ns == n and np.array_equal(sub, np.arange(n))) else 0
    import torch
    dev = _lib.device()
    d_assign = torch.from_numpy(np.asarray(assign).astype(np.int32)).to(dev)
    d_atot = torch.from_numpy(np.array(a_tot, dtype=np.float64)).to(dev)
    d_wint = torch.from_numpy(np.array(w_int, dtype=np.float64)).to(dev)
    d_sizes = torch.from_numpy(np.asarray(sizes).astype(np.int32)).to(dev)
    moves = _lib.i64_host(1)
    _lib.check(_lib.lib().apply(
        _dev(offsets, np.int64, keep), _dev(neighbors, np.int32, keep),
        _dev(weights, np.float64, keep), _dev(kdeg, np.float64, keep),
        _dev(selfw, np.float64, keep), n, _dev(sub, np.int32, keep), ns,
        _dev(targets, np.int32, keep), _dev(moved, np.uint8, keep), None, None, flags,
        _lib.ptr(d_assign), _lib.ptr(d_atot), _lib.ptr(d_wint), _lib.ptr(d_sizes),
        _lib.hp(moves), _lib.stream()), "apply_moves")
    assign[:] = d_assign.cpu().numpy()
    a_tot[:] = d_atot.cpu().numpy()
    w_int[:] = d_wint.cpu().numpy()
    sizes[:] = d_sizes.cpu().numpy()
    return int(moves[0])


def color_assign(offsets, neighbors, active, colors, max_degree, workers, out_colors):
    """PL/_kernels.pyx:148-174 on device."""
    keep = []
    import torch
    na = len(active)
    out = torch.empty(max(na, 1), dtype=torch.int32, device=_lib.device())
    _lib.check(_lib.lib().color_assign(
        _dev(offsets, np.int64, keep), _dev(neighbors, np.int32, keep),
        _dev(active, np.int32, keep), na, _dev(colors, np.int32, keep), _lib.ptr(out),
        _lib.stream()), "color_assign")
    out_colors[:na] = out[:na].cpu().numpy()


def color_conflicts(offsets, neighbors, active, colors, workers, out_keep):
    """PL/_kernels.pyx:177-195 on device."""
    keep = []
    import torch
    na = len(active)
    out = torch.empty(max(na, 1), dtype=torch.uint8, device=_lib.device())
    _lib.check(_lib.lib().color_conflicts(
        _dev(offsets, np.int64, keep), _dev(neighbors, np.int32, keep),
        _dev(active, np.int32, keep), na, _dev(colors, np.int32, keep), _lib.ptr(out),
        _lib.stream()), "color_conflicts")
    out_keep[:na] = out[:na].cpu().numpy()
