"""Multi-GPU local moving: 1D vertex partition, replicated state.

The reference has no distributed mode; this is new design.  decide
(PL/_kernels.pyx:21-101) is independent per vertex given the stage's entry
state, so the vertices of every stage are split across ranks by contiguous,
nnz-balanced vertex ranges.  Because a stage lists its vertices in ascending
id, each rank's share of a stage is one contiguous slice of it, and rank
order is subset order.  Per stage:

  1. every rank decides its slice (target, moved, e_old, e_best);
  2. the slices are all-gathered in rank order (one padded all_gather per
     array over NCCL / gloo);
  3. every rank applies the whole stage with the same exact, order-preserving
     apply, so assignment / a_tot / w_internal / sizes stay bit-identical on
     all ranks and to the 1-GPU run (no reduction of float64 deltas, whose
     order would change the bits).

Modularity needs no communication (replicated aggregates).  Uncoloured
iterations gather (target, moved) and replay the apply with the live rule on
every rank.  The compute steps are callbacks, so the same driver runs the CUDA
kernels (`CudaStageOps`, slice-level C-ABI calls) and a CPU checker over gloo
in the tests.  The production multi-GPU path is `PartitionedPhaseEngine`
(plv_phase_create_part): the same per-stage decide / exchange / replicated
apply, with the NCCL broadcasts captured inside the iteration's CUDA graph.
"""

from __future__ import annotations

import contextlib
from dataclasses import dataclass

import numpy as np


def partition_bounds(offsets, world: int) -> np.ndarray:
    """Contiguous vertex ranges balancing adjacency entries: rank r owns
    vertices [bounds[r], bounds[r+1])."""
    off = np.asarray(offsets, dtype=np.int64)
    n = len(off) - 1
    total = int(off[-1])
    targets = (total * np.arange(1, world, dtype=np.float64) / world).astype(np.int64)
    cuts = np.searchsorted(off, targets, side="left").clip(0, n)
    bounds = np.concatenate([[0], cuts, [n]]).astype(np.int64)
    return np.maximum.accumulate(bounds)


def stage_slices(stage, bounds) -> np.ndarray:
    """Slice boundaries of an ascending stage vertex list per rank:
    rank r decides stage[s[r]:s[r+1]]."""
    return np.searchsorted(np.asarray(stage), np.asarray(bounds), side="left").astype(np.int64)


def allgather_slices(local_arrays, counts, group=None):
    """All-gather 1-D tensors whose per-rank lengths are `counts`, concatenated
    in rank order (padded to the largest count)."""
    import torch
    import torch.distributed as dist
    world = len(counts)
    cmax = max(1, max(counts))
    out = []
    for t in local_arrays:
        pad = torch.zeros(cmax, dtype=t.dtype, device=t.device)
        pad[:t.numel()] = t
        parts = [torch.empty_like(pad) for _ in range(world)]
        dist.all_gather(parts, pad, group=group)
        out.append(torch.cat([parts[r][:counts[r]] for r in range(world)]))
    return out


@dataclass
class DecideSlice:
    target: object
    moved: object
    e_old: object
    e_best: object


class DistributedIteration:
    """One local-move iteration over a stage list, decide split across ranks.

    ops.decide(stage_index, lo, hi) -> DecideSlice for stage[lo:hi]
    ops.apply(stage_index, DecideSlice_full) -> moves (replicated, exact)
    ops.modularity() -> Q (replicated)
    """

    def __init__(self, ops, stages_host, bounds, rank: int, world: int, group=None):
        self.ops, self.rank, self.world, self.group = ops, rank, world, group
        self.slices = [stage_slices(st, bounds) for st in stages_host]

    def run(self):
        moves = 0
        for a, sl in enumerate(self.slices):
            lo, hi = int(sl[self.rank]), int(sl[self.rank + 1])
            d = self.ops.decide(a, lo, hi)
            counts = [int(sl[r + 1] - sl[r]) for r in range(self.world)]
            if self.world > 1:
                t, m, eo, eb = allgather_slices([d.target, d.moved, d.e_old, d.e_best], counts,
                                                self.group)
                d = DecideSlice(t, m, eo, eb)
            moves += self.ops.apply(a, d)
        return moves, self.ops.modularity()


@contextlib.contextmanager
def stdout_to_stderr():
    """Route file descriptor 1 to stderr: NCCL prints its version banner on
    stdout at first use, and stdout may carry machine-read output (bench.py's
    JSON line)."""
    import os
    import sys
    sys.stdout.flush()
    saved = os.dup(1)
    os.dup2(2, 1)
    try:
        yield
    finally:
        sys.stdout.flush()
        os.dup2(saved, 1)
        os.close(saved)


def nccl_communicator(rank: int, world: int, group=None):
    """NCCL communicator for PartitionedPhaseEngine (libplv binds NCCL at run
    time): rank 0 draws the unique id, torch.distributed broadcasts it."""
    import ctypes
    from . import _lib
    L = _lib.lib()
    idbuf = (ctypes.c_uint8 * _lib.NCCL_ID_BYTES)()
    comm = ctypes.c_void_p()
    with stdout_to_stderr():
        if rank == 0:
            _lib.check(L.nccl_unique_id(ctypes.addressof(idbuf)), "nccl_unique_id")
        if world > 1:
            import torch.distributed as dist
            obj = [bytes(idbuf)]
            dist.broadcast_object_list(obj, src=0, group=group)
            ctypes.memmove(idbuf, obj[0], _lib.NCCL_ID_BYTES)
        _lib.check(L.nccl_comm_init(rank, world, ctypes.addressof(idbuf), ctypes.byref(comm)),
                   "nccl_comm_init")
    return comm


def destroy_communicator(comm):
    from . import _lib
    if comm is not None and comm.value:
        _lib.check(_lib.lib().nccl_comm_destroy(comm), "nccl_comm_destroy")


class PartitionedPhaseEngine:
    """The phase engine on one rank of a 1D vertex partition (plv_phase_create_part).

    Rank `rank` decides its slice of every stage; with a communicator the
    slices are exchanged by NCCL broadcasts inside the iteration's CUDA graph
    and `iterate()` is one graph launch, as on one GPU.  Without one
    (world > 1), the caller steps the stages: `step(a, STEP_DECIDE)`, move
    the slices between ranks' `outputs`, `step(a, STEP_APPLY)`, then
    `finish()` (the single-GPU test of the partitioned plan)."""

    def __init__(self, g, s, coloring, rank: int, world: int, bounds=None, comm=None,
                 outputs=None):
        import ctypes
        import torch
        from . import _lib
        self._lib = _lib
        d = s.device()
        dev = d["assignment"].device
        n = g.num_vertices
        self.g, self.s, self.d, self.rank, self.world = g, s, d, rank, world
        if coloring is not None:
            class_off, class_vtx = coloring.device_classes()
            self.stage_off = np.ascontiguousarray(class_off, dtype=np.int64)
            self.vtx = class_vtx
            flags = _lib.F_INDEPENDENT
        else:
            self.stage_off = np.array([0, n], dtype=np.int64)
            self.vtx = torch.arange(n, dtype=torch.int32, device=dev)
            flags = _lib.F_IDENTITY
        self.independent = coloring is not None
        if g.integral:
            flags |= _lib.F_INTEGRAL
        self.nstages = len(self.stage_off) - 1
        if bounds is None:
            bounds = partition_bounds(g.adjacency_offsets, world)
        self.bounds = np.ascontiguousarray(bounds, dtype=np.int64)
        total = int(self.stage_off[-1])
        if outputs is None and comm is None and world > 1:
            outputs = {
                "target": torch.empty(max(total, 1), dtype=torch.int32, device=dev),
                "moved": torch.empty(max(total, 1), dtype=torch.uint8, device=dev),
                "e_old": torch.empty(max(total, 1), dtype=torch.float64, device=dev),
                "e_best": torch.empty(max(total, 1), dtype=torch.float64, device=dev)}
        self.outputs = outputs
        o = outputs or {}
        self.handle = ctypes.c_void_p()
        _lib.check(_lib.lib().phase_create_part(
            _lib.ptr(g.d_off), _lib.ptr(g.d_nbr), _lib.ptr(g.d_w), _lib.ptr(g.d_k),
            _lib.ptr(g.d_selfw), n, g.total_weight, flags, _lib.ptr(d["labels"]),
            self.stage_off.ctypes.data, _lib.ptr(self.vtx), self.nstages,
            _lib.ptr(d["assignment"]), _lib.ptr(d["a_tot"]), _lib.ptr(d["w_internal"]),
            _lib.ptr(d["sizes"]), rank, world, self.bounds.ctypes.data, comm,
            _lib.ptr(o.get("target")), _lib.ptr(o.get("moved")), _lib.ptr(o.get("e_old")),
            _lib.ptr(o.get("e_best")), ctypes.byref(self.handle), _lib.stream()),
            "phase_create_part")
        self._q = _lib.f64_host(1)
        self._mv = _lib.i64_host(1)
        self._cand = _lib.i64_host(1)

    def slices(self) -> np.ndarray:
        """Per stage, the W + 1 slice bounds (relative to the stage start)."""
        return self._stages()[1]

    def engine_stage_off(self) -> np.ndarray:
        """Stage offsets into the engine's (active-vertex) stage lists."""
        return self._stages()[0]

    def _stages(self):
        so = np.empty(self.nstages + 1, np.int64)
        out = np.empty(self.nstages * (self.world + 1), np.int64)
        self._lib.check(self._lib.lib().phase_slices(self.handle, so.ctypes.data,
                                                     out.ctypes.data), "slices")
        return so, out.reshape(self.nstages, self.world + 1)

    def iterate(self):
        _lib = self._lib
        _lib.check(_lib.lib().phase_iterate(self.handle, _lib.hp(self._q), _lib.hp(self._mv),
                                            _lib.hp(self._cand), _lib.stream()), "phase_iterate")
        return float(self._q[0]), int(self._mv[0]), int(self._cand[0])

    def graph_kernels(self) -> int:
        """Kernel nodes of one iteration's CUDA graph (plv_phase_graph_kernels)."""
        _lib = self._lib
        out = _lib.i64_host(1)
        _lib.check(_lib.lib().phase_graph_kernels(self.handle, _lib.hp(out)), "graph_kernels")
        return int(out[0])

    def step(self, stage: int, op: int):
        _lib = self._lib
        _lib.check(_lib.lib().phase_step(self.handle, stage, op, _lib.hp(self._q),
                                         _lib.hp(self._mv), _lib.stream()), "phase_step")

    def finish(self):
        self.step(0, self._lib.STEP_FINISH)
        return float(self._q[0]), int(self._mv[0])

    def close(self):
        if self.handle:
            self._lib.lib().phase_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def stepped_iteration(engines):
    """One iteration of W host-stepped partitioned engines (one per virtual
    rank, same device): decide per rank, copy every slice to every other
    rank (the exchange), apply.  Returns [(q, moves)] per rank."""
    from . import _lib
    sl = [e.slices() for e in engines]
    off = engines[0].engine_stage_off()
    W = len(engines)
    def exchange(a):
        for r in range(W):
            lo, hi = int(off[a] + sl[r][a][r]), int(off[a] + sl[r][a][r + 1])
            if hi == lo:
                continue
            for q in range(W):
                if q != r:
                    for key in ("target", "moved", "e_old", "e_best"):
                        engines[q].outputs[key][lo:hi].copy_(engines[r].outputs[key][lo:hi])

    live = W > 1 and not engines[0].independent
    for a in range(engines[0].nstages):
        if off[a + 1] == off[a]:
            continue
        for e in engines:
            e.step(a, _lib.STEP_DECIDE)
        exchange(a)
        if live:  # uncoloured: each row owner folds its movers' live e_a / e_b
            for e in engines:
                e.step(a, _lib.STEP_LIVE)
            exchange(a)
        for e in engines:
            e.step(a, _lib.STEP_APPLY)
    return [e.finish() for e in engines]


class CudaStageOps:
    """Stage callbacks on the device (libplv): decide a slice of a stage with
    plv_decide_ex, apply a whole stage with plv_apply."""

    def __init__(self, g, state, stages, flags):
        import torch
        from . import _lib
        self._lib = _lib
        self.g, self.d = g, state.device()
        self.stages = stages          # list of device int32 tensors
        self.flags = flags | (_lib.F_INTEGRAL if g.integral else 0)
        dev = self.d["assignment"].device
        cap = max(1, max(int(s.numel()) for s in stages))
        self.tg = torch.empty(cap, dtype=torch.int32, device=dev)
        self.mv = torch.empty(cap, dtype=torch.uint8, device=dev)
        self.eo = torch.empty(cap, dtype=torch.float64, device=dev)
        self.eb = torch.empty(cap, dtype=torch.float64, device=dev)
        self.q = torch.empty(1, dtype=torch.float64, device=dev)

    def decide(self, a, lo, hi):
        L, g, d, _lib = self._lib.lib(), self.g, self.d, self._lib
        sub = self.stages[a][lo:hi]
        ns = hi - lo
        if ns:
            _lib.check(L.decide_ex(
                _lib.ptr(g.d_off), _lib.ptr(g.d_nbr), _lib.ptr(g.d_w), _lib.ptr(g.d_k),
                _lib.ptr(d["labels"]), _lib.ptr(sub), ns, _lib.ptr(d["assignment"]),
                _lib.ptr(d["a_tot"]), _lib.ptr(d["sizes"]), g.total_weight, self.flags,
                _lib.ptr(self.tg), _lib.ptr(self.mv), _lib.ptr(self.eo), _lib.ptr(self.eb),
                None, _lib.stream()), "decide")
        return DecideSlice(self.tg[:ns].clone(), self.mv[:ns].clone(), self.eo[:ns].clone(),
                           self.eb[:ns].clone())

    def apply(self, a, dfull):
        L, g, d, _lib = self._lib.lib(), self.g, self.d, self._lib
        sub = self.stages[a]
        moves = _lib.i64_host(1)
        _lib.check(L.apply(
            _lib.ptr(g.d_off), _lib.ptr(g.d_nbr), _lib.ptr(g.d_w), _lib.ptr(g.d_k),
            _lib.ptr(g.d_selfw), g.num_vertices, _lib.ptr(sub), int(sub.numel()),
            _lib.ptr(dfull.target), _lib.ptr(dfull.moved), _lib.ptr(dfull.e_old),
            _lib.ptr(dfull.e_best), self.flags, _lib.ptr(d["assignment"]), _lib.ptr(d["a_tot"]),
            _lib.ptr(d["w_internal"]), _lib.ptr(d["sizes"]), _lib.hp(moves), _lib.stream()),
            "apply")
        return int(moves[0])

    def modularity(self):
        from .modularity import CommunityState, modularity_device
        s = CommunityState.from_device(self.d["assignment"], self.d["a_tot"],
                                       self.d["w_internal"], self.d["sizes"], self.d["labels"])
        return float(modularity_device(self.g, s, self.q).item())
