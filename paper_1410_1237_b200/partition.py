"""The 1D vertex-partitioned multi-GPU pipeline (C5 = R-MAT s28).

The reference has no distributed mode (it is a single-process OpenMP
package); this is new design whose every output equals the single-graph
result bit for bit.  One process per GPU; rank r owns the vertices
[bounds[r], bounds[r+1]) and holds ONLY their rows (off is n+1 long with
empty rows elsewhere, nbr / w the owned entries).  Replicated on every rank:
the per-vertex graph scalars (k, self-loop weight, degree) and the community
state (assignment, a_tot, w_internal, sizes).  The kernels are libplv's
(csrc/part.cu and the phase engine); this module moves data between ranks:

* construction (Graph.from_edges, PL/graph.py:88-147): each rank generates a
  contiguous range of record draws; every record goes to the owner of each
  endpoint (all-to-all), so a rank's record list is the global list
  restricted to the records touching its rows, in global order; the ordinary
  device CSR build on it yields every owned row exactly; k / self loops /
  degrees are all-reduced from zero-padded vectors (x + 0 = x) and m is the
  pairwise sum of the replicated k;
* vertex following (PL/heuristics.py:46-89): candidates' single neighbours
  all-reduced, the survivor scan replicated, the compacted records built
  from owned rows (kept, then folded, as two ordered exchanges);
* colouring (PL/heuristics.py:92-118): speculative rounds; each rank assigns
  and checks its own active vertices against the replicated colours, the
  tentative colours and the rejects are all-gathered in rank (= id) order;
* local moving (PL/engine.py:140-216): the phase engine decides each rank's
  slice of every stage and exchanges the slices (one NCCL all-gather per stage
  inside the iteration's CUDA graph, or host-stepped over gloo), uncoloured
  stages fold their movers' live e_a / e_b on the row owners, and every rank
  applies whole stages exactly;
* rebuild (PL/engine.py:229-256): renumbering replicated, coarse records
  from owned rows, routed like construction records.

`Exchange` wraps a torch.distributed group: NCCL on device tensors, or gloo
through host copies (the multi-process tests on one GPU).
"""

from __future__ import annotations

import logging
import time
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .engine import RunConfig, _iteration_converged, _rel_gain

log = logging.getLogger(__name__)


# ---------------------------------------------------------------- exchange

class Exchange:
    """Collectives of the partitioned driver over a torch.distributed group."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.host = dist.get_backend(group) != "nccl"

    def _out(self, t):
        return t.cpu() if self.host else t

    def _back(self, t, like):
        return t.to(like.device) if self.host else t

    def all_to_all_v(self, tensors, send_counts):
        """Rank-ordered exchange: tensors[k] holds send_counts[d] rows for
        destination d, d ascending; returns the received tensors (sources in
        rank order) and the receive counts."""
        import torch
        sc = torch.tensor(send_counts, dtype=torch.int64)
        rc = torch.empty_like(sc)
        if self.host:
            self.dist.all_to_all_single(rc, sc, group=self.group)
        else:
            dev = tensors[0].device
            rcd = torch.empty(self.world, dtype=torch.int64, device=dev)
            self.dist.all_to_all_single(rcd, sc.to(dev), group=self.group)
            rc = rcd.cpu()
        recv = [int(x) for x in rc.tolist()]
        out = []
        for t in tensors:
            src = self._out(t)
            dst = torch.empty(sum(recv), dtype=t.dtype, device=src.device)
            self.dist.all_to_all_single(dst, src, recv, list(send_counts), group=self.group)
            out.append(self._back(dst, t))
        return out, recv

    def all_gather_v(self, t):
        """Concatenation over ranks (rank order) of 1-D tensors of any length."""
        lens = self.all_gather_int(int(t.numel()))
        (o,), _ = self.all_to_all_v([t.repeat(self.world)], [int(t.numel())] * self.world)
        assert o.numel() == sum(lens)
        return o

    def all_gather_int(self, x: int):
        import torch
        v = torch.tensor([x], dtype=torch.int64)
        if not self.host:
            v = v.cuda()
        parts = [torch.empty_like(v) for _ in range(self.world)]
        self.dist.all_gather(parts, v, group=self.group)
        return [int(p.item()) for p in parts]

    def all_reduce_(self, t, op="sum"):
        import torch
        ops = {"sum": self.dist.ReduceOp.SUM, "max": self.dist.ReduceOp.MAX,
               "min": self.dist.ReduceOp.MIN}
        if self.host:
            h = t.cpu()
            self.dist.all_reduce(h, op=ops[op], group=self.group)
            t.copy_(h)
        else:
            self.dist.all_reduce(t, op=ops[op], group=self.group)
        return t

    def sum_int(self, x: int) -> int:
        return sum(self.all_gather_int(int(x)))

    def max_int(self, x: int) -> int:
        return max(self.all_gather_int(int(x)))

    def barrier(self):
        self.dist.barrier(group=self.group)


# ------------------------------------------------------------ partitioning

def balanced_bounds(du, dv, n: int, ex: Exchange, buckets: int = 1 << 16) -> np.ndarray:
    """Contiguous vertex ranges with about equal adjacency entries, from the
    records' endpoint histogram (coarse buckets, all-reduced).  Any bounds give
    the same results; these balance the work."""
    import torch
    W = ex.world
    if n == 0 or W == 1:
        return np.array([0] + [n] * W, dtype=np.int64)
    width = max(1, -(-n // buckets))
    nb = -(-n // width)
    h = torch.zeros(nb, dtype=torch.int64, device=du.device)
    if du.numel():
        h += torch.bincount((du // width).long(), minlength=nb)
        h += torch.bincount((dv // width).long(), minlength=nb)
    ex.all_reduce_(h)
    c = torch.cumsum(h, 0).cpu().numpy()
    tot = c[-1]
    cuts = [int(np.searchsorted(c, tot * r / W, side="left")) + 1 for r in range(1, W)]
    b = np.array([0] + [min(n, x * width) for x in cuts] + [n], dtype=np.int64)
    return np.maximum.accumulate(b)


# ----------------------------------------------------------------- graph

@dataclass
class PartGraph:
    """This rank's part of a Graph (PL/graph.py:36-86) under a 1D partition."""
    num_vertices: int
    bounds: np.ndarray
    rank: int
    d_off: object            # int64 [n+1], empty rows outside [lo, hi)
    d_nbr: object            # int32 owned entries
    d_w: object              # f64 owned entries
    d_k: object              # f64 [n] replicated
    d_selfw: object          # f64 [n] replicated
    d_deg: object            # int32 [n] replicated
    total_weight: float
    num_edges: int
    max_degree: int
    integral: bool
    merged_duplicates: int = 0
    num_self_loops: int = 0

    @property
    def lo(self) -> int:
        return int(self.bounds[self.rank])

    @property
    def hi(self) -> int:
        return int(self.bounds[self.rank + 1])

    @property
    def nnz_local(self) -> int:
        return int(self.d_nbr.numel())


ROUTE_CHUNK = 1 << 30  # records per routing call (plv_route_records takes < 2^31)


def _route(du, dv, dw, bounds, ex: Exchange, chunk: int = ROUTE_CHUNK):
    """Every record to the owner of each endpoint.  Returns the received
    records in global order: per sender (rank order), that sender's records
    in input order -- reassembled across routing chunks."""
    import torch
    R = int(du.numel())
    dev = du.device
    db = torch.from_numpy(np.ascontiguousarray(bounds, dtype=np.int64)).to(dev)
    nchunks = max(1, ex.max_int(-(-R // chunk)))
    per_src = [[] for _ in range(ex.world)]
    for c in range(nchunks):
        a, b = min(R, c * chunk), min(R, (c + 1) * chunk)
        m = b - a
        ou = torch.empty(max(2 * m, 1), dtype=torch.int32, device=dev)
        ov = torch.empty_like(ou)
        ow = torch.empty(max(2 * m, 1), dtype=torch.float64, device=dev)
        cnt = _lib.i64_host(ex.world)
        _lib.check(_lib.lib().route_records(_lib.ptr(du) + 4 * a if m else None,
                                            _lib.ptr(dv) + 4 * a if m else None,
                                            _lib.ptr(dw) + 8 * a if m else None, m,
                                            _lib.ptr(db), ex.world, _lib.ptr(ou), _lib.ptr(ov),
                                            _lib.ptr(ow), 2 * m, _lib.hp(cnt), _lib.stream()),
                   "route_records")
        sc = [int(cnt[r]) for r in range(ex.world)]
        tot = sum(sc)
        (ru, rv, rw), recv = ex.all_to_all_v([ou[:tot], ov[:tot], ow[:tot]], sc)
        o = 0
        for src, k in enumerate(recv):
            per_src[src].append((ru[o:o + k], rv[o:o + k], rw[o:o + k]))
            o += k
    cat = lambda i: torch.cat([x[i] for src in per_src for x in src])  # noqa: E731
    return cat(0), cat(1), cat(2)


def from_records_part(segments, n: int, bounds, ex: Exchange, count_merges=True,
                      chunk: int = ROUTE_CHUNK) -> PartGraph:
    """Graph.from_edges (PL/graph.py:88-147) over the records of all ranks,
    this rank keeping its rows.  `segments`: list of (u, v, w) device tensors;
    the global record order is segment 0 of every rank (rank order), then
    segment 1 of every rank, ... (vf_compact's kept-then-folded order)."""
    import torch
    from .graph import Graph
    bounds = np.ascontiguousarray(bounds, dtype=np.int64)
    parts = [_route(u, v, w, bounds, ex, chunk) for (u, v, w) in segments]
    ru = torch.cat([p[0] for p in parts])
    rv = torch.cat([p[1] for p in parts])
    rw = torch.cat([p[2] for p in parts])
    R_total = ex.sum_int(sum(int(u.numel()) for (u, _, _) in segments))
    local = Graph.from_device_records(ru, rv, rw, n, count_merges=False)
    del ru, rv, rw
    lo, hi = int(bounds[ex.rank]), int(bounds[ex.rank + 1])
    dev = local.d_off.device
    off = torch.empty(n + 1, dtype=torch.int64, device=dev)
    cap = max(1, int(local.d_nbr.numel()))
    nbr = torch.empty(cap, dtype=torch.int32, device=dev)
    w = torch.empty(cap, dtype=torch.float64, device=dev)
    deg = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
    info = _lib.i64_host(5)
    _lib.check(_lib.lib().part_own_rows(_lib.ptr(local.d_off), _lib.ptr(local.d_nbr),
                                        _lib.ptr(local.d_w), n, lo, hi, _lib.ptr(off),
                                        _lib.ptr(nbr), _lib.ptr(w), _lib.ptr(deg), _lib.hp(info),
                                        _lib.stream()), "part_own_rows")
    entries, num_self, pairs, maxdeg, frac = (int(info[t]) for t in range(5))
    nbr = nbr[:entries].clone()
    w = w[:entries].clone()
    k = local.d_k.clone()
    selfw = local.d_selfw.clone()
    del local
    for t in (k, selfw, deg):  # zero outside the owned rows, then replicate
        t[:lo] = 0
        t[hi:n] = 0
    ex.all_reduce_(k)
    ex.all_reduce_(selfw)
    ex.all_reduce_(deg)
    msum = torch.empty(1, dtype=torch.float64, device=dev)
    _lib.check(_lib.lib().sum(_lib.ptr(k), n, _lib.ptr(msum), _lib.stream()), "sum")
    m = float(msum.item()) / 2.0
    tot_entries = ex.sum_int(entries)
    tot_self = ex.sum_int(num_self)
    tot_pairs = ex.sum_int(pairs)
    merged = R_total - tot_pairs
    if merged and count_merges and ex.rank == 0:
        log.warning("merged %d duplicate edge records", merged)
    integral = ex.sum_int(frac) == 0 and 2.0 * m < 4503599627370496.0
    return PartGraph(n, bounds, ex.rank, off, nbr, w, k, selfw, deg, m,
                     (tot_entries + tot_self) // 2, ex.max_int(maxdeg), integral,
                     merged if count_merges else 0, tot_self)


def rmat_part(scale: int, ex: Exchange, edge_factor: int = 16, seed: int = 0,
              abc=(0.57, 0.19, 0.19), w_lo: float = 1.0, w_hi: float = 10.0):
    """This rank's contiguous range of R-MAT record draws (synthetic.rmat_records
    restricted); the ranges of all ranks concatenate to the whole list."""
    import torch
    R = edge_factor << scale
    r0 = R * ex.rank // ex.world
    r1 = R * (ex.rank + 1) // ex.world
    dev = _lib.device()
    cap = max(1, r1 - r0)
    u = torch.empty(cap, dtype=torch.int32, device=dev)
    v = torch.empty_like(u)
    w = torch.empty(cap, dtype=torch.float64, device=dev)
    cnt = _lib.i64_host(1)
    a, b, c = abc
    _lib.check(_lib.lib().gen_rmat_range(seed, scale, edge_factor, a, b, c, w_lo, w_hi, r0, r1,
                                         _lib.ptr(u), _lib.ptr(v), _lib.ptr(w), cap,
                                         _lib.hp(cnt), _lib.stream()), "gen_rmat_range")
    k = int(cnt[0])
    return u[:k], v[:k], w[:k], 1 << scale


def rmat_graph_part(scale: int, ex: Exchange, chunk: int = ROUTE_CHUNK, **kw) -> PartGraph:
    u, v, w, n = rmat_part(scale, ex, **kw)
    bounds = balanced_bounds(u, v, n, ex)
    return from_records_part([(u, v, w)], n, bounds, ex, chunk=chunk)


# ---------------------------------------------------------- vertex following

@dataclass
class PartVf:
    vertex_map: object  # int32 [n] replicated
    graph: PartGraph
    merged_count: int


def vf_compact_part(g: PartGraph, ex: Exchange) -> PartVf:
    """vf_compact (PL/heuristics.py:46-89) on a partitioned graph."""
    import torch
    n = g.num_vertices
    dev = g.d_off.device
    L = _lib.lib()
    only = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
    _lib.check(L.part_vf_only(_lib.ptr(g.d_off), _lib.ptr(g.d_nbr), _lib.ptr(g.d_deg),
                              _lib.ptr(g.d_selfw), n, g.lo, g.hi, _lib.ptr(only), _lib.stream()),
               "part_vf_only")
    ex.all_reduce_(only)
    merged = torch.empty(max(n, 1), dtype=torch.uint8, device=dev)
    new_id = torch.empty(n + 1, dtype=torch.int32, device=dev)
    vmap = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
    info = _lib.i64_host(2)
    _lib.check(L.part_vf_map(_lib.ptr(only), n, _lib.ptr(merged), _lib.ptr(new_id),
                             _lib.ptr(vmap), _lib.hp(info), _lib.stream()), "part_vf_map")
    n_new, merged_count = int(info[0]), int(info[1])
    cap = max(1, g.nnz_local)
    capf = max(1, g.hi - g.lo)
    ku = torch.empty(cap, dtype=torch.int32, device=dev)
    kv = torch.empty_like(ku)
    kw = torch.empty(cap, dtype=torch.float64, device=dev)
    fu = torch.empty(capf, dtype=torch.int32, device=dev)
    fv = torch.empty_like(fu)
    fw = torch.empty(capf, dtype=torch.float64, device=dev)
    cnt = _lib.i64_host(2)
    _lib.check(L.part_vf_records(_lib.ptr(g.d_off), _lib.ptr(g.d_nbr), _lib.ptr(g.d_w), n,
                                 g.lo, g.hi, _lib.ptr(merged), _lib.ptr(new_id), _lib.ptr(only),
                                 _lib.ptr(ku), _lib.ptr(kv), _lib.ptr(kw), _lib.ptr(fu),
                                 _lib.ptr(fv), _lib.ptr(fw), _lib.hp(cnt), _lib.stream()),
               "part_vf_records")
    nk, nf = int(cnt[0]), int(cnt[1])
    # a vertex keeps its owner: the new partition is the old one renumbered
    nb = new_id[torch.from_numpy(g.bounds).to(dev)].cpu().numpy().astype(np.int64)
    nb[-1] = n_new
    cg = from_records_part([(ku[:nk], kv[:nk], kw[:nk]), (fu[:nf], fv[:nf], fw[:nf])], n_new,
                           nb, ex, count_merges=False)
    return PartVf(vmap[:n], cg, merged_count)


# ----------------------------------------------------------------- colouring

def color_part(g: PartGraph, ex: Exchange):
    """color_graph (PL/heuristics.py:92-118) on a partitioned graph: the
    replicated colouring (heuristics.Coloring) and the number of rounds."""
    import torch
    from .heuristics import Coloring
    n = g.num_vertices
    dev = g.d_off.device
    L = _lib.lib()
    colors = torch.full((max(n, 1),), -1, dtype=torch.int32, device=dev)
    active = torch.arange(n, dtype=torch.int32, device=dev)
    lohi = torch.tensor([g.lo, g.hi], dtype=torch.int32, device=dev)
    rounds = 0
    cnt = _lib.i64_host(1)
    while active.numel():
        rounds += 1
        a0, a1 = (int(x) for x in torch.searchsorted(active, lohi).cpu().tolist())
        own = active[a0:a1].contiguous()
        na = int(own.numel())
        tent = torch.empty(max(na, 1), dtype=torch.int32, device=dev)
        if na:
            _lib.check(L.color_assign(_lib.ptr(g.d_off), _lib.ptr(g.d_nbr), _lib.ptr(own), na,
                                      _lib.ptr(colors), _lib.ptr(tent), _lib.stream()),
                       "color_assign")
        tent_all = ex.all_gather_v(tent[:na])
        _lib.check(L.scatter_i32(_lib.ptr(active), _lib.ptr(tent_all), 0, int(active.numel()),
                                 _lib.ptr(colors), _lib.stream()), "scatter")
        keep = torch.empty(max(na, 1), dtype=torch.uint8, device=dev)
        rej = torch.empty(max(na, 1), dtype=torch.int32, device=dev)
        nr = 0
        if na:
            _lib.check(L.color_conflicts(_lib.ptr(g.d_off), _lib.ptr(g.d_nbr), _lib.ptr(own), na,
                                         _lib.ptr(colors), _lib.ptr(keep), _lib.stream()),
                       "color_conflicts")
            _lib.check(L.select_rejected(_lib.ptr(own), _lib.ptr(keep), na, _lib.ptr(rej),
                                         _lib.hp(cnt), _lib.stream()), "select_rejected")
            nr = int(cnt[0])
        active = ex.all_gather_v(rej[:nr]).contiguous()
        if active.numel():
            _lib.check(L.scatter_i32(_lib.ptr(active), None, -1, int(active.numel()),
                                     _lib.ptr(colors), _lib.stream()), "scatter")
    num_colors = int(colors[:n].max().item()) + 1 if n else 0
    return Coloring(colors[:n], num_colors, rounds)


# -------------------------------------------------------------- local moving

@dataclass
class PartPhaseStats:
    iterations: int
    total_moves: int
    q_end: float
    theta: float
    colored: bool
    hit_iteration_cap: bool
    q_trace: list = field(default_factory=list)


class PartEngine:
    """The phase engine on this rank of the partition (plv_phase_create_part2).
    With an NCCL communicator one iteration is one graph launch (decide,
    all-gathers, live folds, applies, Q); without one (gloo) the stages are
    stepped from the host and the slices move through `ex`."""

    def __init__(self, g: PartGraph, state, coloring, ex: Exchange, comm=None):
        import ctypes
        import torch
        self.g, self.s, self.ex, self.comm = g, state, ex, comm
        d = state.device()
        dev = d["assignment"].device
        n = g.num_vertices
        self.d = d
        if coloring is not None:
            off, vtx = coloring.device_classes()
            self.stage_off = np.ascontiguousarray(off, dtype=np.int64)
            self.vtx = vtx
            flags = _lib.F_INDEPENDENT
        else:
            self.stage_off = np.array([0, n], dtype=np.int64)
            self.vtx = torch.arange(n, dtype=torch.int32, device=dev)
            flags = _lib.F_IDENTITY
        if g.integral:
            flags |= _lib.F_INTEGRAL
        self.flags = flags
        self.nstages = len(self.stage_off) - 1
        total = int(self.stage_off[-1])
        self.out = {"target": torch.empty(max(total, 1), dtype=torch.int32, device=dev),
                    "moved": torch.empty(max(total, 1), dtype=torch.uint8, device=dev),
                    "e_old": torch.empty(max(total, 1), dtype=torch.float64, device=dev),
                    "e_best": torch.empty(max(total, 1), dtype=torch.float64, device=dev)}
        self.bounds = np.ascontiguousarray(g.bounds, dtype=np.int64)
        self.handle = ctypes.c_void_p()
        o = self.out
        _lib.check(_lib.lib().phase_create_part2(
            _lib.ptr(g.d_off), _lib.ptr(g.d_nbr), _lib.ptr(g.d_w), _lib.ptr(g.d_k),
            _lib.ptr(g.d_selfw), n, g.total_weight, flags, _lib.ptr(d["labels"]),
            self.stage_off.ctypes.data, _lib.ptr(self.vtx), self.nstages,
            _lib.ptr(d["assignment"]), _lib.ptr(d["a_tot"]), _lib.ptr(d["w_internal"]),
            _lib.ptr(d["sizes"]), ex.rank, ex.world, self.bounds.ctypes.data, comm,
            _lib.ptr(g.d_deg), _lib.ptr(o["target"]), _lib.ptr(o["moved"]), _lib.ptr(o["e_old"]),
            _lib.ptr(o["e_best"]), ctypes.byref(self.handle), _lib.stream()),
            "phase_create_part2")
        so = np.empty(self.nstages + 1, np.int64)
        sl = np.empty(max(1, self.nstages * (ex.world + 1)), np.int64)
        _lib.check(_lib.lib().phase_slices(self.handle, so.ctypes.data, sl.ctypes.data),
                   "phase_slices")
        self.eoff = so
        self.slices = sl[:self.nstages * (ex.world + 1)].reshape(self.nstages, ex.world + 1)
        self._q = _lib.f64_host(1)
        self._mv = _lib.i64_host(1)
        self._cand = _lib.i64_host(1)

    def _exchange(self, a: int):
        """Stage a: every rank's decided slice to every rank (gloo path)."""
        import torch
        W, r = self.ex.world, self.ex.rank
        if W == 1:
            return
        g0 = int(self.eoff[a])
        sl = self.slices[a]
        lo, hi = g0 + int(sl[r]), g0 + int(sl[r + 1])
        o = self.out
        rec = torch.cat([o["target"][lo:hi].view(torch.uint8),
                         o["moved"][lo:hi].view(torch.uint8),
                         o["e_old"][lo:hi].view(torch.uint8),
                         o["e_best"][lo:hi].view(torch.uint8)])
        allrec = self.ex.all_gather_v(rec)
        p = 0
        for q in range(W):
            c = int(sl[q + 1] - sl[q])
            nbytes = c * (4 + 1 + 8 + 8)
            if q != r and c:
                blk = allrec[p:p + nbytes]
                s0 = g0 + int(sl[q])
                o["target"][s0:s0 + c].view(torch.uint8).copy_(blk[:4 * c])
                o["moved"][s0:s0 + c].copy_(blk[4 * c:5 * c])
                o["e_old"][s0:s0 + c].view(torch.uint8).copy_(blk[5 * c:13 * c])
                o["e_best"][s0:s0 + c].view(torch.uint8).copy_(blk[13 * c:21 * c])
            p += nbytes

    def _step(self, a: int, op: int):
        _lib.check(_lib.lib().phase_step(self.handle, a, op, _lib.hp(self._q), _lib.hp(self._mv),
                                         _lib.stream()), "phase_step")

    def iterate(self):
        """One local-move iteration (every stage, then Q): (q, moves, cand)."""
        L = _lib.lib()
        if self.comm is not None:
            _lib.check(L.phase_iterate(self.handle, _lib.hp(self._q), _lib.hp(self._mv),
                                       _lib.hp(self._cand), _lib.stream()), "phase_iterate")
            return float(self._q[0]), int(self._mv[0]), int(self._cand[0])
        live = not (self.flags & _lib.F_INDEPENDENT) and self.ex.world > 1
        for a in range(self.nstages):
            if self.eoff[a + 1] == self.eoff[a]:
                continue
            self._step(a, _lib.STEP_DECIDE)
            self._exchange(a)
            if live:
                self._step(a, _lib.STEP_LIVE)
                self._exchange(a)
            self._step(a, _lib.STEP_APPLY)
        self._step(0, _lib.STEP_FINISH)
        return float(self._q[0]), int(self._mv[0]), 0

    def graph_kernels(self) -> int:
        out = _lib.i64_host(1)
        _lib.check(_lib.lib().phase_graph_kernels(self.handle, _lib.hp(out)), "graph_kernels")
        return int(out[0])

    def close(self):
        if self.handle:
            _lib.lib().phase_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def singleton_state_part(g: PartGraph):
    """singleton_state (PL/modularity.py:47-56), replicated on every rank."""
    import torch
    from .modularity import CommunityState
    n = g.num_vertices
    dev = g.d_k.device
    assign = torch.arange(n, dtype=torch.int32, device=dev)
    sizes = torch.ones(n, dtype=torch.int32, device=dev)
    return CommunityState.from_device(assign, g.d_k.clone(), 2.0 * g.d_selfw, sizes)


def run_phase_part(g: PartGraph, cfg: RunConfig, coloring, ex: Exchange, comm=None):
    """run_phase (PL/engine.py:166-216) on the partition; the stopping rule
    on the host, every rank reaching the same decision from replicated Q."""
    s = singleton_state_part(g)
    theta = cfg.theta_color if coloring is not None else cfg.theta_final
    eng = PartEngine(g, s, coloring, ex, comm)
    q_prev = None
    it = total = 0
    hit = False
    qs = []
    try:
        while True:
            q_cur, moves, _ = eng.iterate()
            it += 1
            total += moves
            qs.append(q_cur)
            if moves == 0:
                break
            if q_prev is not None and _iteration_converged(q_cur, q_prev, theta):
                break
            if it >= cfg.max_iterations_per_phase:
                hit = True
                break
            q_prev = q_cur
    finally:
        eng.close()
    return s, PartPhaseStats(it, total, q_cur, theta, coloring is not None, hit, qs)


def rebuild_part(g: PartGraph, s, ex: Exchange):
    """rebuild (PL/engine.py:229-256) on the partition: (coarse PartGraph,
    renumber int32 device tensor, replicated)."""
    import torch
    n = g.num_vertices
    dev = g.d_off.device
    L = _lib.lib()
    d = s.device()
    ren = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
    nn = _lib.i64_host(1)
    _lib.check(L.renumber(_lib.ptr(d["assignment"]), n, _lib.ptr(ren), _lib.hp(nn),
                          _lib.stream()), "renumber")
    n_new = int(nn[0])
    cap = max(1, g.nnz_local)
    ou = torch.empty(cap, dtype=torch.int32, device=dev)
    ov = torch.empty_like(ou)
    ow = torch.empty(cap, dtype=torch.float64, device=dev)
    cnt = _lib.i64_host(1)
    _lib.check(L.part_rebuild_records(_lib.ptr(g.d_off), _lib.ptr(g.d_nbr), _lib.ptr(g.d_w), n,
                                      g.lo, g.hi, _lib.ptr(d["assignment"]), _lib.ptr(ren),
                                      _lib.ptr(ou), _lib.ptr(ov), _lib.ptr(ow), _lib.hp(cnt),
                                      _lib.stream()), "part_rebuild_records")
    k = int(cnt[0])
    # coarse bounds: the communities with ids below each old bound
    present = (ren[:n] >= 0).to(torch.int64)
    csum = torch.cat([torch.zeros(1, dtype=torch.int64, device=dev), torch.cumsum(present, 0)])
    nb = csum[torch.from_numpy(g.bounds).to(dev)].cpu().numpy().astype(np.int64)
    nb[-1] = n_new
    cg = from_records_part([(ou[:k], ov[:k], ow[:k])], n_new, nb, ex, count_merges=False)
    return cg, ren[:n]


@dataclass
class PartHierarchy:
    phases: list
    vertex_map: object
    final_assignment: object  # int32 device tensor, replicated
    final_modularity: float
    num_communities: int
    seconds: dict = field(default_factory=dict)


def run_part(g: PartGraph, ex: Exchange, cfg: RunConfig | None = None, comm=None):
    """run (PL/engine.py:259-315) on the partition (VF, colouring policy,
    phases, rebuilds, flattening); every rank returns the same hierarchy."""
    import torch
    cfg = (cfg or RunConfig()).validate()
    secs = {}
    t0 = time.perf_counter()
    current = g
    vmap = None
    if cfg.use_vf:
        vf = vf_compact_part(g, ex)
        vmap = vf.vertex_map
        current = vf.graph
    secs["vf"] = time.perf_counter() - t0
    s0 = singleton_state_part(current)
    from .modularity import modularity_device
    q_prev_phase = float(modularity_device(current, s0).item())
    coloring_enabled = cfg.use_coloring
    phases = []
    while True:
        if coloring_enabled and current.num_vertices < cfg.color_cutoff:
            coloring_enabled = False
        t1 = time.perf_counter()
        coloring = color_part(current, ex) if coloring_enabled else None
        secs.setdefault("coloring", 0.0)
        secs["coloring"] += time.perf_counter() - t1
        t1 = time.perf_counter()
        s, st = run_phase_part(current, cfg, coloring, ex, comm)
        secs.setdefault("phases", 0.0)
        secs["phases"] += time.perf_counter() - t1
        t1 = time.perf_counter()
        rebuilt, ren = rebuild_part(current, s, ex)
        secs.setdefault("rebuild", 0.0)
        secs["rebuild"] += time.perf_counter() - t1
        phases.append((s.device()["assignment"], ren, st))
        gain = _rel_gain(st.q_end, q_prev_phase)
        if coloring_enabled and gain < cfg.theta_color:
            coloring_enabled = False
        q_prev_phase = st.q_end
        current = rebuilt
        if st.total_moves == 0 or gain < cfg.theta_final:
            break
    n0 = g.num_vertices
    dev = g.d_off.device
    v = vmap if vmap is not None else torch.arange(n0, dtype=torch.int32, device=dev)
    L = _lib.lib()
    for (assign, ren, _) in phases:
        out = torch.empty(max(n0, 1), dtype=torch.int32, device=dev)
        _lib.check(L.compose(_lib.ptr(v), _lib.ptr(assign), _lib.ptr(ren), n0, _lib.ptr(out),
                             _lib.stream()), "compose")
        v = out[:n0]
    return PartHierarchy([p[2] for p in phases], vmap, v, phases[-1][2].q_end,
                         current.num_vertices, secs)
