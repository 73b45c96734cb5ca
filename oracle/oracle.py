"""CPU oracle for the parallel-Louvain hot path (TEST INFRASTRUCTURE ONLY).

Python driver over ``liborc.so`` (plv_oracle.c).  It restates the reference's
engine (PL/engine.py) and graph core (PL/graph.py) so that tests and the bench's
CPU-baseline leg have a fast, dependency-free checker.  Nothing in the product
package imports this module; only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py`` (cpu_baseline / --impl reference) may.

Citations: PL/ = /root/reference/pkg/src/parlouvain/.
Pinned against the compiled reference by tests/test_oracle_pins.py.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None

_i64p = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_u8p = np.ctypeslib.ndpointer(dtype=np.uint8, flags="C_CONTIGUOUS")
_i64 = ctypes.c_int64


def build() -> str:
    """Compile liborc.so (plain gcc; used by __graft_entry__.build())."""
    subprocess.run(["make", "-s", "-C", _HERE, "CC=/usr/bin/gcc"], check=True)
    return os.path.join(_HERE, "liborc.so")


def lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(_HERE, "liborc.so")
        src = os.path.join(_HERE, "plv_oracle.c")
        if not os.path.exists(path) or os.path.getmtime(path) < os.path.getmtime(src):
            build()
        L = ctypes.CDLL(path)
        L.orc_sum.restype = ctypes.c_double
        L.orc_sum.argtypes = [_f64p, _i64]
        L.orc_from_edges.restype = ctypes.c_int
        L.orc_from_edges.argtypes = [_i64p, _i64p, _f64p, _i64, _i64, _i64p, _i64p,
                                     _f64p, _f64p, _f64p, _i64p,
                                     ctypes.POINTER(ctypes.c_double)]
        L.orc_edge_records.restype = _i64
        L.orc_edge_records.argtypes = [_i64, _i64p, _i64p, _f64p, _i64p, _i64p, _f64p]
        L.orc_vf_records.restype = ctypes.c_int
        L.orc_vf_records.argtypes = [_i64, _i64p, _i64p, _f64p, _f64p, _i64p, _i64p,
                                     _i64p, _f64p, _i64p]
        L.orc_color.restype = _i64
        L.orc_color.argtypes = [_i64, _i64p, _i64p, _i64, _i64p]
        L.orc_run_iteration.restype = _i64
        L.orc_run_iteration.argtypes = [_i64, _i64p, _i64p, _f64p, _f64p, _f64p,
                                        ctypes.c_double, ctypes.c_void_p, _i64p, _i64,
                                        _i64p, _f64p, _f64p, _i64p, ctypes.c_void_p,
                                        ctypes.c_void_p]
        L.orc_decide.restype = None
        L.orc_decide.argtypes = [_i64, _i64p, _i64p, _f64p, _f64p, ctypes.c_double,
                                 ctypes.c_void_p, _i64p, _i64, _i64p, _f64p, _i64p, _i64p, _u8p]
        L.orc_apply.restype = _i64
        L.orc_apply.argtypes = [_i64p, _i64p, _f64p, _f64p, _f64p, _i64p, _i64, _i64p, _u8p,
                                _i64p, _f64p, _f64p, _i64p]
        L.orc_modularity.restype = ctypes.c_double
        L.orc_modularity.argtypes = [_i64, _f64p, _f64p, ctypes.c_double]
        L.orc_rebuild_records.restype = ctypes.c_int
        L.orc_rebuild_records.argtypes = [_i64, _i64p, _i64p, _f64p, _i64p, _i64p,
                                          _i64p, _i64p, _f64p, _i64p]
        _LIB = L
    return _LIB


def np_sum(a) -> float:
    """ndarray.sum() restated (numpy pairwise tree)."""
    a = np.ascontiguousarray(a, dtype=np.float64)
    return float(lib().orc_sum(a, len(a)))


@dataclass
class OGraph:
    """CSR arrays with the reference's dtypes (PL/graph.py:36-86)."""
    num_vertices: int
    adjacency_offsets: np.ndarray
    neighbors: np.ndarray
    weights: np.ndarray
    self_loop_weights: np.ndarray
    weighted_degrees: np.ndarray
    total_weight: float
    num_edges: int
    max_degree: int
    merged_duplicates: int = 0

    def edge_records(self):
        n = self.num_vertices
        cap = len(self.neighbors) + 1
        a = np.empty(cap, np.int64)
        b = np.empty(cap, np.int64)
        w = np.empty(cap, np.float64)
        t = lib().orc_edge_records(n, self.adjacency_offsets, self.neighbors,
                                   self.weights, a, b, w)
        return a[:t], b[:t], w[:t]

    def same_as(self, other) -> bool:
        return (self.num_vertices == other.num_vertices
                and self.num_edges == other.num_edges
                and self.total_weight == other.total_weight
                and np.array_equal(np.asarray(self.adjacency_offsets),
                                   np.asarray(other.adjacency_offsets))
                and np.array_equal(np.asarray(self.neighbors), np.asarray(other.neighbors))
                and np.array_equal(np.asarray(self.weights), np.asarray(other.weights)))


def from_edges(u, v, w=None, num_vertices=None, count_merges=True) -> OGraph:
    """Graph.from_edges (PL/graph.py:88-147) + Graph.__init__ (:64-86)."""
    u = np.ascontiguousarray(u, dtype=np.int64)
    v = np.ascontiguousarray(v, dtype=np.int64)
    w = (np.ones(len(u)) if w is None else np.ascontiguousarray(w, dtype=np.float64))
    if num_vertices is None:
        num_vertices = int(max(u.max(), v.max()) + 1) if len(u) else 0
    n = int(num_vertices)
    R = len(u)
    off = np.empty(n + 1, np.int64)
    nbr = np.empty(2 * R + 1, np.int64)
    wts = np.empty(2 * R + 1, np.float64)
    selfw = np.empty(n + 1, np.float64)
    k = np.empty(n + 1, np.float64)
    info = np.zeros(4, np.int64)
    m = ctypes.c_double()
    lib().orc_from_edges(u, v, w, R, n, off, nbr, wts, selfw, k, info, ctypes.byref(m))
    nnz = int(info[0])
    return OGraph(n, off, nbr[:nnz].copy(), wts[:nnz].copy(), selfw[:n].copy(),
                  k[:n].copy(), float(m.value), int(info[2]), int(info[3]),
                  int(info[1]) if count_merges else 0)


@dataclass
class OState:
    """CommunityState (PL/modularity.py:21-56)."""
    assignment: np.ndarray
    labels: np.ndarray
    a_tot: np.ndarray
    w_internal: np.ndarray
    sizes: np.ndarray

    def copy(self):
        return OState(self.assignment.copy(), self.labels.copy(), self.a_tot.copy(),
                      self.w_internal.copy(), self.sizes.copy())


def singleton_state(g: OGraph) -> OState:
    n = g.num_vertices
    return OState(np.arange(n, dtype=np.int64), np.arange(n, dtype=np.int64),
                  g.weighted_degrees.copy(), 2.0 * g.self_loop_weights,
                  np.ones(n, dtype=np.int64))


def modularity(g: OGraph, s: OState) -> float:
    return float(lib().orc_modularity(g.num_vertices, s.w_internal, s.a_tot,
                                      g.total_weight))


def run_iteration(g: OGraph, s: OState, vertices, want_decisions=False):
    """run_iteration (PL/engine.py:140-163); mutates s in place."""
    subset = np.ascontiguousarray(vertices, dtype=np.int64)
    ns = len(subset)
    tg = np.empty(ns + 1, np.int64) if want_decisions else None
    mv = np.empty(ns + 1, np.uint8) if want_decisions else None
    labels = s.labels
    lab_ptr = None
    if not np.array_equal(labels, np.arange(len(labels))):
        labels = np.ascontiguousarray(labels, dtype=np.int64)
        lab_ptr = labels.ctypes.data
    cnt = lib().orc_run_iteration(
        g.num_vertices, g.adjacency_offsets, g.neighbors, g.weights,
        g.weighted_degrees, g.self_loop_weights, g.total_weight, lab_ptr, subset, ns,
        s.assignment, s.a_tot, s.w_internal, s.sizes,
        tg.ctypes.data if tg is not None else None,
        mv.ctypes.data if mv is not None else None)
    if want_decisions:
        return int(cnt), tg[:ns], mv[:ns]
    return int(cnt)


def decide(g: OGraph, s: OState, vertices):
    """decide_moves (PL/_kernels.pyx:21-101) alone: (targets, moved)."""
    subset = np.ascontiguousarray(vertices, dtype=np.int64)
    ns = len(subset)
    tg = np.empty(ns + 1, np.int64)
    mv = np.empty(ns + 1, np.uint8)
    lib().orc_decide(g.num_vertices, g.adjacency_offsets, g.neighbors, g.weights,
                     g.weighted_degrees, g.total_weight, None, subset, ns, s.assignment,
                     s.a_tot, s.sizes, tg, mv)
    return tg[:ns], mv[:ns]


def apply(g: OGraph, s: OState, vertices, targets, moved) -> int:
    """apply_moves (PL/_kernels.pyx:104-145) alone; mutates s."""
    subset = np.ascontiguousarray(vertices, dtype=np.int64)
    return int(lib().orc_apply(g.adjacency_offsets, g.neighbors, g.weights, g.weighted_degrees,
                               g.self_loop_weights, subset, len(subset),
                               np.ascontiguousarray(targets, dtype=np.int64),
                               np.ascontiguousarray(moved, dtype=np.uint8), s.assignment,
                               s.a_tot, s.w_internal, s.sizes))


@dataclass
class OColoring:
    colors: np.ndarray
    num_colors: int
    class_sizes: np.ndarray
    rounds: int = 0

    def classes(self):
        order = np.argsort(self.colors, kind="stable")
        bounds = np.cumsum(self.class_sizes)
        return np.split(order, bounds[:-1])


def color_graph(g: OGraph) -> OColoring:
    """color_graph (PL/heuristics.py:92-118)."""
    colors = np.empty(g.num_vertices + 1, np.int64)
    rounds = lib().orc_color(g.num_vertices, g.adjacency_offsets, g.neighbors,
                             g.max_degree, colors)
    colors = colors[:g.num_vertices].copy()
    nc = int(colors.max()) + 1 if g.num_vertices else 0
    return OColoring(colors, nc, np.bincount(colors, minlength=nc), int(rounds))


@dataclass
class OVf:
    vertex_map: np.ndarray
    graph: OGraph
    merged_count: int


def vf_compact(g: OGraph) -> OVf:
    """vf_compact (PL/heuristics.py:46-89)."""
    n = g.num_vertices
    cap = len(g.neighbors) + n + 1
    vmap = np.empty(n + 1, np.int64)
    ru = np.empty(cap, np.int64)
    rv = np.empty(cap, np.int64)
    rw = np.empty(cap, np.float64)
    info = np.zeros(3, np.int64)
    lib().orc_vf_records(n, g.adjacency_offsets, g.neighbors, g.weights,
                         g.self_loop_weights, vmap, ru, rv, rw, info)
    t = int(info[2])
    cg = from_edges(ru[:t], rv[:t], rw[:t], num_vertices=int(info[0]), count_merges=False)
    return OVf(vmap[:n].copy(), cg, int(info[1]))


def rebuild(g: OGraph, s: OState):
    """rebuild (PL/engine.py:229-256)."""
    n = g.num_vertices
    cap = len(g.neighbors) + 1
    ren = np.empty(n + 1, np.int64)
    lo = np.empty(cap, np.int64)
    hi = np.empty(cap, np.int64)
    w = np.empty(cap, np.float64)
    info = np.zeros(2, np.int64)
    lib().orc_rebuild_records(n, g.adjacency_offsets, g.neighbors, g.weights,
                              np.ascontiguousarray(s.assignment, dtype=np.int64),
                              ren, lo, hi, w, info)
    M = int(info[1])
    rebuilt = from_edges(lo[:M], hi[:M], w[:M], num_vertices=int(info[0]),
                         count_merges=False)
    return rebuilt, ren[:n].copy()


# ---------------------------------------------------------------- engine

_ZERO_GUARD = 1e-15


def _rel_gain(q_new, q_old):
    if abs(q_old) < _ZERO_GUARD:
        return q_new - q_old
    return (q_new - q_old) / abs(q_old)


def _converged(q_cur, q_prev, theta):
    if abs(q_prev) < _ZERO_GUARD:
        return abs(q_cur - q_prev) < theta
    return abs(q_cur - q_prev) / abs(q_prev) < theta


@dataclass
class OPhase:
    assignment: np.ndarray
    renumber: np.ndarray
    iterations: int
    total_moves: int
    q_end: float
    theta: float
    colored: bool
    hit_cap: bool
    q_trace: list = field(default_factory=list)
    moves_trace: list = field(default_factory=list)
    num_colors: int = 0


@dataclass
class OHierarchy:
    phases: list
    vf: OVf | None
    final_assignment: np.ndarray
    final_modularity: float
    num_communities: int


def run_phase(g: OGraph, theta_final=1e-6, theta_color=1e-2, max_iterations=10_000,
              coloring: OColoring | None = None):
    """run_phase (PL/engine.py:166-216)."""
    s = singleton_state(g)
    theta = theta_color if coloring is not None else theta_final
    stages = coloring.classes() if coloring is not None else None
    everything = np.arange(g.num_vertices, dtype=np.int64)
    q_prev = None
    it = 0
    total = 0
    hit = False
    qs, ms = [], []
    while True:
        if stages is None:
            moves = run_iteration(g, s, everything)
        else:
            moves = 0
            for st in stages:
                moves += run_iteration(g, s, st)
        it += 1
        total += moves
        q_cur = modularity(g, s)
        qs.append(q_cur)
        ms.append(moves)
        if moves == 0:
            break
        if q_prev is not None and _converged(q_cur, q_prev, theta):
            break
        if it >= max_iterations:
            hit = True
            break
        q_prev = q_cur
    return s, dict(iterations=it, total_moves=total, q_end=q_cur, theta=theta,
                   colored=coloring is not None, hit_cap=hit, q_trace=qs, moves_trace=ms)


def run(g: OGraph, theta_final=1e-6, theta_color=1e-2, color_cutoff=100_000, use_vf=True,
        use_coloring=True, max_iterations=10_000) -> OHierarchy:
    """run (PL/engine.py:259-315)."""
    current = g
    vf = None
    if use_vf:
        vf = vf_compact(g)
        current = vf.graph
    q_prev_phase = modularity(current, singleton_state(current))
    coloring_enabled = use_coloring
    phases = []
    while True:
        if coloring_enabled and current.num_vertices < color_cutoff:
            coloring_enabled = False
        coloring = color_graph(current) if coloring_enabled else None
        s, st = run_phase(current, theta_final, theta_color, max_iterations, coloring)
        rebuilt, ren = rebuild(current, s)
        phases.append(OPhase(s.assignment, ren, st["iterations"], st["total_moves"],
                             st["q_end"], st["theta"], st["colored"], st["hit_cap"],
                             st["q_trace"], st["moves_trace"],
                             coloring.num_colors if coloring is not None else 0))
        gain = _rel_gain(st["q_end"], q_prev_phase)
        if coloring_enabled and gain < theta_color:
            coloring_enabled = False
        q_prev_phase = st["q_end"]
        current = rebuilt
        if st["total_moves"] == 0 or gain < theta_final:
            break
    v = np.arange(g.num_vertices, dtype=np.int64)
    if vf is not None:
        v = vf.vertex_map[v]
    for p in phases:
        v = p.renumber[p.assignment[v]]
    return OHierarchy(phases, vf, v, phases[-1].q_end, current.num_vertices)
