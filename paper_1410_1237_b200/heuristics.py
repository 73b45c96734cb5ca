"""Vertex following and distance-1 colouring on device (mirror of PL/heuristics.py).

``vf_compact`` (PL/heuristics.py:46-89) emits the compacted records with
``plv_vf_records`` and builds the new CSR with ``plv_csr_build``.
``color_graph`` (PL/heuristics.py:92-118) runs the speculative colouring
rounds with ``plv_color``.  Results expose the reference's numpy attributes
lazily and keep device tensors for the engine.
"""

from __future__ import annotations

import numpy as np

from . import _lib
from .graph import Graph


class VfMapping:
    """Result of vertex-following compaction (PL/heuristics.py:19-24)."""

    def __init__(self, d_vertex_map, graph: Graph, merged_count: int):
        self.d_vertex_map = d_vertex_map
        self.graph = graph
        self.merged_count = int(merged_count)
        self._vm = None

    @property
    def vertex_map(self) -> np.ndarray:
        if self._vm is None:
            self._vm = self.d_vertex_map.cpu().numpy().astype(np.int64)
        return self._vm


class Coloring:
    """Valid distance-1 colouring (PL/heuristics.py:27-43)."""

    def __init__(self, d_colors, num_colors: int, rounds: int = 0):
        self.d_colors = d_colors
        self.num_colors = int(num_colors)
        self.rounds = int(rounds)
        self._colors = None
        self._sizes = None
        self._dev_classes = None

    @property
    def colors(self) -> np.ndarray:
        if self._colors is None:
            self._colors = self.d_colors.cpu().numpy().astype(np.int64)
        return self._colors

    @property
    def class_sizes(self) -> np.ndarray:
        if self._sizes is None:
            self._sizes = np.bincount(self.colors, minlength=self.num_colors)
        return self._sizes

    def device_classes(self):
        """(class offsets on host, class vertices on device): the colour
        classes in ascending colour, ascending vertex id within a class."""
        if self._dev_classes is None:
            import torch
            n = int(self.d_colors.numel())
            dev = self.d_colors.device
            off = torch.empty(self.num_colors + 1, dtype=torch.int64, device=dev)
            vtx = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
            _lib.check(_lib.lib().color_classes(_lib.ptr(self.d_colors), n, self.num_colors,
                                                _lib.ptr(off), _lib.ptr(vtx), _lib.stream()),
                       "color_classes")
            self._dev_classes = (off.cpu().numpy(), vtx[:n])
        return self._dev_classes

    def classes(self):
        """Vertex arrays per colour, ascending vertex id within each class."""
        off, vtx = self.device_classes()
        v = vtx.cpu().numpy().astype(np.int64)
        return [v[off[c]:off[c + 1]] for c in range(self.num_colors)]

    def size_rsd(self) -> float:
        sizes = self.class_sizes.astype(np.float64)
        return float(sizes.std() / sizes.mean())


def vf_compact(g: Graph) -> VfMapping:
    """Merge every single-degree vertex into its sole neighbour (one pass)."""
    import torch
    n = g.num_vertices
    dev = g.d_off.device
    cap = max(g.nnz + n, 1)
    vmap = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
    ru = torch.empty(cap, dtype=torch.int32, device=dev)
    rv = torch.empty(cap, dtype=torch.int32, device=dev)
    rw = torch.empty(cap, dtype=torch.float64, device=dev)
    info = _lib.i64_host(3)
    _lib.check(_lib.lib().vf_records(_lib.ptr(g.d_off), _lib.ptr(g.d_nbr), _lib.ptr(g.d_w),
                                     _lib.ptr(g.d_selfw), n, _lib.ptr(vmap), _lib.ptr(ru),
                                     _lib.ptr(rv), _lib.ptr(rw), _lib.hp(info), _lib.stream()),
               "vf_records")
    n_new, merged, R = int(info[0]), int(info[1]), int(info[2])
    cg = Graph.from_device_records(ru[:R], rv[:R], rw[:R], n_new, count_merges=False)
    return VfMapping(vmap[:n], cg, merged)


def color_graph(g: Graph, workers: int = 1) -> Coloring:
    """Speculative parallel greedy distance-1 colouring (deterministic)."""
    import torch
    n = g.num_vertices
    colors = torch.empty(max(n, 1), dtype=torch.int32, device=g.d_off.device)
    info = _lib.i64_host(2)
    _lib.check(_lib.lib().color(_lib.ptr(g.d_off), _lib.ptr(g.d_nbr), n, g.max_degree,
                                _lib.ptr(colors), _lib.hp(info), _lib.stream()), "color")
    return Coloring(colors[:n], int(info[0]), int(info[1]))


def check_coloring(g: Graph, coloring: Coloring) -> bool:
    """Full edge scan: no non-self edge may join two same-coloured vertices."""
    src = np.repeat(np.arange(g.num_vertices, dtype=np.int64), np.diff(g.adjacency_offsets))
    nonself = src != g.neighbors
    colors = coloring.colors
    if np.any(colors[src[nonself]] == colors[g.neighbors[nonself]]):
        raise AssertionError("adjacent vertices share a color")
    if len(colors) and (colors.min() < 0 or colors.max() >= coloring.num_colors):
        raise AssertionError("color ids out of range")
    if coloring.num_colors and np.any(coloring.class_sizes == 0):
        raise AssertionError("unused color id")
    return True
