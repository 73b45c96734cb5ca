"""Seeded graph generators.

Two families:

* The reference's small test generators (PL/synthetic.py:10-68):
  ``gnm_random_graph``, ``random_geometric_graph``,
  ``random_weighted_multigraph_records`` -- same numpy RNG call sequence, so a
  seed gives the same graph as the reference.
* Counter-based generators for the five BASELINE.json configs (the reference
  ships none).  Every draw is ``rnd01(stream_key(seed, stream), counter)``
  (SplitMix64), so the numpy version here and the CUDA version in
  csrc/gen.cu produce bit-identical record arrays, order included (the
  duplicate-merge order of Graph.from_edges depends on record order).  The
  ``*_records`` functions are the numpy specification (used for CPU oracles
  and to prove device == host), the ``*_device`` functions generate in HBM.
"""

from __future__ import annotations

import functools

import numpy as np

from . import _lib
from .graph import Graph

# ------------------------------------------------------------ SplitMix64

_M64 = (1 << 64) - 1
GAMMA = 0x9E3779B97F4A7C15
_U = np.uint64


def _mix64_int(z: int) -> int:
    z &= _M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
    return z ^ (z >> 31)


def stream_key(seed: int, stream: int) -> int:
    return _mix64_int(seed * 0xD1B54A32D192ED03 + stream * GAMMA + 1)


def _mix64(z: np.ndarray) -> np.ndarray:
    z = (z ^ (z >> _U(30))) * _U(0xBF58476D1CE4E5B9)
    z = (z ^ (z >> _U(27))) * _U(0x94D049BB133111EB)
    return z ^ (z >> _U(31))


def rnd01(key: int, idx) -> np.ndarray:
    """u in [0, 1): 53 high bits of the idx-th SplitMix64 output of `key`."""
    i = np.asarray(idx, dtype=np.uint64)
    x = _mix64(_U(key) + (i + _U(1)) * _U(GAMMA))
    return (x >> _U(11)).astype(np.float64) * (1.0 / 9007199254740992.0)


# ------------------------------------------------------- BASELINE configs

RMAT_ABC = (0.57, 0.19, 0.19)


def rmat_records(scale: int, edge_factor: int = 16, abc=RMAT_ABC, w_lo: float = 1.0,
                 w_hi: float = 10.0, seed: int = 0, chunk: int = 1 << 20, r_begin: int = 0,
                 r_end: int | None = None):
    """R-MAT records (self loops dropped, duplicates kept for from_edges).
    [r_begin, r_end) selects a range of record draws; ranges concatenate."""
    a, b, c = abc
    ab = a + b
    abc_ = ab + c
    R = edge_factor << scale if r_end is None else min(r_end, edge_factor << scale)
    klvl, kw = stream_key(seed, 1), stream_key(seed, 2)
    us, vs, ws = [np.empty(0, np.int64)], [np.empty(0, np.int64)], [np.empty(0)]
    for r0 in range(r_begin, R, chunk):
        r = np.arange(r0, min(R, r0 + chunk), dtype=np.uint64)
        s = np.zeros(len(r), dtype=np.int64)
        d = np.zeros(len(r), dtype=np.int64)
        base = r * _U(scale)
        for lvl in range(scale):
            x = rnd01(klvl, base + _U(lvl))
            ub = x >= ab
            vb = ((x >= a) & (x < ab)) | (x >= abc_)
            s = (s << 1) | ub
            d = (d << 1) | vb
        keep = s != d
        us.append(s[keep])
        vs.append(d[keep])
        ws.append(w_lo + (w_hi - w_lo) * rnd01(kw, r[keep]))
    return np.concatenate(us), np.concatenate(vs), np.concatenate(ws)


def sbm_records(n: int = 10_000, block: int = 100, p_in: float = 0.05, p_out: float = 0.0005,
                seed: int = 0, rows_per_chunk: int = 256):
    """Planted partition: every pair i < j is an edge with prob. p_in / p_out."""
    key = stream_key(seed, 3)
    us, vs = [], []
    for i0 in range(0, n, rows_per_chunk):
        i = np.arange(i0, min(n, i0 + rows_per_chunk), dtype=np.int64)[:, None]
        j = np.arange(n, dtype=np.int64)[None, :]
        p = (i * n + j).astype(np.uint64)
        u = rnd01(key, p)
        pr = np.where(i // block == j // block, p_in, p_out)
        keep = (j > i) & (u < pr)
        ii, jj = np.nonzero(keep)
        us.append(i[ii, 0])
        vs.append(jj.astype(np.int64))
    u = np.concatenate(us)
    return u, np.concatenate(vs), np.ones(len(u), dtype=np.float64)


def grid_records(side: int = 2048, keep: float = 0.9, pendants: int = 1_000_000,
                 w_lo: float = 0.5, seed: int = 0):
    """4-neighbour grid (row-major ids; horizontal then vertical edges, each
    kept with prob. `keep`) plus degree-1 pendants on uniform grid vertices."""
    N = side * side
    H = side * (side - 1)
    E = 2 * H
    e = np.arange(E, dtype=np.int64)
    kept = e[rnd01(stream_key(seed, 4), e.astype(np.uint64)) < keep]
    hor = kept < H
    r = np.where(hor, kept // (side - 1), (kept - H) // side)
    c = np.where(hor, kept % (side - 1), (kept - H) % side)
    a = r * side + c
    b = np.where(hor, a + 1, a + side)
    w = w_lo + rnd01(stream_key(seed, 5), kept.astype(np.uint64))
    p = np.arange(pendants, dtype=np.uint64)
    pu = N + p.astype(np.int64)
    pv = (rnd01(stream_key(seed, 6), p) * float(N)).astype(np.int64)
    pw = w_lo + rnd01(stream_key(seed, 7), p)
    return np.concatenate([a, pu]), np.concatenate([b, pv]), np.concatenate([w, pw])


@functools.lru_cache(maxsize=4)
def chung_lu_cdf(n: int = 1 << 24, gamma: float = 2.1, mean_degree: float = 12.0,
                 max_degree: float = 1e5):
    """Expected-degree sequence w_i ~ i^(-1/(gamma-1)), scaled to the mean and
    capped; returns its cumulative sum (shared by host and device sampling)."""
    i = np.arange(1, n + 1, dtype=np.float64)
    w = i ** (-1.0 / (gamma - 1.0))
    w *= mean_degree / w.mean()
    np.minimum(w, max_degree, out=w)
    c = np.cumsum(w)
    c.setflags(write=False)  # cached: shared by every caller
    return c


def chung_lu_records(n: int = 1 << 24, gamma: float = 2.1, mean_degree: float = 12.0,
                     max_degree: float = 1e5, seed: int = 0, chunk: int = 1 << 22,
                     r_begin: int = 0, r_end: int | None = None):
    """Chung-Lu records; [r_begin, r_end) selects a range of record draws."""
    cdf = chung_lu_cdf(n, gamma, mean_degree, max_degree)
    total = cdf[-1]
    R = int(round(total / 2.0))
    if r_end is not None:
        R = min(R, r_end)
    key = stream_key(seed, 8)
    us, vs = [np.empty(0, np.int64)], [np.empty(0, np.int64)]
    for r0 in range(r_begin, R, chunk):
        r = np.arange(r0, min(R, r0 + chunk), dtype=np.uint64)
        u = np.minimum(np.searchsorted(cdf, rnd01(key, r * _U(2)) * total, side="right"), n - 1)
        v = np.minimum(np.searchsorted(cdf, rnd01(key, r * _U(2) + _U(1)) * total,
                                       side="right"), n - 1)
        keep = u != v
        us.append(u[keep].astype(np.int64))
        vs.append(v[keep].astype(np.int64))
    u = np.concatenate(us)
    return u, np.concatenate(vs), np.ones(len(u), dtype=np.float64)


# ------------------------------------------------------- device versions

def _records_out(cap: int):
    import torch
    dev = _lib.device()
    return (torch.empty(max(cap, 1), dtype=torch.int32, device=dev),
            torch.empty(max(cap, 1), dtype=torch.int32, device=dev),
            torch.empty(max(cap, 1), dtype=torch.float64, device=dev))


def rmat_device(scale: int, edge_factor: int = 16, abc=RMAT_ABC, w_lo: float = 1.0,
                w_hi: float = 10.0, seed: int = 0):
    cap = edge_factor << scale
    u, v, w = _records_out(cap)
    cnt = _lib.i64_host(1)
    _lib.check(_lib.lib().gen_rmat(seed, scale, edge_factor, abc[0], abc[1], abc[2], w_lo, w_hi,
                                   _lib.ptr(u), _lib.ptr(v), _lib.ptr(w), cap, _lib.hp(cnt),
                                   _lib.stream()), "gen_rmat")
    c = int(cnt[0])
    return u[:c], v[:c], w[:c], 1 << scale


def sbm_device(n: int = 10_000, block: int = 100, p_in: float = 0.05, p_out: float = 0.0005,
               seed: int = 0):
    expect = n * (n - 1) / 2 * max(p_in, p_out)
    cap = int(expect * 1.5) + 4096
    u, v, w = _records_out(cap)
    cnt = _lib.i64_host(1)
    _lib.check(_lib.lib().gen_sbm(seed, n, block, p_in, p_out, _lib.ptr(u), _lib.ptr(v),
                                  _lib.ptr(w), cap, _lib.hp(cnt), _lib.stream()), "gen_sbm")
    c = int(cnt[0])
    return u[:c], v[:c], w[:c], n


def grid_device(side: int = 2048, keep: float = 0.9, pendants: int = 1_000_000,
                w_lo: float = 0.5, seed: int = 0):
    cap = 2 * side * (side - 1) + pendants
    u, v, w = _records_out(cap)
    cnt = _lib.i64_host(1)
    _lib.check(_lib.lib().gen_grid(seed, side, keep, pendants, w_lo, _lib.ptr(u), _lib.ptr(v),
                                   _lib.ptr(w), cap, _lib.hp(cnt), _lib.stream()), "gen_grid")
    c = int(cnt[0])
    return u[:c], v[:c], w[:c], side * side + pendants


def chung_lu_device(n: int = 1 << 24, gamma: float = 2.1, mean_degree: float = 12.0,
                    max_degree: float = 1e5, seed: int = 0):
    import torch
    cdf = chung_lu_cdf(n, gamma, mean_degree, max_degree)
    R = int(round(cdf[-1] / 2.0))
    d_cdf = torch.from_numpy(np.array(cdf)).to(_lib.device())  # (the cached cdf is read-only)
    u, v, w = _records_out(R)
    cnt = _lib.i64_host(1)
    _lib.check(_lib.lib().gen_chung_lu(seed, _lib.ptr(d_cdf), n, R, _lib.ptr(u), _lib.ptr(v),
                                       _lib.ptr(w), R, _lib.hp(cnt), _lib.stream()),
               "gen_chung_lu")
    c = int(cnt[0])
    return u[:c], v[:c], w[:c], n


# name -> (host generator, device generator, kwargs): BASELINE.json configs 1-5
CONFIGS = {
    "c1_sbm": (sbm_records, sbm_device, dict(n=10_000, block=100, p_in=0.05, p_out=0.0005)),
    "c2_rmat20": (rmat_records, rmat_device, dict(scale=20, edge_factor=16)),
    "c3_grid": (grid_records, grid_device, dict(side=2048, keep=0.9, pendants=1_000_000)),
    "c4_chung_lu": (chung_lu_records, chung_lu_device,
                    dict(n=1 << 24, gamma=2.1, mean_degree=12.0, max_degree=1e5)),
    "c5_rmat28": (rmat_records, rmat_device, dict(scale=28, edge_factor=16)),
}


def config_num_vertices(name: str, **kw) -> int:
    params = {**CONFIGS[name][2], **kw}
    if "scale" in params:
        return 1 << params["scale"]
    if "side" in params:
        return params["side"] ** 2 + params["pendants"]
    return params["n"]


def config_graph(name: str, seed: int = 0, **kw) -> Graph:
    """Build a BASELINE config graph entirely on device."""
    host, dev, params = CONFIGS[name]
    u, v, w, n = dev(seed=seed, **{**params, **kw})
    return Graph.from_device_records(u, v, w, n)


# ------------------------------------------------- reference test generators

def gnm_random_graph(n: int, num_edges: int, seed: int = 0, weight_range=None) -> Graph:
    """Uniform random simple graph with exactly ``num_edges`` edges
    (same RNG call sequence as PL/synthetic.py:10-41)."""
    u, v, w = gnm_records(n, num_edges, seed, weight_range)
    return Graph.from_edges(u, v, w, num_vertices=n)


def gnm_records(n: int, num_edges: int, seed: int = 0, weight_range=None):
    if num_edges > n * (n - 1) // 2:
        raise ValueError(f"cannot place {num_edges} edges on {n} vertices")
    rng = np.random.default_rng(seed)
    chosen = np.empty(0, dtype=np.int64)
    while len(chosen) < num_edges:
        need = num_edges - len(chosen)
        a = rng.integers(0, n, size=2 * need + 16, dtype=np.int64)
        b = rng.integers(0, n, size=2 * need + 16, dtype=np.int64)
        ok = a != b
        lo, hi = np.minimum(a[ok], b[ok]), np.maximum(a[ok], b[ok])
        chosen = np.unique(np.concatenate([chosen, lo * n + hi]))
    rng.shuffle(chosen)
    chosen = chosen[:num_edges]
    w = None
    if weight_range is not None:
        lo, hi = weight_range
        w = lo + (hi - lo) * (1.0 - rng.random(num_edges))   # uniform on (lo, hi]
    return chosen // n, chosen % n, w


def random_geometric_graph(n: int, radius: float, seed: int = 0) -> Graph:
    """Unit-square geometric graph (PL/synthetic.py:44-53)."""
    from scipy.spatial import cKDTree
    rng = np.random.default_rng(seed)
    pts = rng.random((n, 2))
    pairs = cKDTree(pts).query_pairs(radius, output_type="ndarray")
    pairs = pairs[np.lexsort((pairs[:, 1], pairs[:, 0]))]
    return Graph.from_edges(pairs[:, 0], pairs[:, 1], num_vertices=n)


def random_weighted_multigraph_records(n: int, max_records: int, seed: int,
                                       max_weight: int = 10, allow_self_loops: bool = True):
    """Raw integer-weighted records with duplicates (PL/synthetic.py:56-68)."""
    rng = np.random.default_rng(seed)
    k = rng.integers(1, max_records + 1)
    u = rng.integers(0, n, size=k, dtype=np.int64)
    v = rng.integers(0, n, size=k, dtype=np.int64)
    if not allow_self_loops:
        ok = u != v
        u, v = u[ok], v[ok]
    w = rng.integers(1, max_weight + 1, size=len(u)).astype(np.float64)
    return u, v, w
