"""GPU: the partitioned (multi-GPU) phase engine, plv_phase_create_part.

Only one GPU is available to these tests, so the W-rank exchange is checked
two ways: (1) W host-stepped engines on the same device ("virtual ranks"),
each deciding only its slice of every stage, the slices copied between
their decide outputs as the NCCL broadcasts would, every rank applying whole
stages -- state bit-identical on every rank and to the single-GPU engine;
(2) the captured NCCL path with a 1-rank communicator (broadcasts inside the
iteration's CUDA graph) bit-identical to the single-GPU engine.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

pl = pytest.importorskip("paper_1410_1237_b200")

from paper_1410_1237_b200 import dist as pdist  # noqa: E402
from paper_1410_1237_b200 import synthetic as syn  # noqa: E402
from paper_1410_1237_b200.engine import PhaseEngine  # noqa: E402

KEYS = ("assignment", "a_tot", "w_internal", "sizes")


def _graph(kind):
    if kind == "rmat":
        u, v, w = syn.rmat_records(13, 16, seed=4)
        return pl.Graph.from_edges(u, v, w, num_vertices=1 << 13)
    # hubs (tier 4) plus a sparse background
    rng = np.random.default_rng(5)
    n = 6000
    u = rng.integers(0, n, 30000)
    v = rng.integers(0, n, 30000)
    hu = np.repeat(np.arange(6), 2500)
    hv = rng.integers(10, n, len(hu))
    u, v = np.concatenate([u, hu]), np.concatenate([v, hv])
    keep = u != v
    u, v = u[keep], v[keep]
    return pl.Graph.from_edges(u, v, rng.uniform(1.0, 10.0, len(u)), num_vertices=n)


def _state(g):
    s0 = pl.singleton_state(g)
    d = s0.device()
    st = {k: d[k].clone() for k in KEYS}
    return pl.CommunityState.from_device(st["assignment"], st["a_tot"], st["w_internal"],
                                         st["sizes"]), st


@pytest.mark.parametrize("kind", ["rmat", "hubs"])
@pytest.mark.parametrize("colored", [True, False])
@pytest.mark.parametrize("world", [2, 3])
def test_virtual_ranks_match_single_gpu(kind, colored, world):
    g = _graph(kind)
    col = pl.color_graph(g) if colored else None
    s1, st1 = _state(g)
    ref = PhaseEngine(g, s1, col)
    engines, states = [], []
    for r in range(world):
        s, st = _state(g)
        engines.append(pdist.PartitionedPhaseEngine(g, s, col, r, world))
        states.append(st)
    sl = engines[0].slices()
    assert (sl[:, 0] == 0).all() and (sl[:, -1] == np.diff(engines[0].engine_stage_off())).all()
    for _ in range(3):
        q1, m1, _ = ref.iterate()
        outs = pdist.stepped_iteration(engines)
        for q, m in outs:
            assert m == m1 and q == q1
        for st in states:
            for k in KEYS:
                assert bool((st[k] == st1[k]).all()), k
    ref.close()
    for e in engines:
        e.close()


def test_virtual_ranks_with_an_empty_rank():
    g = _graph("rmat")
    col = pl.color_graph(g)
    n = g.num_vertices
    bounds = np.array([0, 0, n // 3, n], np.int64)  # rank 0 owns nothing
    s1, st1 = _state(g)
    ref = PhaseEngine(g, s1, col)
    engines, states = [], []
    for r in range(3):
        s, st = _state(g)
        engines.append(pdist.PartitionedPhaseEngine(g, s, col, r, 3, bounds=bounds))
        states.append(st)
    for _ in range(2):
        q1, m1, _ = ref.iterate()
        for q, m in pdist.stepped_iteration(engines):
            assert (q, m) == (q1, m1)
    for st in states:
        for k in KEYS:
            assert bool((st[k] == st1[k]).all()), k


@pytest.mark.parametrize("colored", [True, False])
def test_nccl_one_rank_captured_exchange(colored):
    g = _graph("hubs")
    col = pl.color_graph(g) if colored else None
    s1, st1 = _state(g)
    ref = PhaseEngine(g, s1, col)
    s2, st2 = _state(g)
    comm = pdist.nccl_communicator(0, 1)
    try:
        eng = pdist.PartitionedPhaseEngine(g, s2, col, 0, 1, comm=comm)
        for _ in range(3):
            assert eng.iterate()[:2] == ref.iterate()[:2]
        for k in KEYS:
            assert bool((st2[k] == st1[k]).all()), k
        eng.close()
    finally:
        pdist.destroy_communicator(comm)
