"""GPU: the device-side phase loop (plv_phase_run: the iteration inside a CUDA
graph WHILE node, the stopping rule of PL/engine.py:203-212 in a control
kernel) against the host-driven loop of single iterations -- same trace
(Q bits, moves), same stop reason, same final state -- and against the
oracle through run() on graphs whose phases hit the iteration cap."""

import os
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

pl = pytest.importorskip("paper_1410_1237_b200")

from paper_1410_1237_b200 import synthetic as syn  # noqa: E402
from paper_1410_1237_b200.engine import PhaseEngine, _iteration_converged  # noqa: E402

KEYS = ("assignment", "a_tot", "w_internal", "sizes")


def _host_loop(eng, theta, cap):
    qs, mvs = [], []
    q_prev = None
    hit = False
    while True:
        q, m, _ = eng.iterate()
        qs.append(q)
        mvs.append(m)
        if m == 0:
            break
        if q_prev is not None and _iteration_converged(q, q_prev, theta):
            break
        if len(qs) >= cap:
            hit = True
            break
        q_prev = q
    return qs, mvs, hit


def _state(g):
    d = pl.singleton_state(g).device()
    st = {k: d[k].clone() for k in KEYS}
    return pl.CommunityState.from_device(st["assignment"], st["a_tot"], st["w_internal"],
                                         st["sizes"]), st


@pytest.mark.parametrize("colored", [True, False])
@pytest.mark.parametrize("theta,cap", [(1e-6, 10_000), (1e-6, 1), (1e-6, 4), (0.0, 25)])
def test_device_loop_equals_host_loop(colored, theta, cap):
    u, v, w = syn.grid_records(side=40, keep=0.9, pendants=300, seed=3)
    g = pl.vf_compact(pl.Graph.from_edges(u, v, w, num_vertices=40 * 40 + 300)).graph
    col = pl.color_graph(g) if colored else None
    s1, st1 = _state(g)
    s2, st2 = _state(g)
    e1 = PhaseEngine(g, s1, col)
    e2 = PhaseEngine(g, s2, col)
    qs, mvs, hit = _host_loop(e1, theta, cap)
    q2, m2, ms2, it, total, hit2 = e2.run(theta, cap)
    assert e2.device_loop
    assert it == len(qs) and hit2 == hit and total == sum(mvs)
    assert [float(x) for x in q2] == qs and [int(x) for x in m2] == mvs
    assert (np.asarray(ms2) >= 0).all()
    for k in KEYS:
        assert bool((st1[k] == st2[k]).all()), k
    e1.close()
    e2.close()


@pytest.fixture(scope="module")
def orc():
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, os.path.join(root, "oracle"))
    import oracle
    return oracle


@pytest.mark.parametrize("seed", [0, 1])
def test_capped_phases_match_oracle(orc, seed):
    """Small fp-weighted grids oscillate: uncoloured phases run to the cap."""
    u, v, w = syn.grid_records(side=48, keep=0.9, pendants=200, seed=seed)
    n = 48 * 48 + 200
    g = pl.Graph.from_edges(u, v, w, num_vertices=n)
    og = orc.from_edges(u, v, w, num_vertices=n)
    h = pl.run(g, pl.RunConfig(max_iterations_per_phase=300))
    oh = orc.run(og, max_iterations=300)
    assert [p.stats.iterations for p in h.phases] == [p.iterations for p in oh.phases]
    assert np.array_equal(h.final_assignment, oh.final_assignment)
    assert h.final_modularity == oh.final_modularity


def _sbm_integral(n=1200, blocks=12, seed=7):
    rng = np.random.default_rng(seed)
    b = np.arange(n) // (n // blocks)
    iu, ju = np.triu_indices(n, 1)
    p = np.where(b[iu] == b[ju], 0.08, 0.004)
    keep = rng.random(len(iu)) < p
    return iu[keep], ju[keep]


@pytest.mark.parametrize("cap", [10_000, 777])
def test_cycle_skipping_is_exact(cap):
    """Integral weights, one uncoloured stage: the device loop detects the
    oscillation, verifies it bit for bit, skips to the cap -- same trace and
    same final state as iterating every time."""
    u, v = _sbm_integral()
    g = pl.Graph.from_edges(u, v, num_vertices=1200)
    assert g.integral
    s1, st1 = _state(g)
    s2, st2 = _state(g)
    e1 = PhaseEngine(g, s1, None)
    e2 = PhaseEngine(g, s2, None)
    qs, mvs, hit = _host_loop(e1, 1e-6, cap)
    q2, m2, ms2, it, total, hit2 = e2.run(1e-6, cap)
    assert it == len(qs) and hit2 == hit and total == sum(mvs)
    assert [float(x) for x in q2] == qs and [int(x) for x in m2] == mvs
    for k in KEYS:
        assert bool((st1[k] == st2[k]).all()), k
    if hit:
        assert e2.cycle is not None and e2.cycle[1] < cap  # the tail was skipped
    e1.close()
    e2.close()


def test_cycle_skipping_run_matches_oracle(orc):
    u, v = _sbm_integral(seed=11)
    n = 1200
    w = np.ones(len(u))
    g = pl.Graph.from_edges(u, v, w, num_vertices=n)
    og = orc.from_edges(u, v, w, num_vertices=n)
    h = pl.run(g, pl.RunConfig(max_iterations_per_phase=3000))
    oh = orc.run(og, max_iterations=3000)
    assert [p.stats.iterations for p in h.phases] == [p.iterations for p in oh.phases]
    assert np.array_equal(h.final_assignment, oh.final_assignment)
    assert h.final_modularity == oh.final_modularity


def test_iteration_graph_kernel_count():
    """The single-iteration graph is captured on demand and reports its kernel
    nodes (bench.py's gpu_launches)."""
    u, v, w = syn.rmat_records(11, 8, seed=5)
    g = pl.Graph.from_edges(u, v, w, num_vertices=1 << 11)
    s, _ = _state(g)
    col = pl.color_graph(g)
    e = PhaseEngine(g, s, col)
    k = e.graph_kernels()
    assert k >= col.num_colors  # at least one decide kernel per colour stage
    q1 = e.iterate()
    assert e.graph_kernels() == k
    assert q1[1] >= 0
    e.close()
