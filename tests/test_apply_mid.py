"""GPU: the apply of small float-weighted graphs (at most 32,768 vertices):
the counting sort over the communities and the per-community ordered folds
(apply.cu, k_mid_*) against the oracle's sequential apply
(PL/_kernels.pyx:104-145) -- short segments (sorted in registers), segments
ranked by counting (17..128 events) and by the id bitmap (more), in
uncoloured (one stage, live rule) and coloured stages."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

pl = pytest.importorskip("paper_1410_1237_b200")


def _stars(nh, leaves_per_hub, extra, seed):
    """nh hubs with their own leaves (every leaf joins its hub's community in
    the first uncoloured iteration: one long event segment per hub), a ring of
    the hubs, and random leaf-leaf edges; float weights."""
    rng = np.random.default_rng(seed)
    n = nh + nh * leaves_per_hub
    u, v = [], []
    for h in range(nh):
        lv = nh + h * leaves_per_hub + np.arange(leaves_per_hub)
        u.append(np.full(leaves_per_hub, h))
        v.append(lv)
    u.append(np.arange(nh))
    v.append((np.arange(nh) + 1) % nh)
    a = rng.integers(nh, n, extra)
    b = rng.integers(nh, n, extra)
    keep = a != b
    u.append(a[keep])
    v.append(b[keep])
    u, v = np.concatenate(u), np.concatenate(v)
    w = rng.uniform(0.5, 2.0, len(u))
    return u, v, w, n


@pytest.mark.parametrize("nh,lph,extra,seed", [
    (3, 1500, 800, 1),     # three segments of ~1500 events: the bitmap ranking
    (40, 60, 500, 2),      # forty segments of ~60 events: ranking by counting
    (300, 6, 900, 3),      # short segments only
    (2, 9000, 100, 4),     # two very long segments (ordered block folds)
])
@pytest.mark.parametrize("coloring", [False, True])
def test_small_graph_apply(orc, nh, lph, extra, seed, coloring):
    u, v, w, n = _stars(nh, lph, extra, seed)
    assert n <= 32768
    g = pl.Graph.from_edges(u, v, w, num_vertices=n)
    og = orc.from_edges(u, v, w, num_vertices=n)
    cut = 0 if coloring else 10 ** 9
    # (no vertex following: it would fold the leaves into their hubs)
    oh = orc.run(og, color_cutoff=cut, max_iterations=40, use_vf=False)
    h = pl.run(g, pl.RunConfig(color_cutoff=cut, max_iterations_per_phase=40, use_vf=False))
    assert [p.stats.iterations for p in h.phases] == [p.iterations for p in oh.phases]
    assert np.array_equal(h.final_assignment, oh.final_assignment)
    assert h.final_modularity == oh.final_modularity
    # one uncoloured iteration's state, bit for bit
    s = pl.singleton_state(g)
    os_ = orc.singleton_state(og)
    sub = np.arange(n)
    s, mv = pl.run_iteration(g, s, sub)
    omv = orc.run_iteration(og, os_, sub)
    assert mv == omv
    assert np.array_equal(s.assignment, os_.assignment)
    assert np.array_equal(s.a_tot, os_.a_tot)
    assert np.array_equal(s.w_internal, os_.w_internal)
    assert np.array_equal(s.sizes, os_.sizes)
