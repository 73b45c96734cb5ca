"""GPU: the huge-row colouring path (rows above CPEND = 4096 entries keep a
committed-colour bitmap and per-chunk pending lists across rounds; color.cu)
against the oracle's colouring (PL/heuristics.py:92-118) on graphs whose hubs
are adjacent to each other, so they clash and stay active for many rounds
while their leaves commit around them."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

pl = pytest.importorskip("paper_1410_1237_b200")


def _hub_graph(nh, leaves, per_hub, seed, hub_ids="low"):
    rng = np.random.default_rng(seed)
    n = nh + leaves
    hubs = np.arange(nh) if hub_ids == "low" else np.arange(leaves, n)
    others = np.setdiff1d(np.arange(n), hubs)
    iu, ju = np.triu_indices(nh, 1)
    u = [hubs[iu]]
    v = [hubs[ju]]
    for h in hubs:  # each hub: a random set of leaves (rows well above 4096)
        t = rng.choice(others, size=per_hub, replace=False)
        u.append(np.full(per_hub, h))
        v.append(t)
    # sparse leaf-leaf edges so leaves clash among themselves too
    a = rng.choice(others, size=4 * leaves)
    b = rng.choice(others, size=4 * leaves)
    keep = a != b
    u.append(a[keep])
    v.append(b[keep])
    u = np.concatenate(u)
    v = np.concatenate(v)
    w = rng.uniform(1.0, 3.0, len(u))
    return u, v, w, n


@pytest.mark.parametrize("nh,leaves,per_hub,seed,ids", [
    (24, 20000, 9000, 1, "low"),
    (40, 30000, 5000, 2, "high"),
    (12, 12000, 11000, 3, "low"),
])
def test_huge_rows_coloring_matches_oracle(orc, nh, leaves, per_hub, seed, ids):
    u, v, w, n = _hub_graph(nh, leaves, per_hub, seed, ids)
    g = pl.Graph.from_edges(u, v, w, num_vertices=n)
    og = orc.from_edges(u, v, w, num_vertices=n)
    col = pl.color_graph(g)
    oc = orc.color_graph(og)
    assert int(np.diff(g.adjacency_offsets).max()) > 4096
    assert col.num_colors == oc.num_colors
    assert np.array_equal(col.colors, oc.colors)
    assert col.rounds == oc.rounds and col.rounds > 3
    pl.check_coloring(g, col)
