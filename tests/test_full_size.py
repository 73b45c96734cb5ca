"""GPU parity at BASELINE.json's full C2 size (R-MAT scale 20, 16.8 M records):
the device-generated graph, VF, the colouring and one coloured phase-1
local-move iteration, bit-for-bit against the pinned CPU oracle on the
numpy-generated graph (the two generators are the same counter-based RNG),
plus the properties that need no oracle (valid colouring, state aggregates
consistent with the assignment, Q recomputed from scratch)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

pl = pytest.importorskip("paper_1410_1237_b200")


@pytest.fixture(scope="module")
def c2(orc):
    from paper_1410_1237_b200 import synthetic as syn
    g = syn.config_graph("c2_rmat20")  # generated and built on device
    u, v, w = syn.rmat_records(20, 16, seed=0)
    og = orc.from_edges(u, v, w, num_vertices=1 << 20)
    return g, og


def test_c2_csr_vf_coloring(orc, c2):
    g, og = c2
    assert np.array_equal(g.adjacency_offsets, og.adjacency_offsets)
    assert np.array_equal(g.neighbors, og.neighbors)
    assert np.array_equal(g.weights, og.weights)
    assert g.total_weight == og.total_weight
    vf, ovf = pl.vf_compact(g), orc.vf_compact(og)
    assert np.array_equal(vf.vertex_map, ovf.vertex_map)
    gv, ogv = vf.graph, ovf.graph
    assert np.array_equal(gv.neighbors, ogv.neighbors) and np.array_equal(gv.weights, ogv.weights)
    col, ocol = pl.color_graph(gv), orc.color_graph(ogv)
    assert np.array_equal(col.colors, ocol.colors)
    # a valid distance-1 colouring, checked without the oracle
    off, nbr = gv.adjacency_offsets, gv.neighbors
    src = np.repeat(np.arange(gv.num_vertices), np.diff(off))
    other = nbr != src
    assert not np.any(col.colors[src[other]] == col.colors[nbr[other]])


def test_c2_colored_iteration(orc, c2):
    g, og = c2
    vf, ovf = pl.vf_compact(g), orc.vf_compact(og)
    gv, ogv = vf.graph, ovf.graph
    col = pl.color_graph(gv)
    s = pl.singleton_state(gv)
    os_ = orc.singleton_state(ogv)
    moves = 0
    for stage in col.classes():
        s, mv = pl.run_iteration(gv, s, stage)
        moves += orc.run_iteration(ogv, os_, stage)
    assert np.array_equal(s.assignment, os_.assignment)
    assert np.array_equal(s.a_tot, os_.a_tot)
    assert np.array_equal(s.w_internal, os_.w_internal)
    assert np.array_equal(s.sizes, os_.sizes)
    assert pl.modularity(gv, s) == orc.modularity(ogv, os_)
    # aggregates consistent with the assignment (independent of the oracle)
    a = s.assignment
    assert np.array_equal(np.bincount(a, minlength=gv.num_vertices), s.sizes)
    kv = gv.weighted_degrees
    assert np.allclose(np.bincount(a, weights=kv, minlength=gv.num_vertices), s.a_tot,
                       rtol=1e-12, atol=1e-9)


def test_c2_full_run(orc, c2):
    """The whole multi-phase run() on C2 (VF, coloured phase 1, rebuilds),
    final assignment and Q bit-identical to the oracle's."""
    g, og = c2
    oh = orc.run(og, max_iterations=100)
    h = pl.run(g, pl.RunConfig(max_iterations_per_phase=100))
    assert [p.stats.iterations for p in h.phases] == [p.iterations for p in oh.phases]
    assert np.array_equal(h.final_assignment, oh.final_assignment)
    assert h.final_modularity == oh.final_modularity
