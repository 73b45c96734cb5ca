"""GPU parity: the CUDA path (through libplv's C ABI) against the golden
fixtures of the unmodified reference and against the pinned CPU oracle.

Bit-exact for every integer and float64 array the reference produces (CSR,
degrees, m, VF, colours, decide targets, state after apply, phase state,
rebuild), final assignments identical, final modularity bit-equal.
"""

import numpy as np
import pytest

from conftest import GOLDEN_CASES, load_golden

pytestmark = pytest.mark.gpu

pl = pytest.importorskip("paper_1410_1237_b200")


def _same_graph(g, z, prefix=""):
    assert np.array_equal(g.adjacency_offsets, z[prefix + "off"])
    assert np.array_equal(g.neighbors, z[prefix + "nbr"])
    assert np.array_equal(g.weights, z[prefix + "wts"])
    assert np.array_equal(g.self_loop_weights, z[prefix + "selfw"])


@pytest.mark.parametrize("case", GOLDEN_CASES)
def test_from_edges_golden(case):
    z = load_golden(case)
    g = pl.Graph.from_edges(z["u"], z["v"], z["w"], num_vertices=int(z["n"]))
    _same_graph(g, z)
    assert np.array_equal(g.weighted_degrees, z["k"])
    assert g.total_weight == float(z["m"])
    assert g.num_edges == int(z["num_edges"])
    assert g.max_degree == int(z["max_degree"])
    assert g.merged_duplicates == int(z["merged"])


@pytest.mark.parametrize("case", GOLDEN_CASES)
def test_vf_and_coloring_golden(case):
    z = load_golden(case)
    g = pl.Graph.from_edges(z["u"], z["v"], z["w"], num_vertices=int(z["n"]))
    vf = pl.vf_compact(g)
    assert np.array_equal(vf.vertex_map, z["vf_map"])
    assert vf.merged_count == int(z["vf_merged"])
    _same_graph(vf.graph, z, "vf_")
    assert np.array_equal(vf.graph.weighted_degrees, z["vf_k"])
    assert vf.graph.total_weight == float(z["vf_m"])
    col = pl.color_graph(g)
    assert np.array_equal(col.colors, z["colors"])
    pl.check_coloring(g, col)


@pytest.mark.parametrize("case", GOLDEN_CASES)
def test_iteration_golden(case):
    z = load_golden(case)
    n = int(z["n"])
    g = pl.Graph.from_edges(z["u"], z["v"], z["w"], num_vertices=n)
    kern = pl.backend.active()
    s = pl.singleton_state(g)
    tg = np.empty(n, np.int64)
    mv = np.empty(n, np.uint8)
    kern.decide_moves(g.adjacency_offsets, g.neighbors, g.weights, g.weighted_degrees,
                      s.labels, np.arange(n), s.assignment, s.a_tot, s.sizes,
                      g.total_weight, g.max_degree, 1, tg, mv)
    assert np.array_equal(tg, z["it1_targets"])
    assert np.array_equal(mv, z["it1_moved"])
    s = pl.singleton_state(g)
    s, moves = pl.run_iteration(g, s, np.arange(n))
    assert moves == int(z["it1_moves"])
    assert np.array_equal(s.assignment, z["it1_assign"])
    assert np.array_equal(s.a_tot, z["it1_atot"])
    assert np.array_equal(s.w_internal, z["it1_wint"])
    assert np.array_equal(s.sizes, z["it1_sizes"])
    assert pl.modularity(g, s) == float(z["it1_q"])


@pytest.mark.parametrize("case", GOLDEN_CASES)
def test_colored_phase_and_rebuild_golden(case):
    z = load_golden(case)
    g = pl.Graph.from_edges(z["u"], z["v"], z["w"], num_vertices=int(z["n"]))
    col = pl.color_graph(g)
    cfg = pl.RunConfig(use_vf=False, use_coloring=True, color_cutoff=0,
                       max_iterations_per_phase=200)
    s, st = pl.run_phase(g, cfg, col)
    assert np.array_equal(s.assignment, z["ph_assign"])
    assert np.array_equal(s.a_tot, z["ph_atot"])
    assert np.array_equal(s.w_internal, z["ph_wint"])
    assert st.q_end == float(z["ph_q"]) and st.iterations == int(z["ph_iters"])
    rb, ren = pl.rebuild(g, s)
    _same_graph(rb, z, "rb_")
    assert rb.total_weight == float(z["rb_m"])
    assert np.array_equal(ren, z["rb_ren"])


@pytest.mark.parametrize("case", GOLDEN_CASES)
@pytest.mark.parametrize("tag,cutoff", [("run", 100_000), ("runc", 0)])
def test_run_golden(case, tag, cutoff):
    z = load_golden(case)
    g = pl.Graph.from_edges(z["u"], z["v"], z["w"], num_vertices=int(z["n"]))
    trace = []
    h = pl.run(g, pl.RunConfig(color_cutoff=cutoff, max_iterations_per_phase=300), trace)
    assert np.array_equal(h.final_assignment, z[tag + "_assign"])
    assert h.final_modularity == float(z[tag + "_q"])
    assert h.num_communities == int(z[tag + "_ncomm"])
    stages = {"vf": 0, "coloring": 1, "clustering": 2, "rebuild": 3}
    ti = np.array([[r.phase, r.iteration, stages[r.stage], r.moves] for r in trace])
    assert np.array_equal(ti, z[tag + "_trace_i"])
    assert np.array_equal(np.array([r.modularity for r in trace]), z[tag + "_trace_q"])
    assert np.array_equal(np.array([r.theta for r in trace]), z[tag + "_trace_theta"])


@pytest.mark.parametrize("n", [0, 1, 7, 8, 128, 129, 257, 1000, 8193, 100_000, 1_000_003,
                               5_000_000])
def test_device_sum_is_numpy_sum(n):
    import torch
    from paper_1410_1237_b200 import _lib
    rng = np.random.default_rng(n)
    a = rng.random(n) * 10.0 ** rng.uniform(-6, 6, n)
    d = torch.from_numpy(a).cuda()
    out = torch.empty(1, dtype=torch.float64, device="cuda")
    _lib.check(_lib.lib().sum(_lib.ptr(d), n, _lib.ptr(out), _lib.stream()))
    assert float(out.item()) == a.sum()


@pytest.mark.parametrize("name,kw", [
    ("c1_sbm", dict(n=1500, block=100)),
    ("c2_rmat20", dict(scale=12)),
    ("c3_grid", dict(side=64, pendants=500)),
    ("c4_chung_lu", dict(n=1 << 14, max_degree=1000.0)),
])
def test_device_generators_match_numpy(name, kw):
    from paper_1410_1237_b200 import synthetic as syn
    host, dev, params = syn.CONFIGS[name]
    p = {**params, **kw}
    u, v, w = host(seed=7, **p)
    du, dv, dw, n = dev(seed=7, **p)
    assert np.array_equal(du.cpu().numpy(), u)
    assert np.array_equal(dv.cpu().numpy(), v)
    assert np.array_equal(dw.cpu().numpy(), w)


@pytest.mark.parametrize("name,kw,cutoff", [
    ("c1_sbm", dict(), 0),                                  # BASELINE config 1, full size
    ("c2_rmat20", dict(scale=14), 0),
    ("c3_grid", dict(side=128, pendants=4000), 0),
    ("c4_chung_lu", dict(n=1 << 16, max_degree=2000.0), 0),
])
def test_run_matches_oracle(orc, name, kw, cutoff):
    from paper_1410_1237_b200 import synthetic as syn
    host, dev, params = syn.CONFIGS[name]
    p = {**params, **kw}
    u, v, w = host(seed=1, **p)
    n = syn.config_num_vertices(name, **kw)
    og = orc.from_edges(u, v, w, num_vertices=n)
    g = pl.Graph.from_edges(u, v, w, num_vertices=n)
    assert np.array_equal(g.neighbors, og.neighbors) and np.array_equal(g.weights, og.weights)
    assert g.total_weight == og.total_weight
    oh = orc.run(og, color_cutoff=cutoff, max_iterations=200)
    h = pl.run(g, pl.RunConfig(color_cutoff=cutoff, max_iterations_per_phase=200))
    assert np.array_equal(h.final_assignment, oh.final_assignment)
    assert h.final_modularity == oh.final_modularity
    assert [p_.stats.iterations for p_ in h.phases] == [p_.iterations for p_ in oh.phases]


def test_kernel_seam_apply_general_subset(orc):
    """apply_moves with an arbitrary-order subset (live rule through the
    position map) equals the sequential reference order."""
    from paper_1410_1237_b200 import synthetic as syn
    u, v, w = syn.gnm_records(300, 1500, seed=4, weight_range=(0.0, 2.0))
    g = pl.Graph.from_edges(u, v, w, num_vertices=300)
    og = orc.from_edges(u, v, w, num_vertices=300)
    rng = np.random.default_rng(0)
    sub = rng.permutation(300)[:200]
    s = pl.singleton_state(g)
    os_ = orc.singleton_state(og)
    s, mv = pl.run_iteration(g, s, sub)
    omv = orc.run_iteration(og, os_, sub)
    assert mv == omv
    assert np.array_equal(s.assignment, os_.assignment)
    assert np.array_equal(s.a_tot, os_.a_tot)
    assert np.array_equal(s.w_internal, os_.w_internal)


def test_edge_cases():
    with pytest.raises(pl.GraphParseError):
        pl.Graph.from_edges([0], [1], [0.0])
    with pytest.raises(ValueError):
        pl.Graph.from_edges([0], [5], [1.0], num_vertices=3)
    g = pl.Graph.from_edges([], [], num_vertices=3)
    assert g.num_edges == 0 and g.total_weight == 0.0
    with pytest.raises(pl.EdgelessGraphError):
        pl.run(g)
    g = pl.Graph.from_edges([0, 1], [0, 1], [2.0, 1.0])
    s, st = pl.run_phase(g, pl.RunConfig(use_vf=False, use_coloring=False,
                                         max_iterations_per_phase=50))
    assert st.iterations == 1 and st.total_moves == 0
    g = pl.Graph.from_edges([0], [1], num_vertices=4)   # isolated vertices
    assert g.degree(2) == 0 and g.weighted_degrees[3] == 0.0
    g.validate()


def _tie_graph(n_leaves, w=0.1, extra=3):
    """A hub (vertex 0) whose neighbour communities give bitwise-identical
    gains: every leaf has the same fp weight to the hub and the same degree,
    so certification must fall back to exact folds (and, above MAXS ties, to
    the fully exact path)."""
    u, v, ww = [], [], []
    nxt = n_leaves + 1
    for leaf in range(1, n_leaves + 1):
        u.append(0), v.append(leaf), ww.append(w)
        for _ in range(extra):                       # private pendant triangle
            u.append(leaf), v.append(nxt), ww.append(0.3)
            nxt += 1
    return np.array(u), np.array(v), np.array(ww), nxt


@pytest.mark.parametrize("n_leaves", [10, 40, 3000, 12000, 20000])
def test_exact_ties_are_resolved_like_the_reference(orc, n_leaves):
    u, v, w, n = _tie_graph(n_leaves)
    g = pl.Graph.from_edges(u, v, w, num_vertices=n)
    og = orc.from_edges(u, v, w, num_vertices=n)
    for flags_colored in (False, True):
        s = pl.singleton_state(g)
        os_ = orc.singleton_state(og)
        if flags_colored:
            col = pl.color_graph(g)
            for stage in col.classes():
                s, _ = pl.run_iteration(g, s, stage)
                orc.run_iteration(og, os_, stage)
        else:
            s, _ = pl.run_iteration(g, s, np.arange(n))
            orc.run_iteration(og, os_, np.arange(n))
        assert np.array_equal(s.assignment, os_.assignment)
        assert np.array_equal(s.a_tot, os_.a_tot)
        assert np.array_equal(s.w_internal, os_.w_internal)


@pytest.mark.parametrize("scale,cutoff", [(16, 0), (16, 100_000), (17, 0)])
def test_rmat_with_hubs_matches_oracle(orc, scale, cutoff):
    from paper_1410_1237_b200 import synthetic as syn
    u, v, w = syn.rmat_records(scale, 16, seed=5)
    n = 1 << scale
    og = orc.from_edges(u, v, w, num_vertices=n)
    g = pl.Graph.from_edges(u, v, w, num_vertices=n)
    assert g.max_degree > 2048        # the hub tier is exercised
    oh = orc.run(og, color_cutoff=cutoff, max_iterations=30)
    h = pl.run(g, pl.RunConfig(color_cutoff=cutoff, max_iterations_per_phase=30))
    assert np.array_equal(h.final_assignment, oh.final_assignment)
    assert h.final_modularity == oh.final_modularity


def _multi_hub_graph(seed=3):
    """Random background plus vertices on both sides of the block-tier / hub-tier
    boundary (degree 2048) and hubs up to 40000 entries."""
    rng = np.random.default_rng(seed)
    n = 60000
    u = [rng.integers(0, n, 200000)]
    v = [rng.integers(0, n, 200000)]
    for h, d in enumerate([2030, 2049, 9000, 16370, 16385, 20000, 40000]):
        u.append(np.full(d, h))
        v.append(rng.choice(np.arange(100, n), d, replace=False))
    u, v = np.concatenate(u), np.concatenate(v)
    w = rng.uniform(1.0, 10.0, len(u))
    return u, v, w, n


@pytest.mark.parametrize("cutoff", [0, 100_000])
def test_hub_tiers_match_oracle(orc, cutoff):
    u, v, w, n = _multi_hub_graph()
    og = orc.from_edges(u, v, w, num_vertices=n)
    g = pl.Graph.from_edges(u, v, w, num_vertices=n)
    deg = np.diff(g.adjacency_offsets)
    assert (deg <= 2048).sum() >= 1 and (deg > 2048).sum() >= 6
    oh = orc.run(og, color_cutoff=cutoff, max_iterations=30)
    h = pl.run(g, pl.RunConfig(color_cutoff=cutoff, max_iterations_per_phase=30))
    assert np.array_equal(h.final_assignment, oh.final_assignment)
    assert h.final_modularity == oh.final_modularity


@pytest.mark.parametrize("cutoff", [0, 100_000])
def test_many_hubs_hash_tier_matches_oracle(orc, cutoff):
    """Two dozen hubs in one stage (uncoloured, and colour 0 since no two hubs
    are adjacent): more hubs than the dense per-hub arrays take (16), so the
    hash-table hub path runs (the dense path is covered by the tests above)."""
    rng = np.random.default_rng(11)
    n = 40000
    u = [rng.integers(0, n, 120000)]
    v = [rng.integers(0, n, 120000)]
    for h in range(24):
        d = int(rng.integers(2100, 9000))
        u.append(np.full(d, h))
        v.append(rng.choice(np.arange(100, n), d, replace=False))
    u, v = np.concatenate(u), np.concatenate(v)
    w = rng.uniform(1.0, 10.0, len(u))
    og = orc.from_edges(u, v, w, num_vertices=n)
    g = pl.Graph.from_edges(u, v, w, num_vertices=n)
    assert (np.diff(g.adjacency_offsets) > 2048).sum() >= 24
    oh = orc.run(og, color_cutoff=cutoff, max_iterations=30)
    h = pl.run(g, pl.RunConfig(color_cutoff=cutoff, max_iterations_per_phase=30))
    assert np.array_equal(h.final_assignment, oh.final_assignment)
    assert h.final_modularity == oh.final_modularity


def test_distributed_iteration_single_rank_cuda(orc):
    """The multi-GPU driver with the CUDA callbacks (world 1) equals the
    phase engine's coloured iteration and the oracle."""
    from paper_1410_1237_b200 import dist as pdist
    from paper_1410_1237_b200 import synthetic as syn
    import torch
    u, v, w = syn.rmat_records(13, 16, seed=2)
    n = 1 << 13
    g = pl.Graph.from_edges(u, v, w, num_vertices=n)
    og = orc.from_edges(u, v, w, num_vertices=n)
    col = pl.color_graph(g)
    off, vtx = col.device_classes()
    stages = [vtx[int(off[c]):int(off[c + 1])] for c in range(col.num_colors)]
    stages_h = [s_.cpu().numpy().astype(np.int64) for s_ in stages]
    s = pl.singleton_state(g)
    from paper_1410_1237_b200 import _lib
    ops = pdist.CudaStageOps(g, s, stages, _lib.F_INDEPENDENT)
    it = pdist.DistributedIteration(ops, stages_h, pdist.partition_bounds(g.adjacency_offsets, 1),
                                    0, 1)
    os_ = orc.singleton_state(og)
    for _ in range(2):
        moves, q = it.run()
        omoves = sum(orc.run_iteration(og, os_, st) for st in stages_h)
        assert moves == omoves and q == orc.modularity(og, os_)
    assert np.array_equal(s.assignment, os_.assignment)
