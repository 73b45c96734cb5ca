"""Pin the CPU oracle (oracle/) before trusting it.

1. numpy's arithmetic rules that the reference relies on:
   pairwise .sum(), the reduceat seed rule, the sequential weighted bincount
   and lexsort stability -- checked against the installed numpy.
2. Oracle == golden fixtures produced by the unmodified reference
   (tests/golden/make_golden.py), bit for bit.
3. Oracle == live reference (oracle/_ref) on extra random cases when present.
"""

import numpy as np
import pytest

from conftest import GOLDEN_CASES, load_golden

import oracle as O


def py_pairwise(a):
    n = len(a)
    if n < 8:
        r = 0.0
        for x in a:
            r += x
        return r
    if n <= 128:
        r = [float(x) for x in a[:8]]
        i = 8
        while i < n - (n % 8):
            for j in range(8):
                r[j] += a[i + j]
            i += 8
        res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]))
        while i < n:
            res += a[i]
            i += 1
        return res
    n2 = n // 2
    n2 -= n2 % 8
    return py_pairwise(a[:n2]) + py_pairwise(a[n2:])


@pytest.mark.parametrize("n", [0, 1, 5, 8, 9, 100, 128, 129, 257, 1000, 8193, 100_000,
                               1_000_003, 4_000_000])
def test_numpy_sum_is_pairwise(n):
    rng = np.random.default_rng(n)
    a = rng.random(n) * 10.0 ** rng.uniform(-6, 6, n)
    assert O.np_sum(a) == a.sum()
    if n <= 100_000:
        assert 0.0 + py_pairwise(list(a)) == a.sum()


@pytest.mark.parametrize("L", [1, 2, 3, 17, 130, 100_000])
def test_reduceat_seeds_with_first_element(L):
    rng = np.random.default_rng(L)
    w = rng.random(L + 7) * 9 + 1
    got = np.add.reduceat(w, np.array([0, L]))[0]
    want = w[0] if L == 1 else w[0] + O.np_sum(w[1:L])
    assert got == want


def test_weighted_bincount_is_sequential():
    rng = np.random.default_rng(5)
    idx = rng.integers(0, 50, 20000)
    w = rng.random(20000) * 1e3
    got = np.bincount(idx, weights=w, minlength=50)
    want = np.zeros(50)
    for i, x in zip(idx.tolist(), w.tolist()):
        want[i] += x
    assert np.array_equal(got, want)


def test_lexsort_is_stable():
    rng = np.random.default_rng(9)
    a = rng.integers(0, 100, 500_000)
    b = rng.integers(0, 100, 500_000)
    order = np.lexsort((b, a))
    key = a[order] * 1000 + b[order]
    same = key[1:] == key[:-1]
    assert np.all(order[1:][same] > order[:-1][same])


def _graph_matches(og, z, prefix=""):
    assert np.array_equal(og.adjacency_offsets, z[prefix + "off"])
    assert np.array_equal(og.neighbors, z[prefix + "nbr"])
    assert np.array_equal(og.weights, z[prefix + "wts"])
    assert np.array_equal(og.self_loop_weights, z[prefix + "selfw"])


@pytest.mark.parametrize("case", GOLDEN_CASES)
def test_oracle_matches_golden(case):
    z = load_golden(case)
    n = int(z["n"])
    g = O.from_edges(z["u"], z["v"], z["w"], num_vertices=n)
    _graph_matches(g, z)
    assert np.array_equal(g.weighted_degrees, z["k"])
    assert g.total_weight == float(z["m"])
    assert g.num_edges == int(z["num_edges"])
    assert g.max_degree == int(z["max_degree"])
    assert g.merged_duplicates == int(z["merged"])
    vf = O.vf_compact(g)
    assert np.array_equal(vf.vertex_map, z["vf_map"])
    assert vf.merged_count == int(z["vf_merged"])
    _graph_matches(vf.graph, z, "vf_")
    assert vf.graph.total_weight == float(z["vf_m"])
    col = O.color_graph(g)
    assert np.array_equal(col.colors, z["colors"])
    s = O.singleton_state(g)
    moves, tg, mv = O.run_iteration(g, s, np.arange(n), want_decisions=True)
    assert np.array_equal(tg, z["it1_targets"]) and np.array_equal(mv, z["it1_moved"])
    assert moves == int(z["it1_moves"])
    for name, arr in (("assign", s.assignment), ("atot", s.a_tot), ("wint", s.w_internal),
                      ("sizes", s.sizes)):
        assert np.array_equal(arr, z["it1_" + name]), name
    assert O.modularity(g, s) == float(z["it1_q"])
    sp, st = O.run_phase(g, max_iterations=200, coloring=col)
    assert np.array_equal(sp.assignment, z["ph_assign"])
    assert np.array_equal(sp.a_tot, z["ph_atot"]) and np.array_equal(sp.w_internal, z["ph_wint"])
    assert st["q_end"] == float(z["ph_q"]) and st["iterations"] == int(z["ph_iters"])
    rb, ren = O.rebuild(g, sp)
    _graph_matches(rb, z, "rb_")
    assert rb.total_weight == float(z["rb_m"])
    assert np.array_equal(ren, z["rb_ren"])
    for tag, cutoff in (("run", 100_000), ("runc", 0)):
        h = O.run(g, color_cutoff=cutoff, max_iterations=300)
        assert np.array_equal(h.final_assignment, z[tag + "_assign"])
        assert h.final_modularity == float(z[tag + "_q"])
        assert h.num_communities == int(z[tag + "_ncomm"])
        qs = [q for p in h.phases for q in p.q_trace]
        ti, tq = z[tag + "_trace_i"], z[tag + "_trace_q"]
        assert qs == tq[ti[:, 2] == 2].tolist()


def test_oracle_matches_live_reference_random(ref):
    from paper_1410_1237_b200 import synthetic as syn
    for seed in range(12):
        rng = np.random.default_rng(seed)
        n = int(rng.integers(20, 400))
        if seed % 3 == 0:
            u, v, w = syn.random_weighted_multigraph_records(n, 4 * n, seed)
        else:
            u, v, w = syn.gnm_records(n, int(rng.integers(n, 4 * n)), seed,
                                      weight_range=(0.0, 5.0) if seed % 2 else None)
        rg = ref.Graph.from_edges(u, v, w, num_vertices=n)
        og = O.from_edges(u, v, w, num_vertices=n)
        assert og.same_as(rg)
        for cutoff in (0, 100_000):
            cfg = ref.RunConfig(color_cutoff=cutoff, max_iterations_per_phase=80)
            rh = ref.run(rg, cfg)
            oh = O.run(og, color_cutoff=cutoff, max_iterations=80)
            assert np.array_equal(rh.final_assignment, oh.final_assignment)
            assert rh.final_modularity == oh.final_modularity
