"""GPU: the ahead tables (csrc/ahead.cuh) -- small colour classes of an
integral coloured phase decided from per-vertex tables accumulated at the
start of their window of stages and kept current by the applies' pushes --
against the oracle's stage-by-stage decide + apply (PL/engine.py:140-163,
PL/_kernels.pyx:21-145): state bits after every iteration, and whole runs.

PLV_AHEAD_LOWDEG=1 lets low-degree stages qualify, so small graphs drive the
path (every stage but the first becomes an ahead stage); the default rule
(high-degree stages only) is exercised by the hub graphs."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

pl = pytest.importorskip("paper_1410_1237_b200")


def _hub_graph(nh, leaves, per_hub, seed, wmax=3):
    """nh mutually adjacent hubs over random leaves; integer weights."""
    rng = np.random.default_rng(seed)
    n = nh + leaves
    hubs = np.arange(nh)
    others = np.arange(nh, n)
    iu, ju = np.triu_indices(nh, 1)
    u, v = [hubs[iu]], [hubs[ju]]
    for h in hubs:
        t = rng.choice(others, size=per_hub, replace=False)
        u.append(np.full(per_hub, h))
        v.append(t)
    a = rng.choice(others, size=3 * leaves)
    b = rng.choice(others, size=3 * leaves)
    keep = a != b
    u.append(a[keep])
    v.append(b[keep])
    u, v = np.concatenate(u), np.concatenate(v)
    w = rng.integers(1, wmax + 1, len(u)).astype(np.float64)
    return u, v, w, n


def _graphs(name):
    from paper_1410_1237_b200 import synthetic as syn
    if name == "chung_lu":
        host, _, params = syn.CONFIGS["c4_chung_lu"]
        u, v, w = host(seed=5, **{**params, "n": 1 << 15, "max_degree": 3000.0})
        return u, v, w, 1 << 15
    if name == "sbm":
        host, _, params = syn.CONFIGS["c1_sbm"]
        u, v, w = host(seed=2, **params)
        return u, v, w, syn.config_num_vertices("c1_sbm")
    if name == "rmat_int":  # R-MAT hubs (rows of thousands of entries), integer weights
        u, v, w = syn.rmat_records(scale=14, edge_factor=16, seed=11)
        return u, v, np.ceil(w * 3.0), 1 << 14
    if name == "hubs":
        return _hub_graph(40, 6000, 700, 1)
    if name == "hubs_big":
        return _hub_graph(24, 20000, 5000, 3, wmax=1)
    raise KeyError(name)


def _iterations(orc, u, v, w, n, iters):
    from paper_1410_1237_b200.engine import PhaseEngine
    g = pl.Graph.from_edges(u, v, w, num_vertices=n)
    og = orc.from_edges(u, v, w, num_vertices=n)
    col = pl.color_graph(g)
    s = pl.singleton_state(g)
    d = s.device()
    state = pl.CommunityState.from_device(d["assignment"], d["a_tot"], d["w_internal"], d["sizes"])
    eng = PhaseEngine(g, state, col)
    stats = eng.ahead_stats()
    os_ = orc.singleton_state(og)
    classes = col.classes()
    for it in range(iters):
        q, moves, _ = eng.iterate()
        omoves = 0
        for stage in classes:
            omoves += orc.run_iteration(og, os_, stage)
        assert moves == omoves, it
        assert np.array_equal(d["assignment"].cpu().numpy(), os_.assignment), it
        assert np.array_equal(d["a_tot"].cpu().numpy(), os_.a_tot), it
        assert np.array_equal(d["w_internal"].cpu().numpy(), os_.w_internal), it
        assert np.array_equal(d["sizes"].cpu().numpy(), os_.sizes), it
        assert q == orc.modularity(og, os_), it
    eng.close()
    return stats


@pytest.mark.parametrize("name", ["chung_lu", "sbm", "hubs"])
def test_ahead_lowdeg_iterations(orc, monkeypatch, name):
    monkeypatch.setenv("PLV_AHEAD_LOWDEG", "1")
    u, v, w, n = _graphs(name)
    stats = _iterations(orc, u, v, w, n, 4)
    assert stats["stages"] > 0 and stats["vertices"] > 0 and stats["fix_entries"] > 0, stats


@pytest.mark.parametrize("name", ["hubs", "hubs_big", "chung_lu", "rmat_int"])
def test_ahead_default_rule_iterations(orc, monkeypatch, name):
    monkeypatch.delenv("PLV_AHEAD_LOWDEG", raising=False)
    monkeypatch.delenv("PLV_AHEAD", raising=False)
    u, v, w, n = _graphs(name)
    stats = _iterations(orc, u, v, w, n, 3)
    if name != "chung_lu":  # hubs are mutually adjacent: one high-degree stage each
        assert stats["stages"] >= 8 and stats["fix_entries"] > 0, stats
    print(name, stats)


@pytest.mark.parametrize("name,slots", [("chung_lu", "60000"), ("hubs", "20000"), ("sbm", "50000")])
def test_ahead_several_windows(orc, monkeypatch, name, slots):
    """A small slot budget cuts the run of ahead stages into several windows
    that reuse one table region (each window's accumulation at its start)."""
    monkeypatch.setenv("PLV_AHEAD_LOWDEG", "1")
    monkeypatch.setenv("PLV_AHEAD_SLOTS", slots)
    u, v, w, n = _graphs(name)
    stats = _iterations(orc, u, v, w, n, 3)
    assert stats["windows"] >= 2, stats


def test_ahead_off_is_the_tier_path(orc, monkeypatch):
    monkeypatch.setenv("PLV_AHEAD", "0")
    u, v, w, n = _graphs("hubs")
    stats = _iterations(orc, u, v, w, n, 2)
    assert stats["stages"] == 0


@pytest.mark.parametrize("name,lowdeg", [("chung_lu", "1"), ("hubs", "1"), ("hubs_big", "0"),
                                         ("sbm", "1"), ("rmat_int", "0"), ("rmat_int", "1")])
def test_ahead_runs_match_oracle(orc, monkeypatch, name, lowdeg):
    monkeypatch.setenv("PLV_AHEAD_LOWDEG", lowdeg)
    u, v, w, n = _graphs(name)
    g = pl.Graph.from_edges(u, v, w, num_vertices=n)
    og = orc.from_edges(u, v, w, num_vertices=n)
    oh = orc.run(og, color_cutoff=0, max_iterations=60)
    h = pl.run(g, pl.RunConfig(color_cutoff=0, max_iterations_per_phase=60))
    assert [p.stats.iterations for p in h.phases] == [p.iterations for p in oh.phases]
    assert np.array_equal(h.final_assignment, oh.final_assignment)
    assert h.final_modularity == oh.final_modularity


def test_singleton_shortcut_needs_singleton_sizes(orc):
    """The singleton-state kernels skip the size gathers of the singleton-pair
    guard (PL/_kernels.pyx:92-98), so the device check must reject a state whose
    assignment is the identity but whose sizes are not all 1: the general
    kernels then decide it, as the reference does."""
    from paper_1410_1237_b200 import synthetic as syn
    u, v, w = syn.gnm_records(400, 2400, seed=9, weight_range=(0.0, 2.0))
    g = pl.Graph.from_edges(u, v, w, num_vertices=400)
    og = orc.from_edges(u, v, w, num_vertices=400)
    sub = np.arange(400)
    moved = {}
    for sz in (1, 2):
        s = pl.singleton_state(g)
        os_ = orc.singleton_state(og)
        s.sizes[:] = sz
        os_.sizes[:] = sz
        s, mv = pl.run_iteration(g, s, sub)
        omv = orc.run_iteration(og, os_, sub)
        assert mv == omv
        assert np.array_equal(s.assignment, os_.assignment)
        assert np.array_equal(s.sizes, os_.sizes)
        assert np.array_equal(s.a_tot, os_.a_tot)
        moved[sz] = mv
    assert moved[1] != moved[2]  # the guard did decide moves in the consistent state
