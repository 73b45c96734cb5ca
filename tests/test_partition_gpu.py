"""The 1D vertex-partitioned pipeline (paper_1410_1237_b200.partition) with W
ranks as W processes on ONE GPU, exchanging over gloo (host copies), against
the single-graph pipeline bit for bit:

* construction: each rank's owned rows, k, self loops, degrees, m, |E|, max
  degree and merge count equal the whole graph's (PL/graph.py:88-147);
* vertex following's map and colouring's colours (PL/heuristics.py:46-118);
* the whole run (PL/engine.py:259-315): per-phase iterations and q_end, final
  assignment, final Q, community count -- coloured (every stage's decided
  slices exchanged) and uncoloured (live e_a / e_b folded by the row owners
  and exchanged, PLV_STEP_LIVE).

No kernel waits on another rank's kernel: every exchange is a host-side gloo
collective between launches."""

import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

pl = pytest.importorskip("paper_1410_1237_b200")


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _run(world, scale, cfg_kw, chunk=1 << 30, nccl=False):
    import torch.multiprocessing as mp
    import part_worker
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=part_worker.worker,
                         args=(r, world, port, scale, cfg_kw, q, chunk, nccl))
             for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        r, d = q.get(timeout=900)
        res[r] = d
    for p in procs:
        p.join(timeout=60)
    for r in range(world):
        assert "error" not in res[r], res[r]["error"]
    return res


def _whole(scale):
    from paper_1410_1237_b200 import synthetic as syn
    u, v, w, n = syn.rmat_device(scale, 8, seed=5)
    return pl.Graph.from_device_records(u, v, w, n)


@pytest.mark.parametrize("world,cfg,chunk,nccl", [
    (2, "colored", 1 << 30, False), (3, "colored", 7919, False), (2, "uncolored", 1 << 30, False),
    (1, "colored", 1 << 30, True), (1, "uncolored", 1 << 30, True),
    (4, "colored", 1 << 30, False)])
def test_partitioned_pipeline(world, cfg, chunk, nccl):
    """W gloo ranks (host-stepped stages), or one rank with a 1-rank NCCL
    communicator (the iteration graph with its captured all-gathers and, for
    uncoloured phases, the live folds); chunk: records per routing call."""
    scale = 13
    cfg_kw = (dict(color_cutoff=0, max_iterations_per_phase=200) if cfg == "colored"
              else dict(use_coloring=False, max_iterations_per_phase=200))
    res = _run(world, scale, cfg_kw, chunk, nccl)
    g = _whole(scale)
    off, nbr, w = g.adjacency_offsets, g.neighbors, g.weights
    for r in range(world):
        d = res[r]["rows"]
        lo, hi = d["lo"], d["hi"]
        assert np.array_equal(d["off"][lo:hi + 1] + off[lo], off[lo:hi + 1])
        assert np.array_equal(d["nbr"], nbr[off[lo]:off[hi]])
        assert np.array_equal(d["w"], w[off[lo]:off[hi]])
        assert np.array_equal(d["k"], g.weighted_degrees)
        assert np.array_equal(d["selfw"], g.self_loop_weights)
        assert np.array_equal(d["deg"], np.diff(off))
        assert d["m"] == g.total_weight and d["ne"] == g.num_edges
        assert d["md"] == g.max_degree and d["integral"] == g.integral
        assert d["merged"] == g.merged_duplicates
    vf = pl.vf_compact(g)
    col = pl.color_graph(vf.graph)
    h = pl.run(g, pl.RunConfig(**cfg_kw))
    for r in range(world):
        d = res[r]
        assert np.array_equal(d["vmap"], vf.vertex_map)
        assert np.array_equal(d["colors"], col.colors)
        assert d["iters"] == [p.stats.iterations for p in h.phases]
        assert d["qend"] == [p.stats.q_end for p in h.phases]
        assert np.array_equal(d["assign"], h.final_assignment)
        assert d["q"] == h.final_modularity
        assert d["ncomm"] == h.num_communities
