"""Multi-rank host logic of the partitioned local-move iteration, on CPU with
the gloo backend (world_size 2 and 3): partitioning, per-stage slicing, the
rank-ordered all-gather and the replicated exact apply must reproduce the
single-rank result bit for bit.  The per-rank compute is the CPU oracle
(the GPU path uses the same driver with libplv callbacks)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1410_1237_b200 import dist as pdist
from paper_1410_1237_b200 import synthetic as syn


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


class OracleOps:
    """Stage callbacks on the CPU oracle (test infrastructure)."""

    def __init__(self, orc, g, s, stages):
        self.orc, self.g, self.s, self.stages = orc, g, s, stages

    def decide(self, a, lo, hi):
        tg, mv = self.orc.decide(self.g, self.s, self.stages[a][lo:hi])
        z = torch.zeros(hi - lo, dtype=torch.float64)
        return pdist.DecideSlice(torch.from_numpy(tg.copy()), torch.from_numpy(mv.copy()), z, z)

    def apply(self, a, d):
        return self.orc.apply(self.g, self.s, self.stages[a], d.target.numpy(), d.moved.numpy())

    def modularity(self):
        return self.orc.modularity(self.g, self.s)


def _graph(orc):
    u, v, w = syn.rmat_records(11, 8, seed=9)
    return orc.from_edges(u, v, w, num_vertices=1 << 11)


def _worker(rank, world, port, colored, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import sys
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(__file__)), "oracle"))
    import oracle as orc
    g = _graph(orc)
    stages = (orc.color_graph(g).classes() if colored
              else [np.arange(g.num_vertices, dtype=np.int64)])
    s = orc.singleton_state(g)
    bounds = pdist.partition_bounds(g.adjacency_offsets, world)
    it = pdist.DistributedIteration(OracleOps(orc, g, s, stages), stages, bounds, rank, world)
    res = []
    for _ in range(3):
        moves, q = it.run()
        res.append((moves, q))
    out[rank] = (res, s.assignment.copy(), s.a_tot.copy(), s.w_internal.copy(), s.sizes.copy())
    dist.destroy_process_group()


def _single(orc, colored):
    g = _graph(orc)
    stages = (orc.color_graph(g).classes() if colored
              else [np.arange(g.num_vertices, dtype=np.int64)])
    s = orc.singleton_state(g)
    res = []
    for _ in range(3):
        moves = sum(orc.run_iteration(g, s, st) for st in stages)
        res.append((moves, orc.modularity(g, s)))
    return res, s


def test_partition_bounds_balance_entries():
    off = np.concatenate([[0], np.cumsum(np.r_[np.full(10, 100), np.ones(990, np.int64)])])
    b = pdist.partition_bounds(off, 4)
    assert b[0] == 0 and b[-1] == 1000 and np.all(np.diff(b) >= 0)
    loads = np.diff(off[b])
    assert loads.max() <= off[-1] / 4 + 100
    st = np.array([1, 5, 20, 400, 999])
    sl = pdist.stage_slices(st, b)
    assert sl[0] == 0 and sl[-1] == len(st) and np.all(np.diff(sl) >= 0)


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("colored", [True, False])
def test_distributed_iteration_matches_single_rank(orc, world, colored):
    ref_res, ref_s = _single(orc, colored)
    port = _free_port()
    with mp.Manager() as mgr:
        out = mgr.dict()
        mp.spawn(_worker, args=(world, port, colored, out), nprocs=world, join=True)
        results = [out[r] for r in range(world)]
    for res, assign, atot, wint, sizes in results:
        assert res == ref_res
        assert np.array_equal(assign, ref_s.assignment)
        assert np.array_equal(atot, ref_s.a_tot)
        assert np.array_equal(wint, ref_s.w_internal)
        assert np.array_equal(sizes, ref_s.sizes)
