"""Host-side logic of the 1D vertex partition (paper_1410_1237_b200.partition),
on CPU: the Exchange collectives over gloo (world 2 and 3), the balanced
bounds, and -- with the CPU oracle as the CSR builder -- the routing argument
the construction rests on: a rank that builds Graph.from_edges (PL/graph.py:
88-147) from the records touching its rows, in global order, gets every owned
row, weighted degree and self loop exactly as the whole-graph build."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _ex_worker(rank, world, port):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1410_1237_b200.partition import Exchange, balanced_bounds
    ex = Exchange()
    assert (ex.rank, ex.world, ex.host) == (rank, world, True)
    # all_to_all_v: rank r sends (r, d, i) triples, d ascending, i < r + d + 1
    send = [[(rank, d, i) for i in range(rank + d + 1)] for d in range(world)]
    flat = [x for part in send for x in part]
    t = torch.tensor([100 * a + 10 * b + c for a, b, c in flat], dtype=torch.int64)
    (got,), recv = ex.all_to_all_v([t], [len(p) for p in send])
    want = [100 * s + 10 * rank + i for s in range(world) for i in range(s + rank + 1)]
    assert got.tolist() == want and recv == [s + rank + 1 for s in range(world)]
    # all_gather_v: rank r contributes r + 1 copies of r (empty allowed)
    g = ex.all_gather_v(torch.full((rank,), rank, dtype=torch.int32))
    assert g.tolist() == [r for r in range(world) for _ in range(r)]
    x = torch.zeros(6, dtype=torch.float64)
    x[rank] = 1.5 + rank
    ex.all_reduce_(x)
    assert x.tolist()[:world] == [1.5 + r for r in range(world)]
    assert ex.sum_int(rank) == sum(range(world)) and ex.max_int(rank) == world - 1
    rng = np.random.default_rng(rank)
    u = torch.from_numpy(rng.integers(0, 1000, 500).astype(np.int32))
    v = torch.from_numpy(rng.integers(0, 100, 500).astype(np.int32))  # skewed to low ids
    b = balanced_bounds(u, v, 1000, ex, buckets=64)
    assert b[0] == 0 and b[-1] == 1000 and np.all(np.diff(b) >= 0) and len(b) == world + 1
    allb = [torch.from_numpy(b) for _ in range(world)]
    dist.all_gather(allb, torch.from_numpy(b))
    assert all(np.array_equal(x.numpy(), b) for x in allb)
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_exchange_collectives(world):
    mp.start_processes(_ex_worker, args=(world, _free_port()), nprocs=world, join=True,
                       start_method="spawn")


@pytest.mark.parametrize("world", [2, 3, 5])
def test_owner_routed_build_equals_whole(orc, world):
    rng = np.random.default_rng(world)
    n = 300
    u = rng.integers(0, n, 4000)
    v = (u + rng.integers(0, 40, 4000)) % n  # locality, duplicates, self loops
    w = rng.uniform(0.5, 3.0, 4000)
    g = orc.from_edges(u, v, w, num_vertices=n)
    bounds = np.linspace(0, n, world + 1).astype(np.int64)
    owner = lambda x: np.searchsorted(bounds, x, side="right") - 1  # noqa: E731
    # each rank generated a contiguous range of the records
    cuts = np.linspace(0, len(u), world + 1).astype(int)
    for r in range(world):
        lo, hi = bounds[r], bounds[r + 1]
        # received: from every sender in rank order, its records touching [lo, hi)
        idx = np.concatenate([np.arange(cuts[s], cuts[s + 1])[
            (owner(np.minimum(u, v)[cuts[s]:cuts[s + 1]]) == r) |
            (owner(np.maximum(u, v)[cuts[s]:cuts[s + 1]]) == r)] for s in range(world)])
        loc = orc.from_edges(u[idx], v[idx], w[idx], num_vertices=n, count_merges=False)
        o, lo_e, hi_e = loc.adjacency_offsets, g.adjacency_offsets[lo], g.adjacency_offsets[hi]
        assert np.array_equal(np.diff(o)[lo:hi], np.diff(g.adjacency_offsets)[lo:hi])
        assert np.array_equal(loc.neighbors[o[lo]:o[hi]], g.neighbors[lo_e:hi_e])
        assert np.array_equal(loc.weights[o[lo]:o[hi]], g.weights[lo_e:hi_e])
        assert np.array_equal(loc.weighted_degrees[lo:hi], g.weighted_degrees[lo:hi])
        assert np.array_equal(loc.self_loop_weights[lo:hi], g.self_loop_weights[lo:hi])
