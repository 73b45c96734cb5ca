"""GPU parity at BASELINE.json's FULL sizes against committed oracle goldens.

tests/golden/make_fullsize.py ran the pinned CPU oracle on the numpy-generated
records of every config (C1-C4 at full size, R-MAT s22 as the scaled C5) and
stored fingerprints (sha256 of the reference-dtype arrays, float bits).  Here
the same graphs are generated and built on the device and pushed through the
product API; every fingerprint must match bit for bit:

* CSR (PL/graph.py:88-147), vertex following (PL/heuristics.py:46-89),
  colouring (PL/heuristics.py:92-118);
* one coloured phase-1 iteration over all colour classes (PL/engine.py:186-197);
* the whole default run() (PL/engine.py:259-315): per-phase iterations, moves
  and q_end bits, final assignment, final Q bits, community count.
"""

import glob
import hashlib
import json
import os
import struct

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

pl = pytest.importorskip("paper_1410_1237_b200")

HERE = os.path.dirname(os.path.abspath(__file__))
CASES = sorted(glob.glob(os.path.join(HERE, "golden", "fullsize_*.json")))
IDS = [os.path.basename(p)[9:-5] for p in CASES]


def sha(a, dtype) -> str:
    return hashlib.sha256(np.ascontiguousarray(np.asarray(a).astype(dtype, copy=False))
                          .tobytes()).hexdigest()[:16]


def fbits(x: float) -> str:
    return struct.pack(">d", float(x)).hex()


def _graph(fp):
    from paper_1410_1237_b200 import synthetic as syn
    return syn.config_graph(fp["config"], seed=fp["seed"], **fp["params"])


@pytest.mark.parametrize("path", CASES, ids=IDS)
def test_fullsize_pipeline(path):
    fp = json.load(open(path))
    g = _graph(fp)
    c = fp["csr"]
    assert (g.num_vertices, g.nnz, g.num_edges) == (c["n"], c["nnz"], c["num_edges"])
    assert fbits(g.total_weight) == c["total_weight"]
    assert sha(g.adjacency_offsets, np.int64) == c["offsets"]
    assert sha(g.neighbors, np.int64) == c["neighbors"]
    assert sha(g.weights, np.float64) == c["weights"]
    vf = pl.vf_compact(g)
    gv = vf.graph
    assert sha(vf.vertex_map, np.int64) == fp["vf"]["vertex_map"]
    assert (gv.num_vertices, gv.nnz) == (fp["vf"]["n"], fp["vf"]["nnz"])
    assert sha(gv.neighbors, np.int64) == fp["vf"]["neighbors"]
    assert sha(gv.weights, np.float64) == fp["vf"]["weights"]
    col = pl.color_graph(gv)
    assert col.num_colors == fp["coloring"]["num_colors"]
    assert sha(col.colors, np.int64) == fp["coloring"]["colors"]
    s = pl.singleton_state(gv)
    moves = 0
    for stage in col.classes():
        s, mv = pl.run_iteration(gv, s, stage)
        moves += mv
    ci = fp["colored_iteration"]
    assert moves == ci["moves"]
    assert sha(s.assignment, np.int64) == ci["assignment"]
    assert sha(s.a_tot, np.float64) == ci["a_tot"]
    assert sha(s.w_internal, np.float64) == ci["w_internal"]
    assert sha(s.sizes, np.int64) == ci["sizes"]
    assert fbits(pl.modularity(gv, s)) == ci["q"]


@pytest.mark.parametrize("path", CASES, ids=IDS)
def test_fullsize_run(path):
    fp = json.load(open(path))
    g = _graph(fp)
    h = pl.run(g, pl.RunConfig())
    r = fp["run"]
    got = [dict(iterations=p.stats.iterations, moves=int(p.stats.total_moves),
                q_end=fbits(p.stats.q_end), colored=bool(p.stats.colored),
                hit_cap=bool(p.stats.hit_iteration_cap)) for p in h.phases]
    assert got == r["phases"]
    assert h.num_communities == r["num_communities"]
    assert fbits(h.final_modularity) == r["final_modularity"]
    assert sha(h.final_assignment, np.int64) == r["final_assignment"]
