"""Full-size golden fingerprints of the BASELINE configs (TEST INFRASTRUCTURE).

For each config this runs the pinned CPU oracle (oracle/plv_oracle.c, itself
pinned to the compiled reference by tests/test_oracle_pins.py) on the
numpy-generated records -- the same counter-based RNG the device generator
uses (tests/test_gpu_parity.py proves them equal) -- and stores fingerprints
that a GPU test can check without the oracle or /root/reference on the box:

* CSR (Graph.from_edges, PL/graph.py:88-147): n, nnz, M, m bits, sha256 of
  offsets / neighbours / weights;
* vertex following (PL/heuristics.py:46-89): map sha, coarse n / nnz;
* colouring (PL/heuristics.py:92-118): number of colours, colours sha;
* one coloured phase-1 iteration from the singleton state over every colour
  class (PL/engine.py:186-197): moves, Q bits and the sha of assignment,
  a_tot, w_internal, sizes;
* the whole run (PL/engine.py:259-315, default RunConfig): per-phase
  iterations, moves, q_end bits, colored flag; final assignment sha, final Q
  bits, number of communities.

Arrays are hashed in the reference's dtypes (int64 / float64, C order).

    python tests/golden/make_fullsize.py c3_grid c4_chung_lu rmat22 ...

Writes tests/golden/fullsize_<name>.json.  C3 takes ~2 min and C4 ~15 min on
one core of the build container; R-MAT s22 (the scaled C5) ~5 min.
"""

from __future__ import annotations

import hashlib
import json
import os
import struct
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
sys.path.insert(0, ROOT)

import oracle as orc  # noqa: E402

from paper_1410_1237_b200 import synthetic as syn  # noqa: E402  (numpy record generators)

OUT = os.path.dirname(os.path.abspath(__file__))

# name -> (records generator, kwargs, num_vertices, config name for the device)
CASES = {
    "c1_sbm": ("c1_sbm", {}),
    "c2_rmat20": ("c2_rmat20", {}),
    "c3_grid": ("c3_grid", {}),
    "c4_chung_lu": ("c4_chung_lu", {}),
    "rmat22": ("c5_rmat28", {"scale": 22}),
    "rmat24": ("c5_rmat28", {"scale": 24}),
}


def sha(a, dtype) -> str:
    return hashlib.sha256(np.ascontiguousarray(np.asarray(a).astype(dtype, copy=False))
                          .tobytes()).hexdigest()[:16]


def fbits(x: float) -> str:
    return struct.pack(">d", float(x)).hex()


def records(name: str):
    cfg, kw = CASES[name]
    host, _dev, params = syn.CONFIGS[cfg]
    params = {**params, **kw}
    u, v, w = host(seed=0, **params)
    return u, v, w, syn.config_num_vertices(cfg, **kw), cfg, kw


def fingerprint(name: str) -> dict:
    t0 = time.time()
    u, v, w, n, cfg, kw = records(name)
    out = {"name": name, "config": cfg, "params": kw, "seed": 0, "records": int(len(u))}
    g = orc.from_edges(u, v, w, num_vertices=n)
    del u, v, w
    out["csr"] = dict(n=g.num_vertices, nnz=int(len(g.neighbors)), num_edges=g.num_edges,
                      total_weight=fbits(g.total_weight),
                      offsets=sha(g.adjacency_offsets, np.int64),
                      neighbors=sha(g.neighbors, np.int64),
                      weights=sha(g.weights, np.float64))
    t1 = time.time()
    vf = orc.vf_compact(g)
    gv = vf.graph
    out["vf"] = dict(vertex_map=sha(vf.vertex_map, np.int64), n=gv.num_vertices,
                     nnz=int(len(gv.neighbors)), neighbors=sha(gv.neighbors, np.int64),
                     weights=sha(gv.weights, np.float64))
    col = orc.color_graph(gv)
    out["coloring"] = dict(num_colors=col.num_colors, colors=sha(col.colors, np.int64))
    s = orc.singleton_state(gv)
    moves = 0
    for st in col.classes():
        moves += orc.run_iteration(gv, s, st)
    out["colored_iteration"] = dict(
        moves=int(moves), q=fbits(orc.modularity(gv, s)),
        assignment=sha(s.assignment, np.int64), a_tot=sha(s.a_tot, np.float64),
        w_internal=sha(s.w_internal, np.float64), sizes=sha(s.sizes, np.int64))
    del s, col, vf, gv
    t2 = time.time()
    h = orc.run(g)
    out["run"] = dict(
        phases=[dict(iterations=p.iterations, moves=int(p.total_moves), q_end=fbits(p.q_end),
                     colored=bool(p.colored), hit_cap=bool(p.hit_cap)) for p in h.phases],
        final_assignment=sha(h.final_assignment, np.int64),
        final_modularity=fbits(h.final_modularity),
        final_modularity_float=h.final_modularity,
        num_communities=int(h.num_communities))
    t3 = time.time()
    out["oracle_seconds"] = dict(build=round(t1 - t0, 1), iteration=round(t2 - t1, 1),
                                 run=round(t3 - t2, 1))
    return out


def main(names):
    for name in names:
        fp = fingerprint(name)
        path = os.path.join(OUT, f"fullsize_{name}.json")
        with open(path, "w") as f:
            json.dump(fp, f, indent=1, sort_keys=True)
            f.write("\n")
        print(name, fp["run"]["final_assignment"], fp["run"]["final_modularity_float"],
              fp["oracle_seconds"], flush=True)


if __name__ == "__main__":
    main(sys.argv[1:] or ["c1_sbm", "c2_rmat20", "c3_grid", "c4_chung_lu", "rmat22"])
