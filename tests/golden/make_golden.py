"""Generate the golden fixtures in tests/golden/ from the REAL reference.

Runs in the build container only (needs oracle/_ref, built from
/root/reference by oracle/build_ref.sh).  For every case it stores the input
records and what the unmodified reference (compiled Cython backend) returns:
CSR arrays and m (Graph.from_edges), vertex following, colouring, one
uncoloured iteration from the singleton state (decide targets + the state
bits after apply), a coloured phase, rebuild, and a full `run` with its trace.

    python tests/golden/make_golden.py
"""

from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(ROOT, "oracle", "_ref"))
sys.path.insert(0, ROOT)

import ref_parlouvain as ref  # noqa: E402  (the reference itself)

from paper_1410_1237_b200 import synthetic as syn  # noqa: E402  (record generators only)

OUT = os.path.dirname(os.path.abspath(__file__))
KARATE = "/root/reference/pkg/tests/data/karate.el"


def _karate():
    u, v = [], []
    for line in open(KARATE):
        line = line.strip()
        if line and not line.startswith("#"):
            a, b = line.split()[:2]
            u.append(int(a))
            v.append(int(b))
    return np.array(u), np.array(v), np.ones(len(u)), 34


def cases():
    yield "k4", (np.array([0, 0, 0, 1, 1, 2]), np.array([1, 2, 3, 2, 3, 3]), np.ones(6), 4)
    yield "two_triangles", (np.array([0, 0, 1, 3, 3, 4, 2]), np.array([1, 2, 2, 4, 5, 5, 3]),
                            np.ones(7), 6)
    yield "karate", _karate()
    u, v, w = syn.random_weighted_multigraph_records(40, 300, seed=3)
    yield "multigraph", (u, v, w, 40)
    u, v, w = syn.gnm_records(400, 1600, seed=11, weight_range=(0.0, 3.0))
    yield "gnm400", (u, v, w, 400)
    u, v, w = syn.rmat_records(10)
    yield "rmat10", (u, v, w, 1 << 10)
    u, v, w = syn.sbm_records(n=2000, block=100, p_in=0.05, p_out=0.0005)
    yield "sbm2000", (u, v, w, 2000)
    u, v, w = syn.grid_records(side=48, keep=0.9, pendants=300)
    yield "grid48", (u, v, w, 48 * 48 + 300)
    u, v, w = syn.chung_lu_records(n=4096, gamma=2.1, mean_degree=12.0, max_degree=400.0)
    yield "chunglu4096", (u, v, w, 4096)


def trace_arrays(trace):
    stages = {"vf": 0, "coloring": 1, "clustering": 2, "rebuild": 3}
    return (np.array([[r.phase, r.iteration, stages[r.stage], r.moves] for r in trace],
                     dtype=np.int64).reshape(-1, 4),
            np.array([r.modularity for r in trace], dtype=np.float64),
            np.array([r.theta for r in trace], dtype=np.float64))


def main():
    assert ref.backend.name() == "compiled"
    for name, (u, v, w, n) in cases():
        g = ref.Graph.from_edges(u, v, w, num_vertices=n)
        out = dict(u=np.asarray(u, np.int64), v=np.asarray(v, np.int64),
                   w=np.asarray(w, np.float64), n=np.int64(n),
                   off=g.adjacency_offsets, nbr=g.neighbors, wts=g.weights,
                   selfw=g.self_loop_weights, k=g.weighted_degrees,
                   m=np.float64(g.total_weight), num_edges=np.int64(g.num_edges),
                   max_degree=np.int64(g.max_degree), merged=np.int64(g.merged_duplicates))
        vf = ref.vf_compact(g)
        out.update(vf_map=vf.vertex_map, vf_merged=np.int64(vf.merged_count),
                   vf_off=vf.graph.adjacency_offsets, vf_nbr=vf.graph.neighbors,
                   vf_wts=vf.graph.weights, vf_selfw=vf.graph.self_loop_weights,
                   vf_k=vf.graph.weighted_degrees, vf_m=np.float64(vf.graph.total_weight))
        col = ref.color_graph(g)
        out.update(colors=col.colors)
        # one uncoloured iteration from singletons, with the decide outputs
        s = ref.singleton_state(g)
        kern = ref.backend.active()
        tg = np.empty(n, np.int64)
        mv = np.empty(n, np.uint8)
        kern.decide_moves(g.adjacency_offsets, g.neighbors, g.weights, g.weighted_degrees,
                          s.labels, np.arange(n, dtype=np.int64), s.assignment.copy(),
                          s.a_tot.copy(), s.sizes.copy(), g.total_weight, g.max_degree, 1, tg, mv)
        s, moves = ref.run_iteration(g, s, np.arange(n))
        out.update(it1_targets=tg, it1_moved=mv, it1_moves=np.int64(moves),
                   it1_assign=s.assignment, it1_atot=s.a_tot, it1_wint=s.w_internal,
                   it1_sizes=s.sizes, it1_q=np.float64(ref.modularity(g, s)))
        # a coloured phase and the rebuild of its state
        cfg = ref.RunConfig(use_vf=False, use_coloring=True, color_cutoff=0,
                            max_iterations_per_phase=200)
        sp, st = ref.run_phase(g, cfg, col)
        rb, ren = ref.rebuild(g, sp)
        out.update(ph_assign=sp.assignment, ph_atot=sp.a_tot, ph_wint=sp.w_internal,
                   ph_q=np.float64(st.q_end), ph_iters=np.int64(st.iterations),
                   rb_off=rb.adjacency_offsets, rb_nbr=rb.neighbors, rb_wts=rb.weights,
                   rb_selfw=rb.self_loop_weights, rb_m=np.float64(rb.total_weight), rb_ren=ren)
        # full runs: default config and colouring forced on
        for tag, cfg in (("run", ref.RunConfig(max_iterations_per_phase=300)),
                         ("runc", ref.RunConfig(color_cutoff=0, max_iterations_per_phase=300))):
            trace = []
            h = ref.run(g, cfg, trace)
            ti, tq, tt = trace_arrays(trace)
            out.update({f"{tag}_assign": h.final_assignment,
                        f"{tag}_q": np.float64(h.final_modularity),
                        f"{tag}_ncomm": np.int64(h.num_communities),
                        f"{tag}_trace_i": ti, f"{tag}_trace_q": tq, f"{tag}_trace_theta": tt})
        np.savez_compressed(os.path.join(OUT, f"{name}.npz"), **out)
        print(f"{name}: n={n} M={g.num_edges} Q(run)={out['run_q']!r} Q(runc)={out['runc_q']!r}")


if __name__ == "__main__":
    main()
