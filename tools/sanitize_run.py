"""Workload for compute-sanitizer (tools/gpu/sanitize.sh): the golden grid48
and rmat10 graphs through run() (coloured and uncoloured phases, VF,
rebuilds), plus a direct coloured iteration and an uncoloured iteration."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1410_1237_b200 as pl  # noqa: E402

G = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden")
for name in ("grid48", "rmat10"):
    z = np.load(os.path.join(G, name + ".npz"))
    g = pl.Graph.from_edges(z["u"], z["v"], z["w"], num_vertices=int(z["n"]))
    h = pl.run(g, pl.RunConfig(color_cutoff=0, max_iterations_per_phase=50))
    col = pl.color_graph(g)
    s = pl.singleton_state(g)
    for st in col.classes():
        s, _ = pl.run_iteration(g, s, st)
    s2 = pl.singleton_state(g)
    s2, mv = pl.run_iteration(g, s2, np.arange(g.num_vertices))
    print(name, h.final_modularity, len(h.phases), mv)
