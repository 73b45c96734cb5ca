import sys, os
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import numpy as np
import paper_1410_1237_b200 as pl
from paper_1410_1237_b200.engine import PhaseEngine
from test_phase_loop import _sbm_integral, _state
for seed in (7, 11):
    u, v = _sbm_integral(seed=seed)
    g = pl.Graph.from_edges(u, v, num_vertices=1200)
    s2, st2 = _state(g)
    e2 = PhaseEngine(g, s2, None)
    q2, m2, ms2, it, total, hit2 = e2.run(1e-6, 10000)
    print("seed", seed, "it", it, "hit", hit2, "cycle", e2.cycle, "moves tail", list(m2[-4:]))
