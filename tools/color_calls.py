"""Every color_graph call of a full run(): graph size, colours, rounds, wall
time (synchronised).   python tools/color_calls.py [config]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1410_1237_b200 as pl  # noqa: E402
from paper_1410_1237_b200 import engine, heuristics  # noqa: E402
from paper_1410_1237_b200 import synthetic as syn  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c4_chung_lu"
orig = heuristics.color_graph
rows = []


def timed(g, *a, **k):
    torch.cuda.synchronize()
    t = time.perf_counter()
    c = orig(g, *a, **k)
    torch.cuda.synchronize()
    rows.append((g.num_vertices, g.nnz,
                 c.num_colors, getattr(c, "rounds", -1), (time.perf_counter() - t) * 1e3))
    return c


heuristics.color_graph = timed
engine.color_graph = timed
g = syn.config_graph(cfg)
for rep in range(2):
    rows.clear()
    pl.run(g)
    torch.cuda.synchronize()
    for r in rows:
        print(f"rep {rep}: n={r[0]} nnz={r[1]} colours={r[2]} rounds={r[3]} {r[4]:.1f} ms")
