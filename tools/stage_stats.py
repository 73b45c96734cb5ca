"""Per-colour-class statistics of the phase-1 coloured iteration of a config:
class size, degree profile, and how many classes consist only of vertices
above a degree threshold.

    python tools/stage_stats.py c4_chung_lu
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1410_1237_b200 as pl  # noqa: E402
from paper_1410_1237_b200 import synthetic as syn  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c4_chung_lu"
g = pl.vf_compact(syn.config_graph(cfg)).graph
col = pl.color_graph(g)
deg = np.diff(g.adjacency_offsets)
rows = []
for a, st in enumerate(col.classes()):
    d = deg[st]
    d = d[d > 1]  # active (a self loop alone is inactive)
    rows.append((a, len(st), len(d), int((d <= 12).sum()), int(((d > 12) & (d <= 128)).sum()),
                 int(((d > 128) & (d <= 2048)).sum()), int((d > 2048).sum()),
                 int(d.max()) if len(d) else 0, int(d.sum())))
print(f"{cfg}: n={g.num_vertices} nnz={g.nnz} colours={col.num_colors}")
print("class size active t0 t1 t2/3 hub maxdeg entries")
for r in rows:
    if r[0] < 20 or r[0] % 10 == 0:
        print(*r)
R = np.array(rows)
small = R[(R[:, 3] == 0) & (R[:, 4] == 0)]
print("classes with only deg>128 active vertices:", len(small),
      "max vertices", small[:, 2].max() if len(small) else 0,
      "max deg", small[:, 7].max() if len(small) else 0,
      "entries p50/p90/max", np.percentile(small[:, 8], [50, 90, 100]) if len(small) else 0)
for lim in (8, 16, 32, 64):
    m = R[:, 2] <= lim
    print(f"classes with <= {lim} active vertices: {m.sum()}, max deg {R[m, 7].max() if m.any() else 0}, "
          f"deg>16k in them: {(R[m, 7] > 16384).sum()}, entries max {R[m, 8].max() if m.any() else 0}")
