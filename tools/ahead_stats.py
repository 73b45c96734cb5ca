"""The ahead tables a phase-1 coloured plan of a config uses (plv_phase_ahead_stats).

    python tools/ahead_stats.py c4_chung_lu
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import paper_1410_1237_b200 as pl  # noqa: E402
from paper_1410_1237_b200 import synthetic as syn  # noqa: E402
from paper_1410_1237_b200.engine import PhaseEngine  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c4_chung_lu"
g = pl.vf_compact(syn.config_graph(cfg)).graph
col = pl.color_graph(g)
s = pl.singleton_state(g)
d = s.device()
state = pl.CommunityState.from_device(d["assignment"], d["a_tot"], d["w_internal"], d["sizes"])
eng = PhaseEngine(g, state, col)
st = eng.ahead_stats()
deg = np.diff(g.adjacency_offsets)
classes = col.classes()
print(f"{cfg}: n={g.num_vertices} nnz={g.nnz} colours={col.num_colors} integral={g.integral if hasattr(g, 'integral') else '?'}")
print("ahead:", st)
if st["stages"]:
    first = len(classes) - st["stages"]
    ent = sum(int(deg[c].sum()) for c in classes[first:])
    print(f"(if the ahead stages are the last {st['stages']}: stages {first}..{len(classes) - 1}, "
          f"{ent} row entries; table bytes {16 * st['slots']}, fix list bytes {16 * st['fix_entries']})")
eng.close()
