"""One phase-1 local-move iteration of a BASELINE config between
cudaProfilerStart/Stop, for `ncu --profile-from-start off`.

    ncu --profile-from-start off --metrics ... python tools/profile_iter.py [--mode colored]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1410_1237_b200 as pl  # noqa: E402
from paper_1410_1237_b200 import synthetic as syn  # noqa: E402
from paper_1410_1237_b200.engine import PhaseEngine  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--config", default="c2_rmat20")
p.add_argument("--mode", choices=["colored", "uncolored"], default="colored")
p.add_argument("--iters", type=int, default=1)
a = p.parse_args()
g = pl.vf_compact(syn.config_graph(a.config)).graph
col = pl.color_graph(g) if a.mode == "colored" else None
s0 = pl.singleton_state(g)
d0 = s0.device()
st = {k: (t.clone() if t is not None else None) for k, t in d0.items()}
state = pl.CommunityState.from_device(st["assignment"], st["a_tot"], st["w_internal"], st["sizes"])
eng = PhaseEngine(g, state, col)


def reset():
    for k in ("assignment", "a_tot", "w_internal", "sizes"):
        st[k].copy_(d0[k])


reset()
eng.iterate()  # warm-up (graph upload, caches)
reset()
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
for _ in range(a.iters):
    q, moves, cand = eng.iterate()
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print(f"n={g.num_vertices} nnz={g.nnz} M={g.num_edges} moves={moves} cand={cand} q={q!r}")
