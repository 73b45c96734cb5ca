"""Kernel timeline of one warm phase-1 iteration (CUPTI through
torch.profiler; graph-launched kernels included).  Prints the per-kernel
in-graph time split and the gaps between consecutive kernels.

    python tools/timeline.py [--mode colored|uncolored] [--config c2_rmat20]
"""
import argparse
import collections
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import paper_1410_1237_b200 as pl  # noqa: E402
from paper_1410_1237_b200 import synthetic as syn  # noqa: E402
from paper_1410_1237_b200.engine import PhaseEngine  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--mode", default="colored")
ap.add_argument("--config", default="c2_rmat20")
ap.add_argument("--dump", default="")
a = ap.parse_args()
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
eng.iterate()
reset()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    q, moves, cand = eng.iterate()
    torch.cuda.synchronize()
ev = []
for e in prof.events():
    if e.device_type.name != "CUDA":
        continue
    ev.append((e.time_range.start, e.time_range.end, e.name))
ev.sort()
ks = [x for x in ev if "Memcpy" not in x[2] and "Memset" not in x[2]]
t0, t1 = ev[0][0], max(x[1] for x in ev)
print(f"events {len(ev)} kernels {len(ks)} span {(t1 - t0) / 1e3:.3f} ms  moves {moves} q {q!r}")
agg = collections.defaultdict(lambda: [0, 0.0])
for s, e, n in ks:
    k = n.split("(")[0].replace("void ", "")[:48]
    agg[k][0] += 1
    agg[k][1] += (e - s)
busy = 0.0
cur_s, cur_e = None, None
for s, e, n in ks:  # union of kernel intervals
    if cur_e is None or s > cur_e:
        if cur_e is not None:
            busy += cur_e - cur_s
        cur_s, cur_e = s, e
    else:
        cur_e = max(cur_e, e)
busy += cur_e - cur_s
print(f"GPU busy (union of kernel intervals) {busy / 1e3:.3f} ms; idle {(t1 - t0 - busy) / 1e3:.3f} ms")
print(f"{'kernel':48s} {'n':>5s} {'sum_ms':>8s} {'mean_us':>8s}")
for k, (n, tt) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:20]:
    print(f"{k:48s} {n:5d} {tt / 1e3:8.3f} {tt / n:8.2f}")
if a.dump:
    with open(a.dump, "w") as fh:
        for s, e, n in ev:
            fh.write(f"{s - t0:.3f}\t{e - t0:.3f}\t{n.split('(')[0]}\n")
