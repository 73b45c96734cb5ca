"""Kernel timeline of iterations inside a capped (oscillating) phase.

Runs run() on a BASELINE config, keeps the input graph of phase P, then
iterates it from the singleton state (--warm iterations), and profiles
--iters more with CUPTI: per-kernel in-graph time, GPU busy vs span, and the
host wall time per iteration.

    python tools/capped_timeline.py c3_grid --phase 4
"""
import argparse
import collections
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import paper_1410_1237_b200 as pl  # noqa: E402
from paper_1410_1237_b200 import engine, synthetic as syn  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("config")
ap.add_argument("--phase", type=int, default=4)
ap.add_argument("--warm", type=int, default=200)
ap.add_argument("--iters", type=int, default=5)
a = ap.parse_args()

grabbed = {}
orig = engine.run_phase


def hook(g, cfg, coloring=None, trace=None, phase_index=1):
    if phase_index == a.phase:
        grabbed["g"] = g
        grabbed["col"] = coloring
        raise StopIteration
    return orig(g, cfg, coloring, trace, phase_index)


engine.run_phase = hook
try:
    pl.run(syn.config_graph(a.config), pl.RunConfig())
except StopIteration:
    pass
engine.run_phase = orig
g, col = grabbed["g"], grabbed["col"]
print(f"phase {a.phase}: n={g.num_vertices} nnz={g.nnz} M={g.num_edges} coloured={col is not None} "
      f"integral={g.integral} max_degree={g.max_degree}")
s = pl.singleton_state(g)
eng = engine.PhaseEngine(g, s, col)
mv = []
for _ in range(a.warm):
    mv.append(eng.iterate()[1])
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(100):
    eng.iterate()
t1 = time.perf_counter()
print(f"host wall per iteration {(t1 - t0) * 1e4:.1f} us; moves last warm iters {mv[-6:]}")
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(a.iters):
        eng.iterate()
    torch.cuda.synchronize()
ev = sorted((e.time_range.start, e.time_range.end, e.name) for e in prof.events()
            if e.device_type.name == "CUDA")
ks = [x for x in ev if "Memcpy" not in x[2] and "Memset" not in x[2]]
span = (max(x[1] for x in ev) - ev[0][0]) / a.iters
agg = collections.defaultdict(lambda: [0, 0.0])
for s_, e_, n_ in ks:
    k = n_.split("(")[0].replace("void ", "")[:56]
    agg[k][0] += 1
    agg[k][1] += (e_ - s_)
busy = 0.0
cs, ce = None, None
for s_, e_, n_ in ev:
    if ce is None or s_ > ce:
        if ce is not None:
            busy += ce - cs
        cs, ce = s_, e_
    else:
        ce = max(ce, e_)
busy += ce - cs
print(f"per iteration: events {len(ev) / a.iters:.0f} span {span:.1f} us busy {busy / a.iters:.1f} us")
for k, (n_, tt) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:25]:
    print(f"  {k:56s} {n_ / a.iters:5.1f}/it {tt / a.iters:8.2f} us/it")
