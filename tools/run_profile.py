"""Wall-clock breakdown of run() by host call (synchronised): vf, colouring,
phase-engine creation, the phase loop, rebuild, flatten.

    python tools/run_profile.py [config] [--bench-like]
"""
import collections
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1410_1237_b200 as pl  # noqa: E402
from paper_1410_1237_b200 import engine, synthetic as syn  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 and not sys.argv[1].startswith("--") else "c2_rmat20"
acc = collections.defaultdict(lambda: [0, 0.0])


def timed(name, fn):
    def w(*a, **k):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = fn(*a, **k)
        torch.cuda.synchronize()
        acc[name][0] += 1
        acc[name][1] += time.perf_counter() - t0
        return r
    return w


engine.vf_compact = timed("vf_compact", engine.vf_compact)
engine.color_graph = timed("color_graph", engine.color_graph)
engine.rebuild_device = timed("rebuild_device", engine.rebuild_device)
engine.PhaseEngine.__init__ = timed("PhaseEngine.__init__", engine.PhaseEngine.__init__)
engine.PhaseEngine.run = timed("PhaseEngine.run", engine.PhaseEngine.run)
engine.PhaseEngine.close = timed("PhaseEngine.close", engine.PhaseEngine.close)
engine.Hierarchy.flatten = timed("Hierarchy.flatten", engine.Hierarchy.flatten)
engine.singleton_state = timed("singleton_state", engine.singleton_state)
from paper_1410_1237_b200 import graph as _graph  # noqa: E402
_fs = _graph.Graph.from_sorted_device_records.__func__
_graph.Graph.from_sorted_device_records = classmethod(
    lambda cls, *a, **k: timed("  from_sorted_records", _fs)(cls, *a, **k))
_fd = _graph.Graph.from_device_records.__func__
_graph.Graph.from_device_records = classmethod(
    lambda cls, *a, **k: timed("  from_device_records", _fd)(cls, *a, **k))
engine.modularity_device = timed("modularity_device", engine.modularity_device)
if "--bench-like" in sys.argv:
    g0 = syn.config_graph(cfg)
    g = pl.vf_compact(g0).graph
    col = pl.color_graph(g)
    s = pl.singleton_state(g)
    e = engine.PhaseEngine(g, s, col)
    for _ in range(5):
        e.iterate()
    acc.clear()
for rep in range(3):
    acc.clear()
    g = syn.config_graph(cfg)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    h = pl.run(g, pl.RunConfig(color_cutoff=0 if cfg == "c1_sbm" else 100_000))
    torch.cuda.synchronize()
    tot = time.perf_counter() - t0
    print(f"rep {rep}: run {tot * 1e3:.1f} ms, Q={h.final_modularity!r}")
    for k, (n, t) in sorted(acc.items(), key=lambda kv: -kv[1][1]):
        print(f"   {k:24s} {n:3d} {t * 1e3:9.1f} ms")
