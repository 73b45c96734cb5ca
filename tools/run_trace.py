"""Time a full run() on a BASELINE config and print the per-stage trace summary.

    python tools/run_trace.py c2_rmat20 [--scale 20] [--cutoff 100000]
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1410_1237_b200 as pl  # noqa: E402
from paper_1410_1237_b200 import synthetic as syn  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("config", default="c2_rmat20", nargs="?")
p.add_argument("--cutoff", type=int, default=100_000)
p.add_argument("--max-iters", type=int, default=10_000)
p.add_argument("--repeat", type=int, default=2)
a, extra = p.parse_known_args()
kw = {}
for item in extra:
    k, v = item.lstrip("-").split("=")
    kw[k] = type(syn.CONFIGS[a.config][2].get(k, 0))(v)
for rep in range(a.repeat):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    g = syn.config_graph(a.config, **kw)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    trace = []
    h = pl.run(g, pl.RunConfig(color_cutoff=a.cutoff, max_iterations_per_phase=a.max_iters),
               trace)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    by = {}
    for r in trace:
        by.setdefault(r.stage, 0.0)
        by[r.stage] += r.millis
    its = [p_.stats.iterations for p_ in h.phases]
    print(f"rep {rep}: n={g.num_vertices} M={g.num_edges} build={t1 - t0:.3f}s run={t2 - t1:.3f}s "
          f"Q={h.final_modularity!r} communities={h.num_communities} iterations={its} "
          f"stages_ms={ {k: round(v, 1) for k, v in by.items()} }", flush=True)
    per = {}
    for r in trace:
        key = (r.phase, r.stage)
        c, ms = per.get(key, (0, 0.0))
        per[key] = (c + 1, ms + r.millis)
    if rep == a.repeat - 1:
        print("   phase graph sizes (n per phase input):", [len(p_.assignment) for p_ in h.phases], flush=True)
        for (ph, stg), (c, ms) in sorted(per.items()):
            print(f"   phase {ph} {stg:10s} n={c:6d} ms={ms:10.1f}", flush=True)
