"""Kernel breakdown (CUPTI) of the k-th colouring inside run().
   python tools/color_timeline_k.py config k"""
import collections
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import paper_1410_1237_b200 as pl  # noqa: E402
from paper_1410_1237_b200 import engine, heuristics  # noqa: E402
from paper_1410_1237_b200 import synthetic as syn  # noqa: E402

cfg, want = sys.argv[1], int(sys.argv[2])
orig = heuristics.color_graph
calls = [0]


def wrapped(g, *a, **k):
    calls[0] += 1
    if calls[0] != want:
        return orig(g, *a, **k)
    orig(g, *a, **k)
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        c = orig(g, *a, **k)
        torch.cuda.synchronize()
    ev = sorted((e.time_range.start, e.time_range.end, e.name) for e in prof.events()
                if e.device_type.name == "CUDA")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for s_, e_, n_ in ev:
        kk = n_.split("(")[0].replace("void ", "")[:60]
        agg[kk][0] += 1
        agg[kk][1] += e_ - s_
    span = ev[-1][1] - ev[0][0]
    print(f"{cfg} colouring {want}: n={g.num_vertices} nnz={g.nnz} colours={c.num_colors} "
          f"rounds={c.rounds} span {span / 1e3:.1f} ms")
    for kk, (cn, t) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:14]:
        print(f"  {kk:60s} {cn:6d} {t / 1e3:9.2f} ms {t / cn:8.2f} us")
    return c


heuristics.color_graph = wrapped
engine.color_graph = wrapped
pl.run(syn.config_graph(cfg))
