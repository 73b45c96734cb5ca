"""Kernel breakdown of one colouring (CUPTI): per kernel count / total time,
GPU busy vs span.   python tools/color_timeline.py [config]"""
import collections
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import paper_1410_1237_b200 as pl  # noqa: E402
from paper_1410_1237_b200 import synthetic as syn  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c4_chung_lu"
g = pl.vf_compact(syn.config_graph(cfg)).graph
pl.color_graph(g)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    col = pl.color_graph(g)
    torch.cuda.synchronize()
ev = sorted((e.time_range.start, e.time_range.end, e.name) for e in prof.events()
            if e.device_type.name == "CUDA")
agg = collections.defaultdict(lambda: [0, 0.0])
for s_, e_, n_ in ev:
    k = n_.split("(")[0].replace("void ", "")[:60]
    agg[k][0] += 1
    agg[k][1] += e_ - s_
span = ev[-1][1] - ev[0][0]
print(f"{cfg}: n={g.num_vertices} colours={col.num_colors} rounds={col.rounds if hasattr(col, 'rounds') else '?'} "
      f"span {span / 1e3:.1f} ms, busy {sum(v[1] for v in agg.values()) / 1e3:.1f} ms")
for k, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:20]:
    print(f"  {k:60s} {c:6d} {t / 1e3:9.2f} ms {t / c:8.2f} us")
