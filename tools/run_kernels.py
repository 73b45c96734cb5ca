"""Kernel-time breakdown (CUPTI via torch.profiler) of a warm full run() on a
BASELINE config, graph generation and CSR build included.

    python tools/run_kernels.py c4_chung_lu [top]
"""
import collections
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import paper_1410_1237_b200 as pl  # noqa: E402
from paper_1410_1237_b200 import synthetic as syn  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c4_chung_lu"
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25


def once():
    g = syn.config_graph(cfg)
    return pl.run(g, pl.RunConfig(color_cutoff=0 if cfg == "c1_sbm" else 100_000))


once()
torch.cuda.synchronize()
t0 = time.perf_counter()
with profile(activities=[ProfilerActivity.CUDA], acc_events=True) as prof:
    h = once()
    torch.cuda.synchronize()
wall = time.perf_counter() - t0
agg = collections.defaultdict(lambda: [0, 0.0])
for e in prof.events():
    if e.device_type.name != "CUDA":
        continue
    k = e.name.split("(")[0].replace("void ", "")[:60]
    agg[k][0] += 1
    agg[k][1] += e.time_range.end - e.time_range.start
tot = sum(v[1] for v in agg.values())
print(f"{cfg}: run() wall {wall * 1e3:.1f} ms under CUPTI; kernel+copy time {tot / 1e3:.1f} ms; "
      f"Q={h.final_modularity!r}")
for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:top]:
    print(f"  {t / 1e3:9.2f} ms {100 * t / tot:5.1f}% {n:7d}  {k}")
