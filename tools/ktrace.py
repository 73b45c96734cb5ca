"""Per-block timeline of the hub-tier kernels over one warm coloured
iteration (plv_debug_trace: thread 0 of every block records globaltimer
stamps).  Kernel ids: 1 hub_accum (begin, loads done, atomics done, end),
2 hub_pass1, 3 hub_pass2, 4 hub_decide (begin, end)."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1410_1237_b200 as pl  # noqa: E402
from paper_1410_1237_b200 import _lib  # noqa: E402
from paper_1410_1237_b200 import synthetic as syn  # noqa: E402
from paper_1410_1237_b200.engine import PhaseEngine  # noqa: E402

mode = sys.argv[1] if len(sys.argv) > 1 else "colored"
cfg = sys.argv[2] if len(sys.argv) > 2 else "c2_rmat20"
g = pl.vf_compact(syn.config_graph(cfg)).graph
col = pl.color_graph(g) if mode == "colored" else None
s0 = pl.singleton_state(g)
d0 = s0.device()
st = {k: (t.clone() if t is not None else None) for k, t in d0.items()}
state = pl.CommunityState.from_device(st["assignment"], st["a_tot"], st["w_internal"], st["sizes"])
eng = PhaseEngine(g, state, col)
_lib.lib()
cl = ctypes.CDLL(_lib.LIB_PATH)
cl.plv_debug_trace_read.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.POINTER(ctypes.c_int64)]


def reset():
    for k in ("assignment", "a_tot", "w_internal", "sizes"):
        st[k].copy_(d0[k])


reset()
eng.iterate()
reset()
torch.cuda.synchronize()
cl.plv_debug_trace(int(os.environ.get("KTRACE_ON", "1")))  # 2: the ahead pass only
eng.iterate()
torch.cuda.synchronize()
buf = np.zeros(8 << 18, dtype=np.uint64)  # (records beyond 2^18 are dropped)
n = ctypes.c_int64(0)
cl.plv_debug_trace_read(buf.ctypes.data, 1 << 18, ctypes.byref(n))
cl.plv_debug_trace(0)
r = buf[: 8 * n.value].reshape(-1, 8).astype(np.int64)
kid = r[:, 0] >> 32
names = {1: "hub_accum", 2: "hub_pass", 5: "t2b_wide", 6: "t2a_wide", 7: "t2_narrow",
         8: "ah_pass", 9: "ah_pass_dec"}  # ah_pass: begin, wait, gains, best, ticket, end
print(f"records {len(r)}")
for k, nm in names.items():
    m = kid == k
    if not m.any():
        continue
    t = r[m, 1:7]
    ns = r[m, 7].clip(1, 6)
    nmk = int(ns.max())
    full = ns == nmk  # blocks that recorded every mark (others took a shorter path)
    segs = [np.mean(t[full, i + 1] - t[full, i]) / 1e3 for i in range(nmk - 1)]
    last = t[np.arange(len(t)), ns - 1]
    print(f"{nm:11s} blocks {m.sum():6d} ({full.sum()} with all {nmk} marks)  mean per-block "
          f"segments (us): " + " / ".join(f"{x:.2f}" for x in segs) +
          f"   total {np.mean(last - t[:, 0]) / 1e3:.2f}")
# per launch (records of one kernel id clustered by time): start spread and span
for k, nm in names.items():
    m = kid == k
    if not m.any():
        continue
    t0 = r[m, 1]
    ns = r[m, 7]
    tend = r[m, :][np.arange(m.sum()), ns.clip(1, 6)]
    o = np.argsort(t0)
    t0, tend = t0[o], tend[o]
    cuts = np.where(np.diff(t0) > 3000)[0] + 1  # a new launch after a 3 us gap in starts
    starts = np.split(t0, cuts)
    ends = np.split(tend, cuts)
    spread = np.array([s.max() - s.min() for s in starts]) / 1e3
    span = np.array([e.max() - s.min() for s, e in zip(starts, ends)]) / 1e3
    blk = np.array([len(s) for s in starts])
    print(f"{nm:11s} launches ~{len(starts):4d}  blocks/launch {blk.mean():7.1f}  "
          f"start spread {spread.mean():5.2f} us  span {span.mean():5.2f} us (median {np.median(span):5.2f})")
