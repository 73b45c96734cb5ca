"""Time the device modularity (plv_modularity) at several n (CUDA events)."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1410_1237_b200 import _lib  # noqa: E402

L = _lib.lib()
for n in [int(x) for x in (sys.argv[1:] or ["24824", "1573370", "908790"])]:
    g = torch.Generator(device="cuda").manual_seed(0)
    w = torch.rand(n, device="cuda", dtype=torch.float64, generator=g)
    a = torch.rand(n, device="cuda", dtype=torch.float64, generator=g)
    out = torch.empty(1, device="cuda", dtype=torch.float64)
    for _ in range(3):
        _lib.check(L.modularity(_lib.ptr(w), _lib.ptr(a), n, 1000.0, _lib.ptr(out), _lib.stream()))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        _lib.check(L.modularity(_lib.ptr(w), _lib.ptr(a), n, 1000.0, _lib.ptr(out), _lib.stream()))
    e1.record()
    torch.cuda.synchronize()
    print(f"n={n}: {e0.elapsed_time(e1) / 20 * 1e3:.1f} us per call (incl. scratch alloc)")
