"""Host-copy options for a 16.7M-entry device assignment (flatten)."""
import time
import numpy as np
import torch

n = 1 << 24
d = torch.randint(0, 1 << 20, (n,), dtype=torch.int32, device="cuda")
torch.cuda.synchronize()


def t(name, f):
    for rep in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        f()
        torch.cuda.synchronize()
        print(f"{name} rep{rep}: {(time.perf_counter() - t0) * 1e3:.1f} ms")


t("i32 pageable + astype", lambda: d.cpu().numpy().astype(np.int64))
t("i64 pageable", lambda: d.to(torch.int64).cpu().numpy())


def pinned():
    h = torch.empty(n, dtype=torch.int64, pin_memory=True)
    h.copy_(d.to(torch.int64))
    return h.numpy()


t("i64 pinned (alloc each)", pinned)


def np_pinned():
    a = np.empty(n, dtype=np.int64)
    torch.from_numpy(a).copy_(d.to(torch.int64))
    return a


t("i64 into numpy (pageable copy_)", np_pinned)
