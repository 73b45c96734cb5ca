"""GPU: device post-processing against the host
restatements of the reference: the assignment file (PL/engine.py:318-322)
byte for byte, and compare_partitions' pair counts (PL/evaluation.py:68-86)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

pl = pytest.importorskip("paper_1410_1237_b200")

from paper_1410_1237_b200 import evaluation as ev  # noqa: E402


def _host_text(a):
    return "".join(f"{v} {c}\n" for v, c in enumerate(np.asarray(a).tolist())).encode()


@pytest.mark.parametrize("dtype", ["int32", "int64"])
def test_assignment_file_bytes(tmp_path, dtype):
    import torch
    rng = np.random.default_rng(2)
    a = rng.integers(0, 10 ** 6, 250_000).astype(dtype)
    a[:5] = [0, 9, 10, 99, 100]
    p = tmp_path / "a.txt"
    pl.write_assignment(str(p), a)                                  # large host array
    assert p.read_bytes() == _host_text(a)
    pl.write_assignment(str(p), torch.from_numpy(a).cuda())        # device tensor
    assert p.read_bytes() == _host_text(a)


def test_assignment_file_from_run(tmp_path):
    from paper_1410_1237_b200 import synthetic as syn
    u, v, w = syn.rmat_records(12, 8, seed=4)
    h = pl.run(pl.Graph.from_edges(u, v, w, num_vertices=1 << 12))
    p = tmp_path / "c.txt"
    pl.write_assignment(str(p), h.flatten_device())
    assert p.read_bytes() == _host_text(h.final_assignment)


def _host_counts(s, p):
    n = len(s)
    _, si = np.unique(s, return_inverse=True)
    _, pi = np.unique(p, return_inverse=True)
    cells = np.bincount(si.astype(np.int64) * (int(pi.max()) + 1) + pi.astype(np.int64))
    tp = ev._pairs(cells)
    fn = ev._pairs(np.bincount(si)) - tp
    fp = ev._pairs(np.bincount(pi)) - tp
    return ev._counts(tp, fp, fn, n * (n - 1) // 2 - tp - fp - fn)


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_pair_counts_match_host(seed):
    rng = np.random.default_rng(seed)
    n = 300_000
    s = rng.integers(-50, 400, n)
    p = rng.integers(0, 3000, n) * (10 ** 12) - 5
    if seed == 2:
        p = s.copy()                          # identical partitions
        s[::7] = 10 ** 15
    got = ev.compare_partitions(s, p)
    assert ev._device_pair_counts(np.asarray(s), np.asarray(p)) is not None
    assert got == _host_counts(s, p)
    assert got.csv_line() == _host_counts(s, p).csv_line()
