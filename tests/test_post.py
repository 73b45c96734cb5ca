"""GPU: device post-processing against the REFERENCE
itself (ref_parlouvain from oracle/_ref): the assignment file written by its
write_assignment (PL/engine.py:318-322) byte for byte, and its
compare_partitions (PL/evaluation.py:68-86) field for field."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

pl = pytest.importorskip("paper_1410_1237_b200")

from paper_1410_1237_b200 import evaluation as ev  # noqa: E402


def _ref():
    import conftest
    r = conftest.reference_module()
    if r is None:
        pytest.skip("reference build (oracle/_ref) not present")
    return r


def _host_text(a):
    import os
    import tempfile
    fd, path = tempfile.mkstemp()
    os.close(fd)
    try:
        _ref().write_assignment(path, np.asarray(a))
        with open(path, "rb") as fh:
            return fh.read()
    finally:
        os.unlink(path)


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
    return _ref().compare_partitions(s, p)


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
    want = _host_counts(s, p)
    for f in ("tp", "fp", "fn", "tn", "sp", "se", "oq", "rand"):
        assert getattr(got, f) == getattr(want, f), f
    assert got.csv_line() == want.csv_line()
