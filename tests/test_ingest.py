"""GPU: ingest on the device (plv_parse_edge_list) against
the REFERENCE itself (ref_parlouvain.load_graph from oracle/_ref, PL/graph.py:
245-478) -- identical CSR (records in file order, so duplicate merges fold in
the same order), and the same exceptions and messages whenever the device
hands the file to the host rules."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

pl = pytest.importorskip("paper_1410_1237_b200")

from paper_1410_1237_b200 import graph as G  # noqa: E402
from paper_1410_1237_b200.errors import EdgelessGraphError, GraphParseError  # noqa: E402


_REF = None


def _host(path):
    """The reference's load_graph (the checker), its exceptions mapped onto
    this package's classes of the same names."""
    global _REF
    if _REF is None:
        import conftest
        _REF = conftest.reference_module()
        if _REF is None:
            pytest.skip("reference build (oracle/_ref) not present")
    try:
        return _REF.load_graph(path)
    except (_REF.GraphParseError, _REF.EdgelessGraphError) as e:
        cls = GraphParseError if isinstance(e, _REF.GraphParseError) else EdgelessGraphError
        raise cls(str(e)) from None


def _same(g, h):
    assert g.num_vertices == h.num_vertices
    assert np.array_equal(g.adjacency_offsets, h.adjacency_offsets)
    assert np.array_equal(g.neighbors, h.neighbors)
    assert np.array_equal(g.weights, h.weights)
    assert np.array_equal(g.self_loop_weights, h.self_loop_weights)
    assert np.array_equal(g.weighted_degrees, h.weighted_degrees)
    assert g.total_weight == h.total_weight
    assert g.merged_duplicates == h.merged_duplicates


def _write(tmp_path, text, name="g.txt", mode="w"):
    p = tmp_path / name
    if mode == "wb":
        p.write_bytes(text)
    else:
        p.write_text(text)
    return str(p)


DEVICE_OK = [
    "0 1\n1 2\n2 0\n",
    "# comment\n\n0 1 2.5\n1 2 0.1\n  2 3\t1e-3 \n3 0 +3.25\n0 2 .5\n1 3 5.\n2 2 1.5E2\n",
    "0 1 1\r\n1 2 2\r\n2 3 3\r\n3 0 4",           # CRLF, no final newline
    "0 1 0.25\n0 1 0.5\n1 0 0.125\n2 1 7\n",      # duplicates in both directions
    "0\t1\t3\n 1   2   4\n\n#x\n   # y\n2 0 1000000\n",
]


@pytest.mark.parametrize("text", DEVICE_OK)
def test_device_parse_matches_host(tmp_path, text):
    path = _write(tmp_path, text)
    assert G._load_edge_list_device(path) is not None  # the device took it
    _same(pl.load_graph(path), _host(path))


HOST_ONLY = [
    "0 1 0.30000000000000004\n1 2 1\n",           # 17 significant digits
    "5 7 1\n7 9 2\n9 5 3\n",                      # ids not 0..n-1: renumbered
    "0 1 1_0\n1 2 1\n",                           # Python float() accepts underscores
    "0 1 1e400\n",                                # inf
    "0 1\r1 2\n",                                 # a lone CR ends a line for Python
]


@pytest.mark.parametrize("text", HOST_ONLY)
def test_host_rules_take_over(tmp_path, text):
    path = _write(tmp_path, text)
    assert G._load_edge_list_device(path) is None
    try:
        want = _host(path)
    except Exception as e:  # the reference's error, raised by load_graph too
        with pytest.raises(type(e)) as got:
            pl.load_graph(path)
        assert str(got.value) == str(e)
        return
    _same(pl.load_graph(path), want)


ERRORS = [
    ("0 1\n1 2 3 4\n", GraphParseError),
    ("0 1\n1 x\n", GraphParseError),
    ("0 1 -2\n", GraphParseError),
    ("0 1 0\n", GraphParseError),
    ("0 1 abc\n", GraphParseError),
    ("# only a comment\n\n", EdgelessGraphError),
    ("", EdgelessGraphError),
]


@pytest.mark.parametrize("text,exc", ERRORS)
def test_errors_match_host(tmp_path, text, exc):
    path = _write(tmp_path, text)
    with pytest.raises(exc) as want:
        _host(path)
    with pytest.raises(exc) as got:
        pl.load_graph(path)
    assert str(got.value) == str(want.value)


def test_large_file(tmp_path):
    rng = np.random.default_rng(1)
    n = 50_000
    u = rng.integers(0, n, 400_000)
    v = rng.integers(0, n, 400_000)
    u[:n] = np.arange(n)  # every id appears: dense
    w = np.round(rng.uniform(0.5, 9.5, len(u)), 3)
    lines = [f"{a} {b} {x:.3f}\n" for a, b, x in zip(u.tolist(), v.tolist(), w.tolist())]
    lines.insert(1000, "# a comment in the middle\n")
    path = _write(tmp_path, "".join(lines))
    assert G._load_edge_list_device(path) is not None
    _same(pl.load_graph(path), _host(path))
