"""GPU: METIS and Matrix Market ingest on the device (plv_parse_metis,
plv_parse_mm) against the REFERENCE's load_graph
(ref_parlouvain from oracle/_ref, PL/graph.py:326-478): identical graphs when
the device takes the file, and -- for files only the host rules may judge
(duplicates to merge, tolerated asymmetric weights, malformed lines) -- the
reference's result or its exception and message."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

pl = pytest.importorskip("paper_1410_1237_b200")

from paper_1410_1237_b200 import graph as G  # noqa: E402
from paper_1410_1237_b200.errors import EdgelessGraphError, GraphParseError  # noqa: E402


def _ref():
    import conftest
    r = conftest.reference_module()
    if r is None:
        pytest.skip("reference build (oracle/_ref) not present")
    return r


def _ref_load(path):
    r = _ref()
    try:
        return r.load_graph(path)
    except (r.GraphParseError, r.EdgelessGraphError) as e:
        cls = GraphParseError if isinstance(e, r.GraphParseError) else EdgelessGraphError
        raise cls(str(e)) from None


def _same(g, h):
    assert g.num_vertices == h.num_vertices
    assert np.array_equal(g.adjacency_offsets, h.adjacency_offsets)
    assert np.array_equal(g.neighbors, h.neighbors)
    assert np.array_equal(g.weights, h.weights)
    assert np.array_equal(g.self_loop_weights, h.self_loop_weights)
    assert np.array_equal(g.weighted_degrees, h.weighted_degrees)
    assert g.total_weight == h.total_weight


def _graph(seed, n=400, m=1500, weighted=True, loops=True):
    rng = np.random.default_rng(seed)
    u = rng.integers(0, n, m)
    v = rng.integers(0, n, m)
    if not loops:
        v = np.where(u == v, (v + 1) % n, v)
    key = np.unique(np.minimum(u, v) * n + np.maximum(u, v))
    a, b = key // n, key % n
    w = (np.round(rng.uniform(0.5, 9.5, len(a)), 2) if weighted else np.ones(len(a)))
    return n, a, b, w


def _metis_text(n, a, b, w, weighted, comments=False, crlf=False):
    adj = [[] for _ in range(n)]
    for x, y, z in zip(a.tolist(), b.tolist(), w.tolist()):
        adj[x].append((y, z))
        if x != y:
            adj[y].append((x, z))
    nl = "\r\n" if crlf else "\n"
    out = ["% a comment" + nl] if comments else []
    out.append(f"{n} {len(a)}{' 1' if weighted else ''}{nl}")
    for i in range(n):
        if comments and i == n // 2:
            out.append("   % mid comment" + nl)
        out.append(" ".join(f"{y + 1} {z!r}" if weighted else f"{y + 1}" for y, z in adj[i]) + nl)
    return "".join(out)


def _mm_text(n, a, b, w, field="real", comments=False):
    out = [f"%%MatrixMarket matrix coordinate {field} symmetric\n"]
    if comments:
        out.append("% generated\n%\n")
    out.append(f"{n} {n} {len(a)}\n")
    for x, y, z in zip(a.tolist(), b.tolist(), w.tolist()):
        if comments and x % 97 == 0:
            out.append("% row\n")
        if field == "pattern":
            out.append(f"{y + 1} {x + 1}\n")
        elif field == "integer":
            out.append(f"{x + 1} {y + 1} {int(z * 100)}\n")
        else:
            out.append(f"{x + 1} {y + 1} {z!r}\n")
    return "".join(out)


@pytest.mark.parametrize("weighted,comments,crlf", [(True, False, False), (False, True, False),
                                                    (True, True, True)])
def test_metis_device(tmp_path, weighted, comments, crlf):
    n, a, b, w = _graph(1, weighted=weighted)
    n += 3  # trailing isolated vertices: blank adjacency lines
    p = tmp_path / "g.metis"
    p.write_bytes(_metis_text(n, a, b, w, weighted, comments, crlf).encode())
    assert G._load_metis_device(str(p)) is not None
    _same(pl.load_graph(str(p)), _ref_load(str(p)))


@pytest.mark.parametrize("field,comments", [("real", False), ("pattern", True),
                                            ("integer", True)])
def test_mm_device(tmp_path, field, comments):
    n, a, b, w = _graph(2, weighted=field != "pattern")
    p = tmp_path / "g.mtx"
    p.write_text(_mm_text(n, a, b, w, field, comments))
    assert G._load_mm_device(str(p)) is not None
    _same(pl.load_graph(str(p)), _ref_load(str(p)))


def test_metis_large(tmp_path):
    n, a, b, w = _graph(3, n=60_000, m=500_000)
    p = tmp_path / "big.graph"
    p.write_text(_metis_text(n, a, b, w, True))
    assert G._load_metis_device(str(p)) is not None
    _same(pl.load_graph(str(p)), _ref_load(str(p)))


HOST_METIS = [
    "3 2\n2 2\n1 1 3\n2\n",               # duplicate neighbour: merged with a warning
    "2 1 1\n2 1.0\n1 1.0000000000001\n",  # asymmetric within tolerance: accepted
    "3 2\n2\n1 3\n\n",                    # 2-3 listed one way: error
    "3 3\n2\n1 3\n2\n",                   # declared edge count wrong: error
    "2 1\n2\n1\n3\n",                     # more adjacency lines than vertices
    "3 1\n2\n1\n",                        # fewer adjacency lines
    "2 1\n2\n1 x\n",                      # bad token
    "2 1 11\n2\n1\n",                     # vertex weights
    "2 1 1\n2 1\n1\n",                    # odd weighted token count
    "2 1\n3\n1\n",                        # neighbour out of range
]


@pytest.mark.parametrize("text", HOST_METIS)
def test_metis_host_rules(tmp_path, text):
    p = tmp_path / "h.metis"
    p.write_text(text)
    assert G._load_metis_device(str(p)) is None
    try:
        want = _ref_load(str(p))
    except Exception as e:
        with pytest.raises(type(e)) as got:
            pl.load_graph(str(p))
        assert str(got.value) == str(e)
        return
    _same(pl.load_graph(str(p)), want)


HOST_MM = [
    "%%MatrixMarket matrix coordinate real symmetric\n3 3 2\n1 2 1.5\n",       # count mismatch
    "%%MatrixMarket matrix coordinate real symmetric\n3 3 1\n1 4 1.5\n",       # out of range
    "%%MatrixMarket matrix coordinate real general\n3 3 1\n1 2 1.5\n",         # unsupported
    "%%MatrixMarket matrix coordinate pattern symmetric\n3 3 1\n1 2 3\n",      # extra token
    "%%MatrixMarket matrix coordinate real symmetric\n3 3 1\n1 2 -1\n",        # bad weight
    "%%MatrixMarket matrix coordinate real symmetric\n%c\n",                   # no size line
]


@pytest.mark.parametrize("text", HOST_MM)
def test_mm_host_rules(tmp_path, text):
    p = tmp_path / "h.mtx"
    p.write_text(text)
    assert G._load_mm_device(str(p)) is None
    try:
        want = _ref_load(str(p))
    except Exception as e:
        with pytest.raises(type(e)) as got:
            pl.load_graph(str(p))
        assert str(got.value) == str(e)
        return
    _same(pl.load_graph(str(p)), want)
