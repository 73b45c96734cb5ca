"""Host-side logic that needs no GPU: configuration, trace records, file
parsing, the CLI's error paths, partition metrics, the numpy generators and
the backend policy (mirrors of the reference's unit tests, PL/ tests)."""

import math

import numpy as np
import pytest

import paper_1410_1237_b200 as pl
from paper_1410_1237_b200 import cli, synthetic as syn
from paper_1410_1237_b200.engine import TraceRecord, _iteration_converged, _rel_gain
from paper_1410_1237_b200.graph import densify_ids, parse_records


def test_config_validation():
    with pytest.raises(ValueError):
        pl.RunConfig(theta_final=0.0).validate()
    with pytest.raises(ValueError):
        pl.RunConfig(theta_color=1e-7, theta_final=1e-6).validate()
    with pytest.raises(ValueError):
        pl.RunConfig(worker_count=0).validate()
    with pytest.raises(ValueError):
        pl.RunConfig(max_iterations_per_phase=0).validate()
    with pytest.raises(ValueError):
        pl.RunConfig(color_cutoff=-1).validate()
    pl.RunConfig().validate()


def test_trace_csv_row_matches_reference_format():
    r = TraceRecord(2, 3, "clustering", 0.1 + 0.2, 7, 1.23456, 1e-6)
    assert TraceRecord.CSV_HEADER == "phase,iteration,stage,modularity,moves,millis"
    assert r.csv_row() == "2,3,clustering,0.30000000000000004,7,1.235"


def test_threshold_rules():
    assert _rel_gain(0.5, 0.0) == 0.5
    assert _rel_gain(0.6, 0.5) == pytest.approx(0.2)
    assert _iteration_converged(0.5, 0.5, 1e-6)
    assert not _iteration_converged(0.6, 0.5, 1e-6)
    assert _iteration_converged(1e-16, 0.0, 1e-6)


def test_edge_list_parsing_and_densify(tmp_path):
    p = tmp_path / "g.el"
    p.write_text("# comment\n100 7\n\n7 42 2.5\n")
    u, v, w, n = parse_records(p)
    assert n == 3 and u.tolist() == [0, 1] and v.tolist() == [1, 2]
    assert w.tolist() == [1.0, 2.5]
    u, v, n = densify_ids([0, 3], [1, 2])
    assert n == 4 and u.tolist() == [0, 3]


def test_parse_errors(tmp_path):
    p = tmp_path / "g.el"
    p.write_text("0 1\nnot an edge at all here\n")
    with pytest.raises(pl.GraphParseError, match=r":2: malformed line"):
        parse_records(p)
    p.write_text("0 1 0.0\n")
    with pytest.raises(pl.GraphParseError, match="non-positive weight"):
        parse_records(p)
    p.write_text("# only comments\n")
    with pytest.raises(pl.EdgelessGraphError):
        parse_records(p)


def test_metis_and_mtx_parsing(tmp_path):
    p = tmp_path / "g.metis"
    p.write_text("% tiny weighted graph\n3 3 1\n2 1 3 4\n1 1 3 2\n1 4 2 2\n")
    u, v, w, n = parse_records(p)
    assert n == 3 and sorted(zip(u.tolist(), v.tolist(), w.tolist())) == \
        [(0, 1, 1.0), (0, 2, 4.0), (1, 2, 2.0)]
    p.write_text("3 2\n2\n1 3\n\n")
    with pytest.raises(pl.GraphParseError, match="one direction only"):
        parse_records(p)
    q = tmp_path / "g.mtx"
    q.write_text("%%MatrixMarket matrix coordinate real general\n2 2 1\n2 1 1.0\n")
    with pytest.raises(pl.GraphParseError, match="unsupported symmetry"):
        parse_records(q)
    q.write_text("%%MatrixMarket matrix coordinate pattern symmetric\n3 3 2\n1 2\n2 3\n")
    u, v, w, n = parse_records(q)
    assert n == 3 and u.tolist() == [0, 1] and w.tolist() == [1.0, 1.0]


def test_cli_error_exit_codes(tmp_path, capsys):
    assert cli.main(["detect", "--input", str(tmp_path / "nope.el")]) == 2
    bad = tmp_path / "bad.el"
    bad.write_text("0 1\nbogus line here\n")
    assert cli.main(["detect", "--input", str(bad), "--output", str(tmp_path / "o"),
                     "--trace", str(tmp_path / "t")]) == 3
    empty = tmp_path / "e.el"
    empty.write_text("# no edges\n")
    assert cli.main(["detect", "--input", str(empty)]) == 4
    err = capsys.readouterr().err
    assert "modularity undefined for edgeless graph" in err
    with pytest.raises(SystemExit):
        cli.main(["detect", "--input", "x.el", "--frobnicate"])


def test_cli_compare(tmp_path, capsys):
    ref = tmp_path / "ref.txt"
    ref.write_text("0 7\n1 7\n2 7\n3 7\n")
    cand = tmp_path / "cand.txt"
    cand.write_text("0 1\n1 1\n2 2\n3 2\n")
    assert cli.main(["compare", str(ref), str(cand)]) == 0
    assert capsys.readouterr().out.strip() == "2,0,4,0,1.0,0.333333,0.333333,0.333333"
    b = tmp_path / "b.txt"
    b.write_text("0 0\n1 0\n")
    assert cli.main(["compare", str(ref), str(b)]) == 5


def test_graph_threads_env(monkeypatch):
    monkeypatch.setenv("GRAPH_THREADS", "3")
    args = cli.build_parser().parse_args(["detect", "--input", "x.el"])
    assert cli._config_from_args(args).worker_count == 3


def test_compare_partitions_matches_bruteforce():
    rng = np.random.default_rng(42)
    for _ in range(50):
        n = int(rng.integers(2, 300))
        s = rng.integers(0, max(1, n // 3), size=n)
        p = rng.integers(0, max(1, n // 3), size=n)
        assert pl.compare_partitions(s, p) == pl.compare_partitions_bruteforce(s, p)
    r = pl.compare_partitions([0, 1, 2], [4, 4, 4])
    assert (r.tp, r.fp, r.fn, r.tn) == (0, 3, 0, 0) and r.se == 1.0 and r.sp == 0.0
    with pytest.raises(pl.PartitionMismatchError):
        pl.compare_partitions([0, 1], [0, 1, 2])


def test_backend_policy():
    assert pl.backend.name() == "cuda"
    assert pl.backend.has_compiled()
    assert pl.backend.use("compiled") == "cuda"
    assert pl.backend.use("auto") == "cuda"
    with pytest.raises(ValueError):
        pl.backend.use("python")


def test_counter_rng_is_splitmix64():
    # SplitMix64 with state 0: first output 0xE220A8397B1DCDAF
    assert syn._mix64_int(0x9E3779B97F4A7C15) == 0xE220A8397B1DCDAF
    key = syn.stream_key(7, 3)
    a = syn.rnd01(key, np.arange(5, dtype=np.uint64))
    assert np.all((a >= 0) & (a < 1))
    assert np.array_equal(a, syn.rnd01(key, np.arange(5, dtype=np.uint64)))


def test_config_generators_shapes():
    u, v, w = syn.rmat_records(10)
    assert len(u) == len(v) == len(w) and np.all(u != v)
    assert np.all((w >= 1.0) & (w < 10.0)) and u.max() < 1024
    u, v, w = syn.sbm_records(n=400, block=100)
    assert np.all(u < v) and np.all(w == 1.0)
    u, v, w = syn.grid_records(side=16, pendants=10)
    assert u.max() < 16 * 16 + 10 and np.all((w >= 0.5) & (w < 1.5))
    assert np.array_equal(u[-10:], np.arange(256, 266))
    cdf = syn.chung_lu_cdf(1 << 12, max_degree=100.0)
    assert np.all(np.diff(cdf) > 0)
    u, v, w = syn.chung_lu_records(n=1 << 12, max_degree=100.0)
    assert np.all(u != v) and u.max() < 4096


def test_gnm_matches_reference_generator(ref):
    import importlib
    rsyn = importlib.import_module(ref.__name__ + ".synthetic")
    for seed in range(4):
        u, v, w = syn.gnm_records(50, 120, seed=seed, weight_range=(0.0, 2.0))
        g = rsyn.gnm_random_graph(50, 120, seed=seed, weight_range=(0.0, 2.0))
        rg = ref.Graph.from_edges(u, v, w, num_vertices=50)
        assert rg.same_as(g)


def test_stdout_to_stderr_routes_fd1(capfd):
    """NCCL's stdout banner is diverted so bench.py's stdout is one JSON line."""
    import os
    from paper_1410_1237_b200.dist import stdout_to_stderr
    with stdout_to_stderr():
        os.write(1, b"banner\n")
    os.write(1, b"json\n")
    out, err = capfd.readouterr()
    assert out == "json\n" and "banner" in err
