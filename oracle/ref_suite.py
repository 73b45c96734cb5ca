"""Run the REFERENCE's own test suite against this package (TEST INFRASTRUCTURE).

oracle/build_ref.sh stages the reference's tests verbatim (pkg/tests, with
their data files) at oracle/_ref/ref_tests.  This runner aliases the
reference's module names to the drop-in -- `parlouvain` and every submodule
the tests import resolve to `paper_1410_1237_b200` -- and runs pytest on the
staged suite, so it exercises the CUDA package exactly as the reference's
tests exercise theirs.  Needs a B200 (the package has no CPU fallback).

    python oracle/ref_suite.py [pytest args...]

Documented deviations (tests/ref_suite_waivers.txt) are deselected by id;
every other test must pass.
"""

from __future__ import annotations

import importlib
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
SUITE = os.path.join(HERE, "_ref", "ref_tests")
WAIVERS = os.path.join(ROOT, "tests", "ref_suite_waivers.txt")
SUBMODULES = ("backend", "cli", "engine", "errors", "evaluation", "graph", "heuristics",
              "modularity", "synthetic")


def alias():
    sys.path.insert(0, ROOT)
    pkg = importlib.import_module("paper_1410_1237_b200")
    sys.modules["parlouvain"] = pkg
    for m in SUBMODULES:
        sys.modules[f"parlouvain.{m}"] = importlib.import_module(f"paper_1410_1237_b200.{m}")


def waived():
    out = []
    if os.path.exists(WAIVERS):
        for line in open(WAIVERS):
            line = line.split("#", 1)[0].strip()
            if line:
                out.append(line)
    return out


class _Waive:
    """pytest plugin: deselect the waived node ids (matched as suffixes)."""

    def __init__(self, ids):
        self.ids = ids
        self.hit = set()

    def pytest_collection_modifyitems(self, config, items):
        keep, drop = [], []
        for it in items:
            w = next((w for w in self.ids if it.nodeid.endswith(w)), None)
            (drop if w else keep).append(it)
            if w:
                self.hit.add(w)
        if drop:
            config.hook.pytest_deselected(items=drop)
            items[:] = keep


def main(argv):
    import pytest
    if not os.path.isdir(SUITE):
        print(f"reference suite not staged at {SUITE} (run oracle/build_ref.sh)", file=sys.stderr)
        return 2
    alias()
    plug = _Waive(waived())
    rc = pytest.main([SUITE, "-q", "-p", "no:cacheprovider", "--rootdir", SUITE] + list(argv),
                     plugins=[plug])
    missing = set(plug.ids) - plug.hit
    if missing:
        print(f"waivers that matched no test: {sorted(missing)}", file=sys.stderr)
        return rc or 3
    return rc


if __name__ == "__main__":
    sys.exit(main(sys.argv[1:]))
