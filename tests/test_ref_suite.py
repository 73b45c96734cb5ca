"""The reference's own test suite (pkg/tests, staged verbatim by
oracle/build_ref.sh) run against this package with `parlouvain` aliased to it
(oracle/ref_suite.py).  Waived tests are listed with reasons in
tests/ref_suite_waivers.txt."""

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SUITE = os.path.join(ROOT, "oracle", "_ref", "ref_tests")


@pytest.mark.skipif(not os.path.isdir(SUITE), reason="reference suite not staged")
def test_reference_suite_passes():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "oracle", "ref_suite.py"), "-x"],
                       capture_output=True, text=True, timeout=1800)
    tail = (r.stdout + r.stderr)[-4000:]
    assert r.returncode == 0, tail
    assert " passed" in r.stdout, tail
