#!/usr/bin/env bash
# Build the UNMODIFIED reference package (arxiv 1410.1237 `parlouvain`) into
# oracle/_ref/ref_parlouvain so it can be imported next to this repo's package.
#
# Test infrastructure only: the reference is the CPU checker and the CPU
# baseline arm of bench.py, never part of the product path.  Output goes only to
# oracle/_ref/ (git-ignored, shipped to the GPU box with the gpurun snapshot).
# The reference tree is read-only, so its pure-Python modules are staged here
# verbatim and its Cython kernel is translated + compiled with the flags of
# pkg/setup.py:32 (-O3 -fopenmp -ffp-contract=off).
set -euo pipefail
REF=${REF:-/root/reference/pkg/src/parlouvain}
HERE="$(cd "$(dirname "${BASH_SOURCE[0]}")" && pwd)"
OUT="$HERE/_ref/ref_parlouvain"
if [ ! -d "$REF" ]; then
  echo "reference not present at $REF; keeping prebuilt $OUT" >&2
  exit 0
fi
mkdir -p "$OUT"
cp "$REF"/*.py "$OUT"/
cp "$REF"/_kernels.pyx "$HERE/_ref/_kernels.pyx"
PY=${PYTHON:-python3}
"$PY" -m cython -3 -o "$HERE/_ref/_kernels.c" "$HERE/_ref/_kernels.pyx" \
  --module-name ref_parlouvain._kernels
INC_PY=$("$PY" -c 'import sysconfig; print(sysconfig.get_paths()["include"])')
SUFFIX=$("$PY" -c 'import sysconfig; print(sysconfig.get_config_var("EXT_SUFFIX"))')
/usr/bin/gcc -O3 -fopenmp -ffp-contract=off -fPIC -shared \
  -I"$INC_PY" "$HERE/_ref/_kernels.c" -o "$OUT/_kernels$SUFFIX" -fopenmp
echo "built $OUT/_kernels$SUFFIX"
# the reference's own test suite, verbatim, for oracle/ref_suite.py
TESTS=${REF_TESTS:-$(dirname "$(dirname "$REF")")/tests}
if [ -d "$TESTS" ]; then
  rm -rf "$HERE/_ref/ref_tests"
  cp -r "$TESTS" "$HERE/_ref/ref_tests"
  echo "staged $HERE/_ref/ref_tests"
fi
