"""Build libplv.so (the sm_100a CUDA hot path + C ABI) in-tree with nvcc.

    python -m paper_1410_1237_b200.build        # or __graft_entry__.build()

Objects go to paper_1410_1237_b200/_build/, the shared library to
paper_1410_1237_b200/libplv.so (both git-ignored; the .so ships to the GPU box
with the repo snapshot).  Flags: sm_100a only, -lineinfo for ncu source
mapping, --fmad=false so no product or sum is contracted into an FMA
(the reference is built with -ffp-contract=off, pkg/setup.py:32).
"""

from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
# Experiment variants (A/B sweeps without editing sources):
#   PLV_VARIANT=name PLV_DEFINES="-DKNOB=1 ..." python -m paper_1410_1237_b200.build
# builds _build_name/ and libplv_name.so; PLV_VARIANT=name at run time loads it.
VARIANT = os.environ.get("PLV_VARIANT", "")
DEFINES = os.environ.get("PLV_DEFINES", "").split()
OUT_DIR = os.path.join(HERE, "_build" + (f"_{VARIANT}" if VARIANT else ""))
LIB = os.path.join(HERE, f"libplv_{VARIANT}.so" if VARIANT else "libplv.so")
INCLUDE = os.path.join(os.path.dirname(HERE), "include")

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-std=c++17", "--fmad=false", "-lineinfo", "--extended-lambda",
         "-Xcompiler", "-fPIC",
         "-Xcompiler", "-Wno-deprecated-declarations", f"-I{INCLUDE}"]


def _sources():
    return sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith(".cu"))


def _headers():
    hs = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h"))]
    hs += [os.path.join(INCLUDE, f) for f in os.listdir(INCLUDE) if f.endswith(".h")]
    return hs


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def _compile(src, verbose=False):
    obj = os.path.join(OUT_DIR, os.path.basename(src)[:-3] + ".o")
    if _stale(obj, [src] + _headers()):
        cmd = [NVCC, *ARCH, *FLAGS, *DEFINES, "-c", src, "-o", obj]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
        if verbose:
            sys.stderr.write(r.stderr)
    return obj


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(OUT_DIR, exist_ok=True)
    srcs = _sources()
    if force:
        for f in os.listdir(OUT_DIR):
            os.remove(os.path.join(OUT_DIR, f))
    with ThreadPoolExecutor(max_workers=min(8, len(srcs))) as ex:
        objs = list(ex.map(lambda s: _compile(s, verbose), srcs))
    if force or _stale(LIB, objs):
        cmd = [NVCC, *ARCH, "-shared", "-o", LIB, *objs, "-cudart", "static"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
