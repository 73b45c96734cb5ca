"""GPU: the bench's multi-GPU code path runs end to end on one GPU -- torchrun
with one rank and `--partitioned` drives the 1D-partitioned pipeline
(partitioned construction, VF, colouring, the NCCL-captured iteration graph
with its all-gather, the double-buffered e2e) -- and prints one JSON line
with the contract's keys."""

import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_partitioned_bench_one_rank():
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=1",
           "--master-addr=127.0.0.1", f"--master-port={_port()}", os.path.join(ROOT, "bench.py"),
           "--partitioned", "--scale", "14", "--steps", "2", "--warmup", "1",
           "--no-cpu-baseline", "--no-louvain"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "dtype", "config", "roofline", "e2e",
              "gpu_launches", "clocks"):
        assert k in line, k
    assert line["value"] > 0 and line["e2e"]["value"] > 0 and line["gpu_launches"] > 0
    assert "rmat_s14" in line["config"]["workload"]
