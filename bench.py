#!/usr/bin/env python3
"""Benchmark: parallel-Louvain local-move iteration on B200 (BASELINE.json config 2).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Workload (config 2 of BASELINE.json): R-MAT scale 20, edge factor 16,
(a,b,c,d) = (.57,.19,.19,.05), self loops dropped, duplicates merged,
f64 weights U[1,10), int32 ids -- generated on device from a counter-based
RNG (bit-identical to the numpy generator the CPU arms use).  As `run()` does
with the default RunConfig, the graph is vertex-followed (n 1,048,576 ->
908,790) and, since n >= color_cutoff, phase 1 is coloured (210 colours).

One step = one phase-1 local-move iteration exactly as the reference's
run_phase performs it (PL/engine.py:186-197): the state is reset to the
singleton state, every colour class is swept in ascending colour (decide +
exact apply per class), then Q is reduced.  Metric: local-move edges/s per
iteration = M / t_iter with M = num_edges of the iterated graph
(pkg/benchmarks/bench_backends.py:81 uses num_edges / seconds).  The CSR
(~380 MB) is larger than L2 (126 MB), so no explicit flush is needed.

`value`: device-resident inputs, CUDA-event timing over K steps, max over
ranks.  `e2e`: the same step through the C-ABI with host buffers -- the
step's input state is copied from pinned host memory and the resulting
assignment + Q are copied back inside the timed region.
`roofline`: the decide kernels (the dominant kernel family), algorithmic
bytes 41 n + 16 nnz + 8 sum(cand) per iteration over their summed CUDA-event
time.  `cpu_baseline`: the unmodified reference (oracle/_ref, compiled
Cython/OpenMP, all host cores) running the same iteration on the same graph.

Multi-GPU (torchrun): the graph is 1D vertex-partitioned over the N ranks
(strong scaling): each rank decides its slice of every colour stage, the
decided slices are exchanged by NCCL broadcasts captured in the iteration's
CUDA graph, and every rank replays the exact apply; see DESIGN.md.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIG = dict(scale=20, edge_factor=16, seed=0)
METRIC = "local-move edges/sec per iteration"
UNIT = "edges/s"


def _args():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=10)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--scale", type=int, default=None,
                   help="R-MAT scale (c2 config; N > 1: default 25 + log2 N)")
    p.add_argument("--config", default="c4_chung_lu",
                   choices=["c1_sbm", "c2_rmat20", "c3_grid", "c4_chung_lu"],
                   help="BASELINE config to run (default: config 4, the largest that fits "
                        "one GPU -- the headline)")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-louvain", action="store_true", help="skip the full run() timing")
    p.add_argument("--mode", choices=["colored", "uncolored"], default="colored")
    p.add_argument("--partitioned", action="store_true",
                   help="under torchrun with one rank: the partitioned pipeline (1-rank NCCL)")
    p.add_argument("--partitioned-replicated", action="store_true",
                   help="N > 1: the older replicated-CSR partitioned engine on the config graph")
    a = p.parse_args()
    a.scale_set = a.scale is not None
    if a.scale is None:
        a.scale = CONFIG["scale"]
    return a


def _dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


# ------------------------------------------------------------------ clocks

class ClockSampler:
    """SM clocks + throttle reasons during the timed region (NVML every 5 ms,
    nvidia-smi as a fallback)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    # NVML clocks-event reason bits: hw_slowdown, hw_thermal, sw_thermal, sw_power_cap
    BITS = (0x8, 0x40, 0x20, 0x4)

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self._stop = threading.Event()
        self._t = None

    def _loop(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            mx = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
            while not self._stop.is_set():
                sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                rs = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                self.rows.append([str(self.index), str(sm), str(mx), "", ""] +
                                 ["Active" if rs & b else "Not Active" for b in self.BITS])
                self._stop.wait(0.005)
            return
        except Exception:
            pass
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True,
                                     text=True, timeout=5).stdout.strip()
                if out:
                    self.rows.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._loop, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4)
                          if len(r) > 5 + i and r[5 + i].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


def _traffic(mode: str, scale: int, config: str = "c4_chung_lu"):
    """DRAM bytes per iteration of the decide kernels, from the committed ncu
    capture (profiles/traffic.json, keyed "config/mode"), else None."""
    if config == "c2_rmat20" and scale != CONFIG["scale"]:
        return None
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as fh:
            return float(json.load(fh)[f"{config}/{mode}"])
    except Exception:
        return None


def _peak_hbm():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


DECIDE_KERNELS = ("k_decide_", "k_hub_accum", "k_hub_pass", "k_single_", "k_ah_accum", "k_ah_pass")


def _cupti_decide_ms(step):
    """One replay of `step` under CUPTI: (union of the decide kernels'
    intervals in ms, span of all kernels in ms, candidates)."""
    import torch
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        _, _, cand = step()
        torch.cuda.synchronize()
    ks = sorted((e.time_range.start, e.time_range.end, e.name) for e in prof.events()
                if e.device_type.name == "CUDA")
    span = (max(k[1] for k in ks) - ks[0][0]) / 1e3 if ks else 0.0
    busy, cs, ce = 0.0, None, None
    for s0, e0, nm in ks:
        if not any(d in nm for d in DECIDE_KERNELS):
            continue
        if ce is None or s0 > ce:
            if ce is not None:
                busy += ce - cs
            cs, ce = s0, e0
        else:
            ce = max(ce, e0)
    if ce is not None:
        busy += ce - cs
    return busy / 1e3, span, cand


# ------------------------------------------------------------- CPU arms

def _reference_module():
    ref_dir = os.path.join(ROOT, "oracle", "_ref")
    if os.path.isdir(os.path.join(ref_dir, "ref_parlouvain")):
        sys.path.insert(0, ref_dir)
        try:
            import ref_parlouvain
            return ref_parlouvain
        except ImportError:
            return None
    return None


def cpu_iteration_rate(off, nbr, wts, selfw, classes, steps: int, warmup: int = 0,
                       nslices: int = 10):
    """Time the reference's phase-1 local moving (or the oracle port) on host
    cores, in bounded samples: step s sweeps the colour classes s mod
    `nslices`, s mod nslices + nslices, ... (a strided 1/nslices of the
    iteration's stages; `nslices` consecutive steps cover one whole iteration)
    on one evolving state, plus 1/nslices of a modularity reduction.  An
    uncoloured iteration is cut into `nslices` contiguous vertex blocks.
    Returns (per-step (entries, seconds) list, kind, cores, M, nnz)."""
    ref = _reference_module()
    n = len(off) - 1
    if len(classes) == 1:
        classes = np.array_split(np.asarray(classes[0]), nslices)
    deg = np.diff(off)
    slices = [classes[j::nslices] for j in range(nslices)]
    entries = [int(sum(int(deg[c].sum()) for c in sl)) for sl in slices]
    if ref is not None:
        g = ref.Graph(n, off.astype(np.int64), nbr.astype(np.int64), wts.astype(np.float64),
                      selfw.astype(np.float64))
        cores = os.cpu_count() or 1
        kind = "reference"
        s = ref.singleton_state(g)

        def sweep(sl):
            for st in sl:
                ref.run_iteration(g, s, st, cores)

        def q():
            ref.modularity(g, s)
    else:
        sys.path.insert(0, os.path.join(ROOT, "oracle"))
        import oracle as orc
        g = orc.from_edges(*_csr_to_records(off, nbr, wts, selfw), num_vertices=n)
        cores = 1
        kind = "port"
        s = orc.singleton_state(g)

        def sweep(sl):
            for st in sl:
                orc.run_iteration(g, s, st)

        def q():
            orc.modularity(g, s)
    t0 = time.perf_counter()
    q()
    tq = (time.perf_counter() - t0) / nslices
    out = []
    for k in range(warmup + steps):
        j = k % nslices
        t0 = time.perf_counter()
        sweep(slices[j])
        dt = time.perf_counter() - t0 + tq
        if k >= warmup:
            out.append((entries[j], dt))
    return out, kind, cores, g.num_edges, int(len(nbr))


def _sampled_value(samples, M, nnz):
    """edges/s of sampled steps: each step's edges = M x its share of the
    adjacency entries swept."""
    ent = sum(e for e, _ in samples)
    sec = sum(t for _, t in samples)
    return M * ent / nnz / sec, sec / len(samples), ent / nnz


def _parallel_records(config: str, scale: int, procs: int):
    """The numpy record generator of a config, its record-draw range split
    over `procs` forked workers (counter-based draws: ranges concatenate to
    the serial output)."""
    import multiprocessing as mp
    from paper_1410_1237_b200 import synthetic as syn
    if config == "c2_rmat20":
        fn, params = syn.rmat_records, dict(scale=scale, edge_factor=CONFIG["edge_factor"])
        R = CONFIG["edge_factor"] << scale
    elif config == "c4_chung_lu":
        fn, params = syn.chung_lu_records, dict(syn.CONFIGS[config][2])
        R = int(round(syn.chung_lu_cdf(**params)[-1] / 2.0))
    else:
        host, _, params = syn.CONFIGS[config]
        return host(seed=CONFIG["seed"], **params)
    params["seed"] = CONFIG["seed"]
    step = -(-R // procs)
    jobs = [(fn, params, a, min(R, a + step)) for a in range(0, R, step)]
    with mp.get_context("fork").Pool(len(jobs)) as pool:
        parts = pool.map(_records_range, jobs)
    return tuple(np.concatenate([p[i] for p in parts]) for i in range(3))


def _records_range(job):
    fn, params, a, b = job
    return fn(**params, r_begin=a, r_end=b)


def _csr_to_records(off, nbr, wts, selfw):
    n = len(off) - 1
    src = np.repeat(np.arange(n, dtype=np.int64), np.diff(off))
    keep = nbr >= src
    return src[keep], nbr[keep].astype(np.int64), wts[keep]


def _config_desc(args):
    return f"c2_rmat{args.scale}" if args.config == "c2_rmat20" else args.config


def host_phase1_inputs(scale: int, config: str = "c2_rmat20"):
    """The VF'd phase-1 graph and its colour classes without the GPU: the
    numpy generator (record ranges on all host cores), the CPU oracle's CSR
    build and vertex following (pinned to the reference), and the
    reference's own compiled colouring on all host cores when it is present
    (else the oracle's)."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as orc
    from paper_1410_1237_b200 import synthetic as syn
    cores = os.cpu_count() or 1
    u, v, w = _parallel_records(config, scale, cores)
    n = (1 << scale) if config == "c2_rmat20" else syn.config_num_vertices(config)
    g = orc.from_edges(u, v, w, num_vertices=n)
    del u, v, w
    vf = orc.vf_compact(g)
    del g
    gg = vf.graph
    ref = _reference_module()
    if ref is not None:
        rg = ref.Graph(gg.num_vertices, gg.adjacency_offsets, gg.neighbors, gg.weights,
                       gg.self_loop_weights)
        col = ref.color_graph(rg, cores)
    else:
        col = orc.color_graph(gg)
    return gg, col.classes(), col.num_colors


def reference_louvain(cores: int):
    """The reference's whole run() (PL/engine.py:259-315, compiled backend,
    worker_count = all host cores) on config 2, timed from its own
    Graph.from_edges of the records; None if the reference is absent."""
    ref = _reference_module()
    if ref is None:
        return None
    u, v, w = _parallel_records("c2_rmat20", CONFIG["scale"], cores)
    t0 = time.perf_counter()
    g = ref.Graph.from_edges(u, v, w, num_vertices=1 << CONFIG["scale"])
    t1 = time.perf_counter()
    h = ref.run(g, ref.RunConfig(worker_count=cores))
    t2 = time.perf_counter()
    return {"config": "c2_rmat20", "seconds": t2 - t1, "graph_build_seconds": t1 - t0,
            "includes": "reference run() (VF, colouring, all phases, rebuilds) on all host "
                        "cores; Graph.from_edges timed separately",
            "cores": cores, "final_modularity": h.final_modularity,
            "phases": len(h.phases), "communities": h.num_communities}


def run_reference(args):
    ws, rank, _ = _dist()
    if rank != 0:
        return
    scale = args.scale
    gg, classes, ncol = host_phase1_inputs(scale, args.config)
    if args.mode == "uncolored":
        classes = [np.arange(gg.num_vertices, dtype=np.int64)]
    samples, kind, cores, M, nnz = cpu_iteration_rate(
        gg.adjacency_offsets, gg.neighbors, gg.weights, gg.self_loop_weights, classes,
        args.steps, args.warmup)
    val, t_step, cover = _sampled_value(samples, M, nnz)
    sample = (f"{len(samples)} steps after {args.warmup} warm-up steps; a step = a strided "
              f"1/10 of the phase-1 {'coloured (' + str(ncol) + ' stages)' if args.mode == 'colored' else 'uncoloured'} "
              f"local-move iteration of {_config_desc(args)} after VF (every 10th colour class, "
              f"one evolving state from the singleton start); the steps swept {cover:.2f} "
              f"iterations' worth of adjacency entries")
    louv = None if args.no_louvain else reference_louvain(cores)
    line = {
        "impl": "reference", "metric": METRIC, "value": val, "unit": UNIT, "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_step * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (counter-based generator of the BASELINE config, numpy)",
        "config": {"workload": f"{_config_desc(args)} phase-1 {args.mode} local-move iteration",
                   "graph": {"n": gg.num_vertices, "M": M, "nnz": nnz, "colours": ncol}},
        "cpu_baseline": {"value": val, "unit": UNIT, "cores": cores, "kind": kind,
                         "sample": sample},
        "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "louvain_reference": louv,
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ ours

def run_partitioned(args):
    """N > 1 ranks: the 1D vertex-partitioned pipeline (paper_1410_1237_b200.
    partition) on R-MAT scale 25 + log2 N (weak scaling: N = 8 is config 5,
    R-MAT s28; --scale overrides).  Each rank generates 1/N of the record
    draws, owns 1/N of the rows (entry-balanced ranges) and holds the
    replicated state; construction, VF and colouring run partitioned; one
    step = one phase-1 coloured local-move iteration (every colour class:
    decide own slice, one NCCL all-gather of the slices, replicated exact
    apply), timed with CUDA events, max over ranks."""
    import torch
    import torch.distributed as dist
    import paper_1410_1237_b200 as pl
    from paper_1410_1237_b200 import partition as P
    from paper_1410_1237_b200 import dist as pdist
    ws, rank, local = _dist()
    dev = torch.device("cuda", local)
    ex = P.Exchange()
    scale = args.scale if args.scale_set else 25 + int(round(math.log2(ws)))
    comm = pdist.nccl_communicator(rank, ws)

    def tmax(x):
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    torch.cuda.synchronize()
    t0 = time.perf_counter()
    g0 = P.rmat_graph_part(scale, ex, edge_factor=CONFIG["edge_factor"], seed=CONFIG["seed"])
    torch.cuda.synchronize()
    t_build = tmax(time.perf_counter() - t0)
    t0 = time.perf_counter()
    vf = P.vf_compact_part(g0, ex)
    g = vf.graph
    del g0
    col = P.color_part(g, ex)
    torch.cuda.synchronize()
    t_vfcol = tmax(time.perf_counter() - t0)
    s0 = P.singleton_state_part(g)
    d0 = s0.device()
    st = {k: (t.clone() if t is not None else None) for k, t in d0.items()}
    state = pl.CommunityState.from_device(st["assignment"], st["a_tot"], st["w_internal"],
                                          st["sizes"])
    eng = P.PartEngine(g, state, col, ex, comm=comm)

    def reset():
        for k in ("assignment", "a_tot", "w_internal", "sizes"):
            st[k].copy_(d0[k])

    def step():
        reset()
        return eng.iterate()

    for _ in range(args.warmup):
        step()
    dist.barrier()
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream()
    with ClockSampler(local) as clk:
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        ev0.record(stream)
        for _ in range(args.steps):
            q, moves, cand = step()
        ev1.record(stream)
        torch.cuda.synchronize()
    dist.barrier()
    ms = tmax(ev0.elapsed_time(ev1)) / args.steps
    M = g.num_edges
    value = M / (ms / 1e3)
    reset()
    torch.cuda.synchronize()
    dm, span, cand = _cupti_decide_ms(eng.iterate)
    dm = tmax(dm)
    n = g.num_vertices
    nnz_own = g.nnz_local
    own = g.hi - g.lo
    decide_bytes = 41 * own + 16 * nnz_own + 8 * cand
    peak, peak_kind = _peak_hbm()
    achieved = decide_bytes / (dm / 1e3) / 1e9 if dm > 0 else 0.0
    # e2e: the step's input state from pinned host memory, the assignment back
    h = {k: torch.empty(d0[k].shape, dtype=d0[k].dtype, pin_memory=True)
         for k in ("assignment", "a_tot", "w_internal", "sizes")}
    for k in h:
        h[k].copy_(d0[k].cpu())
    o_assign = torch.empty(n, dtype=torch.int32, pin_memory=True)

    def e2e_step():
        for k in h:
            st[k].copy_(h[k], non_blocking=True)
        eng.iterate()
        o_assign.copy_(st["assignment"], non_blocking=True)
        stream.synchronize()

    e2e_step()
    dist.barrier()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        e2e_step()
    e1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = tmax(e0.elapsed_time(e1)) / args.steps
    launches = eng.graph_kernels() * args.steps
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (counter-based R-MAT, generated on device, 1/N of the draws "
                    "per rank)",
            "config": {"workload": f"rmat_s{scale} phase-1 colored local-move iteration "
                                   f"(1D vertex partition over {ws} ranks)",
                       "graph": {"n": n, "M": M, "colours": col.num_colors,
                                 "nnz_rank0": nnz_own, "bounds": [int(b) for b in g.bounds]},
                       "parallelism": f"vertex-partition{ws} (NCCL all-gather of the decided "
                                      f"slices per colour class, replicated exact apply)",
                       "construction_seconds": t_build, "vf_coloring_seconds": t_vfcol,
                       "l2": "inputs larger than L2"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": None, "peak_kind": peak_kind,
                         "kernel": "decide (tiers 0-4), rank 0's slices",
                         "bytes_per_iter": decide_bytes, "ms_per_iter": dm,
                         "timing": "union of decide-kernel intervals (CUPTI), max over ranks"},
            "iteration": {"q": q, "moves": moves},
            "cpu_baseline": None,
            "e2e": {"value": M / (e2e_ms / 1e3), "unit": UNIT,
                    "h2d_bytes_per_step": 24 * n, "d2h_bytes_per_step": 4 * n},
            "gpu_launches": int(launches),
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    eng.close()
    pdist.destroy_communicator(comm)


def run_ours(args):
    import torch
    import torch.distributed as dist
    ws, rank, local = _dist()
    torch.cuda.set_device(local)
    if ws > 1 or (args.partitioned and "WORLD_SIZE" in os.environ):
        from paper_1410_1237_b200.dist import stdout_to_stderr
        with stdout_to_stderr():  # NCCL's banner must not share stdout with the JSON line
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
            dist.barrier()
        if not args.partitioned_replicated:
            run_partitioned(args)
            dist.destroy_process_group()
            return
    import paper_1410_1237_b200 as pl
    from paper_1410_1237_b200 import _lib, synthetic as syn
    from paper_1410_1237_b200.engine import PhaseEngine

    L = _lib.lib()
    dev = torch.device("cuda", local)
    scale = args.scale
    # ---- setup (untimed): generate, build, VF, colour -- all on device
    if args.config == "c2_rmat20":
        u, v, w, n0 = syn.rmat_device(scale, CONFIG["edge_factor"], seed=CONFIG["seed"])
        g0 = pl.Graph.from_device_records(u, v, w, n0)
        del u, v, w
    else:
        g0 = syn.config_graph(args.config, seed=CONFIG["seed"])
    vf = pl.vf_compact(g0)
    g = vf.graph
    n = g.num_vertices
    col = pl.color_graph(g) if args.mode == "colored" else None
    ncol = col.num_colors if col is not None else 0
    s0 = pl.singleton_state(g)
    d0 = s0.device()
    st = {k: (t.clone() if t is not None else None) for k, t in d0.items()}
    state = pl.CommunityState.from_device(st["assignment"], st["a_tot"], st["w_internal"],
                                          st["sizes"])
    coloring = col if args.mode == "colored" else None
    comm = None
    if ws > 1 or args.partitioned:
        # 1D vertex partition: each rank decides its slice of every stage, NCCL
        # broadcasts of the decided slices inside the iteration graph, every
        # rank replays the exact apply
        from paper_1410_1237_b200 import dist as pdist
        comm = pdist.nccl_communicator(rank, ws)
        eng = pdist.PartitionedPhaseEngine(g, state, coloring, rank, ws, comm=comm)
    else:
        eng = PhaseEngine(g, state, coloring)
    stream = torch.cuda.current_stream()

    def reset():
        st["assignment"].copy_(d0["assignment"])
        st["a_tot"].copy_(d0["a_tot"])
        st["w_internal"].copy_(d0["w_internal"])
        st["sizes"].copy_(d0["sizes"])

    def step(e=eng):
        reset()
        return e.iterate()

    for _ in range(args.warmup):
        step()
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        ev0.record(stream)
        for _ in range(args.steps):
            q, moves_it, _ = step()
        ev1.record(stream)
        torch.cuda.synchronize()
    # kernels launched by graph replays are not counted by the host-side
    # counter: gpu_launches = the iteration graph's kernel nodes x steps
    if ws > 1:
        dist.barrier()
    ms = ev0.elapsed_time(ev1)
    if ws > 1:
        t = torch.tensor([ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    t_iter = ms / 1e3 / args.steps
    M = g.num_edges
    nnz = g.nnz
    value = M / t_iter  # one graph, partitioned over the ranks (strong scaling)
    # decide-kernel time INSIDE the timed step's graph: CUPTI (torch.profiler)
    # records every graph-launched kernel of extra replays of the same engine;
    # the decide family's time is the union of its kernel intervals per
    # iteration (never more than the step itself)
    per_iter_launches = eng.graph_kernels()  # kernel nodes of the timed step's graph
    dms, cands, spans = [], [], []
    for _ in range(3):
        reset()
        torch.cuda.synchronize()
        dm, span, cand = _cupti_decide_ms(eng.iterate)
        dms.append(dm)
        spans.append(span)
        cands.append(cand)
    decide_ms = float(np.median(dms))
    span_ms = float(np.median(spans))
    cand_per_iter = float(np.mean(cands))
    moves_per_iter = float(moves_it)
    launches = per_iter_launches * args.steps
    # the first stage starts from the singleton state: its rows' neighbours
    # are their own communities, so it reads no assign[j] (4 B per entry)
    off_h = g.adjacency_offsets
    first = col.classes()[0] if col is not None else np.arange(n)
    e_first = int((off_h[np.asarray(first) + 1] - off_h[np.asarray(first)]).sum())
    decide_bytes = 41 * n + 16 * nnz + 8 * cand_per_iter - 4 * e_first
    iter_bytes = decide_bytes + 84 * moves_per_iter + 16 * n
    peak, peak_kind = _peak_hbm()
    achieved = decide_bytes / (decide_ms / 1e3) / 1e9
    qbuf = torch.tensor([q], dtype=torch.float64, device=dev)

    # ---- e2e through the C ABI with host buffers (pinned), same step.  Two
    # state buffers, each bound to its own engine: step k+1's inputs go up on
    # a copy stream while step k computes, and step k's assignment comes back
    # while step k+1 computes (every step's copies are inside the timed region)
    keys = ("assignment", "a_tot", "w_internal", "sizes")
    hin = {k: torch.empty(d0[k].shape, dtype=d0[k].dtype, pin_memory=True) for k in keys}
    for k in keys:
        hin[k].copy_(d0[k].cpu())
    st2 = {k: torch.empty_like(st[k]) for k in keys}
    state2 = pl.CommunityState.from_device(st2["assignment"], st2["a_tot"], st2["w_internal"],
                                           st2["sizes"])
    eng2 = PhaseEngine(g, state2, coloring) if comm is None else None
    bufs = [(st, eng), (st2, eng2)] if eng2 is not None else [(st, eng)]
    nb = len(bufs)
    o_assign = [torch.empty(n, dtype=torch.int32, pin_memory=True) for _ in range(nb)]
    o_q = [0.0] * nb
    cs = torch.cuda.Stream()
    ev_in = [torch.cuda.Event() for _ in range(nb)]
    ev_done = [torch.cuda.Event() for _ in range(nb)]

    def h2d(b):
        with torch.cuda.stream(cs):
            for k in keys:
                bufs[b][0][k].copy_(hin[k], non_blocking=True)
            ev_in[b].record(cs)

    def run_steps(k_steps):
        h2d(0)
        for k in range(k_steps):
            b = k % nb
            if k + 1 < k_steps and nb > 1:
                h2d((k + 1) % nb)
            stream.wait_event(ev_in[b])
            qq, _, _ = bufs[b][1].iterate()   # Q comes back to the host inside
            o_q[b] = qq
            ev_done[b].record(stream)
            cs.wait_event(ev_done[b])
            with torch.cuda.stream(cs):
                o_assign[b].copy_(bufs[b][0]["assignment"], non_blocking=True)
            if nb == 1 and k + 1 < k_steps:
                cs.synchronize()
                h2d(0)

    run_steps(max(2, args.warmup))
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(cs)
    run_steps(args.steps)
    e1.record(cs)
    torch.cuda.synchronize()
    e2e_ms = e0.elapsed_time(e1)
    if ws > 1:
        t = torch.tensor([e2e_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())
    e2e_val = M / (e2e_ms / 1e3 / args.steps)
    if eng2 is not None:
        eng2.close()

    # ---- full Louvain run() (end-to-end Louvain time, final modularity):
    # the graph generated and built on device (Graph.from_edges), then run()
    # timed on its own -- the reference's louvain_reference line times its
    # run() apart from its Graph.from_edges the same way
    louv = None
    if not args.no_louvain:
        secs, builds = [], []
        for _ in range(3):  # first: cold (graph captures, pool growth); then warm
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            if args.config == "c2_rmat20":
                uu, vv, ww, nn = syn.rmat_device(scale, CONFIG["edge_factor"], seed=CONFIG["seed"])
                gg = pl.Graph.from_device_records(uu, vv, ww, nn)
                del uu, vv, ww
            else:
                gg = syn.config_graph(args.config, seed=CONFIG["seed"])
            torch.cuda.synchronize()
            t1 = time.perf_counter()
            h = pl.run(gg, pl.RunConfig(color_cutoff=0 if args.config == "c1_sbm" else 100_000))
            torch.cuda.synchronize()
            secs.append(time.perf_counter() - t1)
            builds.append(t1 - t0)
            del gg
        louv = {"seconds": min(secs), "cold_seconds": secs[0], "runs_seconds": secs,
                "build_seconds": min(builds),
                "includes": "run() (VF, colouring, every phase, rebuilds, flatten) on the "
                            "device-built graph; build_seconds = generation + Graph.from_edges "
                            "on device",
                "final_modularity": h.final_modularity,
                "phases": len(h.phases), "communities": h.num_communities,
                "iterations": [p.stats.iterations for p in h.phases]}

    # ---- CPU baseline (rank 0, N == 1)
    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        off = g.adjacency_offsets
        nb = g.neighbors
        wt = g.weights
        sw = g.self_loop_weights
        if args.mode == "colored":
            cl = col.classes()
        else:
            cl = [np.arange(n, dtype=np.int64)]
        smp, kind, cores, Mc, nnzc = cpu_iteration_rate(off, nb, wt, sw, cl, steps=3, warmup=1)
        cval, tc, cover = _sampled_value(smp, Mc, nnzc)
        cpu = {"value": cval, "unit": UNIT, "cores": cores, "kind": kind,
               "sample": f"3 steps after 1 warm-up step on the same graph; a step = a strided "
                         f"1/10 of the phase-1 {args.mode} iteration ({len(cl)} stages; every "
                         f"10th class), one evolving state from the singleton start; "
                         f"{tc * 1e3:.0f} ms per step, {cover:.2f} iterations' worth of entries"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (counter-based generator of the BASELINE config, on device)",
            "config": {"workload": f"{_config_desc(args)} phase-1 {args.mode} local-move iteration",
                       "graph": {"n": n, "M": M, "nnz": nnz, "colours": ncol,
                                 "integral": g.integral},
                       "parallelism": f"vertex-partition{ws} (NCCL slice broadcasts per stage)"
                       if comm is not None else "single",
                       "l2": "inputs larger than L2 (CSR %.0f MB)" % (nnz * 12 / 1e6)},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": _traffic(args.mode, scale, args.config),
                         "traffic_unit": "bytes per iteration (ncu, warm caches)",
                         "peak_kind": peak_kind,
                         "kernel": "decide (tiers 0-4 and the ahead tables)",
                         "bytes_per_iter": decide_bytes, "ms_per_iter": decide_ms,
                         "share_of_step": decide_ms / span_ms,
                         "timing": "union of decide-kernel intervals in the iteration graph "
                                   "(CUPTI), median of 3 replays; span %.3f ms" % span_ms},
            "iteration": {"bytes": iter_bytes, "gbs": iter_bytes / t_iter / 1e9,
                          "frac": iter_bytes / t_iter / 1e9 / peak,
                          "moves": moves_per_iter, "cand": cand_per_iter, "q": q,
                          "kernels_per_iter": per_iter_launches},
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_val, "unit": UNIT, "h2d_bytes_per_step": 24 * n,
                    "d2h_bytes_per_step": 4 * n + 8,
                    "how": "per step: the state (assignment, a_tot, w_internal, sizes) from "
                           "pinned host memory, the iteration through the engine's C ABI, Q and "
                           "the assignment back; double-buffered so step k+1's upload and step "
                           "k's download overlap compute on a copy stream"},
            "gpu_launches": int(launches),
            "clocks": clk.summary(),
            "louvain": louv,
        }
        print(json.dumps(line), flush=True)
    if comm is not None:
        eng.close()
        from paper_1410_1237_b200 import dist as pdist
        pdist.destroy_communicator(comm)
    if ws > 1:
        dist.destroy_process_group()


def _self_launch(args) -> bool:
    """`--gpus N` without torchrun: re-exec this script under torchrun with N
    ranks (one per GPU).  With WORLD_SIZE set, N must equal it."""
    ws = os.environ.get("WORLD_SIZE")
    if ws is not None:
        if int(ws) != args.gpus:
            raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={ws}")
        return False
    if args.gpus <= 1:
        return False
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
           f"--master-port={29500 + os.getpid() % 1000}", os.path.abspath(__file__)]
    cmd += sys.argv[1:]
    raise SystemExit(subprocess.run(cmd).returncode)


def main():
    args = _args()
    _self_launch(args)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
