"""Benchmark of the B200 time-stepping hot path (driver contract: one JSON line).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Metric: FP64 cell updates per second (fluid cells x steps / device time), the
reference's own throughput measure (timestepper.py:216-217) and the paper's
"volumes processed per second".  Workload: the wall-impact dambreak (C5,
SURVEY.md 8(d)) as an x-slab of 4096 x 16384 cells per GPU; with N GPUs the
global grid is (4096 N) x 16384 over the same physical domain (weak scaling).
The state (4.3 GB per GPU) is far larger than L2, so no flush is needed.

--impl reference times the reference algorithm on the host CPU (the C
restatement in oracle/, all host threads) on a bounded sample of the same
workload; see DESIGN.md "Measurement".
"""
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

METRIC = "FP64 cell updates/sec at 1/2/4/8 B200; % of HBM/FP64 roofline; CPU baseline"
UNIT = "cell-updates/s"
PUBLISHED = 2.0e7  # PAPER.md:26-27 "twenty million volumes/s"
SLAB = (4096, 16384)
HBM_BYTES_PER_CELL = 64.0  # read 4 + write 4 FP64 dynamic components


def committed_traffic(nx, ny):
    """DRAM bytes per k_step launch and the ncu counters of the committed
    capture (profiles/kstep_traffic.json) when it was taken on this slab shape
    (an N-rank run's per-rank slab has the N = 1 shape)."""
    tpath = os.path.join(ROOT, "profiles", "kstep_traffic.json")
    if not os.path.exists(tpath):
        return None, None
    with open(tpath) as f:
        tj = json.load(f)
    if tj.get("grid") != [nx, ny]:
        return None, None
    ncu = {k: tj.get(k) for k in ("fp64_pipe_active_pct", "issue_active_pct",
                                   "warps_per_sm", "registers_per_thread")}
    ncu["source"] = tj.get("source")
    return tj.get("dram_bytes_per_launch"), ncu


def flops_per_step(n_fluid, n2nd, ex, ey):
    """Algorithmic FP64 work of one step (dynamic counts of
    the reference code paths)."""
    return 224.0 * n_fluid + 125.0 * n2nd + 276.0 * ex + 494.0 * ey


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except OSError:
        return {}


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 50 ms during the
    timed region (B200_PROFILING.md clocks line)."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")
    NAMES = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")

    def __init__(self, gpu=0):
        self.gpu = gpu  # index or comma-separated list of indices
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            time.sleep(0.5)  # let the sampler start before the timed region
        except OSError:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        time.sleep(0.1)
        self.proc.terminate()
        out, _ = self.proc.communicate(timeout=10)
        rows = [[x.strip() for x in ln.split(",")] for ln in out.splitlines() if ln.strip()]
        rows = [r for r in rows if len(r) >= 6]
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        reasons = sorted({self.NAMES[k] for r in rows for k in range(4) if r[2 + k] == "Active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(rows)}


def slab():
    """Per-GPU workload grid; WB_BENCH_SLAB=NXxNY shrinks it (CPU tests only)."""
    v = os.environ.get("WB_BENCH_SLAB")
    if v:
        a, b = v.lower().split("x")
        return int(a), int(b)
    return SLAB


def bench_config(nx, ny, n_fluid, gpus, extra=None):
    """The workload description shared by both arms (same dict = same config)."""
    c = {"workload": f"wall-impact (C5) dambreak, x-slab {nx // gpus}x{ny} per GPU",
         "grid": [nx, ny], "fluid_cells": n_fluid, "domain": [0, 3.2, 0, 1.8],
         "l2": "state 4.3 GB per GPU >> 126 MB L2 (no flush needed)"}
    if extra:
        c.update(extra)
    return c


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def _oracle():
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as orc  # CPU-baseline / reference-arm legs only
    return orc


def oracle_window(res, warmup, steps, threads, budget_s):
    """The reference algorithm (C restatement in oracle/, pinned bit-exactly to
    the reference) on the bench workload and the bench's step window: `warmup`
    untimed steps, then up to `steps` timed steps (stopping early once
    `budget_s` of wall time is used).  Returns (cell-updates/s, steps timed,
    seconds)."""
    orc = _oracle()
    from paper_1806_04960_b200.scenarios import build_scenario
    orc.set_threads(threads)
    sc = build_scenario("wall-impact", res)
    sim = orc.OracleSimulation(sc.grid, sc.params, sc.q0, sc.boundary)
    sim.run_steps(warmup)
    n_fluid = sc.grid.fluid_cell_count()
    t0 = time.perf_counter()
    k = 0
    while k < steps and (k == 0 or time.perf_counter() - t0 < budget_s):
        sim.advance()
        k += 1
    wall = time.perf_counter() - t0
    del sim
    return n_fluid * k / wall, k, wall


def numba_check(res=(1024, 2048), steps=3):
    """The stock reference (wbflow, Numba, installed unmodified in
    baseline/_ref) and the port on the same bounded sample, at all host
    threads and at workers=1: validates the port's speed relative to the
    reference's own CPU path (timestepper.py:213-217 cells_per_second)."""
    ref_dir = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref_dir, "wbflow")):
        return {"unavailable": "baseline/_ref not installed"}
    os.environ.setdefault("NUMBA_CACHE_DIR", os.path.join("/tmp", "wb_numba_cache"))
    sys.path.insert(0, ref_dir)
    try:
        from wbflow import timestepper as TS
        from wbflow.grid import BoundaryCondition as RBC, BoundarySpec as RBS
    except Exception as e:  # numba missing etc.
        return {"unavailable": f"cannot import the reference: {e}"}
    from paper_1806_04960_b200.scenarios import build_scenario
    sc = build_scenario("wall-impact", res)
    conv = lambda c: RBC(c.kind, c.state, c.segment)  # noqa: E731
    b = sc.boundary
    rb = RBS(conv(b.left), conv(b.right), conv(b.bottom), conv(b.top))
    n_fluid = sc.grid.fluid_cell_count()
    cores = os.cpu_count() or 1
    out = {"grid": list(res), "steps": steps, "unit": UNIT}
    for label, w in (("all_threads", cores), ("workers_1", 1)):
        t_jit = time.perf_counter()
        sim = TS.Simulation(sc.grid, sc.params, sc.q0, rb, cfl=0.45, workers=w)
        sim.advance()  # JIT compile (first call) + warm-up
        t0 = time.perf_counter()
        for _ in range(steps):
            sim.advance()
        wall = time.perf_counter() - t0
        out[f"numba_{label}"] = n_fluid * steps / wall
        if label == "all_threads":
            out["numba_setup_and_jit_s"] = t0 - t_jit
        del sim
        v, k, wall = oracle_window(res, 1, steps, w, 1e9)
        out[f"port_{label}"] = v
    out["port_over_numba_all_threads"] = out["port_all_threads"] / out["numba_all_threads"]
    out["port_over_numba_workers_1"] = out["port_workers_1"] / out["numba_workers_1"]
    out["cores"] = cores
    return out


def cpu_baseline(args, res, budget_s=20.0):
    """Reference algorithm on the host cores over a bounded sample of the SAME
    workload and window as the GPU line (the slab, W warm-up steps, then up to
    K steps within ~budget_s)."""
    cores = os.cpu_count() or 1
    v, k, wall = oracle_window(res, args.warmup, args.steps, cores, budget_s)
    return {"value": v, "unit": UNIT, "cores": cores, "kind": "port",
            "cpu_model": cpu_model(),
            "sample": f"wall-impact {res[0]}x{res[1]} (the bench slab), steps "
                      f"{args.warmup + 1}-{args.warmup + k} after {args.warmup} untimed "
                      f"warm-up steps, {wall:.1f} s, C restatement of the reference "
                      f"(oracle/, bit-identical to it), {cores} OpenMP threads"}


def run_reference(args):
    """--impl reference: the reference algorithm on the host CPU on the same
    workload and step window as our arm (N = 1); rank 0 only under torchrun,
    where it runs one GPU's slab of the weak-scaling grid."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    nx, ny = slab()
    from paper_1806_04960_b200.grid import build_grid  # noqa: F401  (package import check)
    from paper_1806_04960_b200.scenarios import build_scenario
    n_fluid = build_scenario("wall-impact", (nx, ny)).grid.fluid_cell_count()
    cores = os.cpu_count() or 1
    v, k, wall = oracle_window((nx, ny), args.warmup, args.steps, cores, 240.0)
    base = {"value": v, "unit": UNIT, "cores": cores, "kind": "port",
            "cpu_model": cpu_model(),
            "sample": f"wall-impact {nx}x{ny}: steps {args.warmup + 1}-{args.warmup + k} "
                      f"after {args.warmup} untimed warm-up steps ({wall:.1f} s), C "
                      f"restatement of the reference (oracle/, bit-identical to it), "
                      f"{cores} OpenMP threads"}
    if os.environ.get("WB_BENCH_NUMBA", "1") != "0":
        base["numba_check"] = numba_check()
    line = {"metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
            "steps": k, "warmup": args.warmup, "ms_per_step": wall / k * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": v / PUBLISHED,
            "dtype": "f64", "data": "synthetic", "impl": "reference",
            "config": bench_config(nx, ny, n_fluid, 1),
            "cpu_baseline": base,
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    if args.gpus > 1:
        line["config"]["note"] = ("one GPU's slab of the weak-scaling grid: the full "
                                  f"{nx * args.gpus}x{ny} grid needs "
                                  f"{nx * args.gpus * ny * 560 / 2**30:.0f} GiB of host memory")
    print(json.dumps(line), flush=True)


def run_ours(args):
    import torch
    from paper_1806_04960_b200 import _lib
    from paper_1806_04960_b200.scenarios import build_scenario
    from paper_1806_04960_b200.timestepper import Simulation
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world > 1:
        return run_ours_distributed(args)
    if args.gpus != 1:
        sys.stderr.write("bench.py: --gpus > 1 needs torchrun (one process per GPU); "
                         "running the single-GPU benchmark\n")
        args.gpus = 1
    dev = 0
    torch.cuda.set_device(dev)
    nx, ny = slab()
    sc = build_scenario("wall-impact", (nx, ny))
    n_fluid = sc.grid.fluid_cell_count()
    # the timed run starts from the initial condition built on the device
    # (bit-identical to sc.q0, tests/test_gpu_ic.py); the e2e leg below
    # uploads the host copy through the public API
    sim = Simulation.from_scenario(sc, device=dev)
    L = sim._L
    stream = torch.cuda.Stream(device=dev)
    _lib.check(L.wb_set_stream(sim._h, ctypes_void(stream.cuda_stream)), "wb_set_stream")
    sim.run_steps(args.warmup, chunk=args.warmup)
    # ---- timed region: K steps, device-side loop in CUDA-graph chunks ----
    clocks = ClockSampler(dev)
    clocks.start()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    sim.run_steps(args.steps, chunk=max(d for d in range(1, 17) if args.steps % d == 0))
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    clk = clocks.stop()
    ms_step = ms / args.steps
    value = n_fluid * args.steps / (ms * 1e-3)
    # per step reset_counters, k_step, prefinalize, finalize; one set_run per wb_run call
    launches = 4 * args.steps + 1
    # ---- kernel-level roofline: k_step timed alone with CUDA events ----
    import ctypes
    md, mst, mtot = ctypes.c_double(), ctypes.c_double(), ctypes.c_double()
    _lib.check(L.wb_profile_steps(sim._h, 5, ctypes.byref(md), ctypes.byref(mst),
                                  ctypes.byref(mtot)), "wb_profile_steps")
    wc = sim.work_counters()
    F = flops_per_step(n_fluid, wc["n_second_order"], wc["x_faces"], wc["y_faces"])
    tf = ctypes.c_double()
    _lib.check(L.wb_fp64_peak(dev, ctypes.byref(tf)), "wb_fp64_peak")
    fp64_achieved = F / (mst.value * 1e-3) / 1e12
    peaks = measured_peaks()
    hbm_peak = peaks.get("hbm_gbs", 6650.0)
    hbm_achieved = HBM_BYTES_PER_CELL * n_fluid / (mst.value * 1e-3) / 1e9
    t_hbm = HBM_BYTES_PER_CELL * n_fluid / (hbm_peak * 1e9)
    t_fp64 = F / (tf.value * 1e12)
    traffic, ncu = committed_traffic(nx, ny)
    roof = {"bound": "fp64" if t_fp64 >= t_hbm else "hbm",
            "achieved": fp64_achieved if t_fp64 >= t_hbm else hbm_achieved,
            "peak": tf.value if t_fp64 >= t_hbm else hbm_peak,
            "unit": "TFLOP/s" if t_fp64 >= t_hbm else "GB/s",
            "traffic": traffic,
            "kernel": "k_step (fused reconstruct + x/y faces + update)",
            "kernel_ms": mst.value, "pipeline_ms": mtot.value,
            "note": "detection of q^{n+1} is fused into k_step (ordered row-segment chain)",
            "share_of_step": mst.value / mtot.value if mtot.value else None,
            "flop_per_step": F, "counters": wc,
            "fp64_peak_source": "measured DFMA microbenchmark (wb_fp64_peak), burst",
            "hbm": {"achieved": hbm_achieved, "peak": hbm_peak, "unit": "GB/s",
                    "frac": hbm_achieved / hbm_peak,
                    "bytes_per_cell": HBM_BYTES_PER_CELL},
            "fp64": {"achieved": fp64_achieved, "peak": tf.value, "unit": "TFLOP/s",
                     "frac": fp64_achieved / tf.value},
            # hardware view of the same kernel from the committed ncu capture:
            # exact IEEE divisions cost ~9 FP64-pipe instructions per flop
            "ncu": ncu}
    roof["frac"] = roof["achieved"] / roof["peak"]
    # ---- end to end through the public API with host buffers ----
    q_host = torch.empty((nx, ny, 5), dtype=torch.float64, pin_memory=True).numpy()
    q_host[...] = sc.q0
    out_host = torch.empty((nx, ny, 5), dtype=torch.float64, pin_memory=True).numpy()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    sim.q = q_host                      # H2D of the state
    for _ in range(args.steps):
        sim.advance()                   # per step: dt + status read back
    sim.get_state(out=out_host)         # D2H of the result
    e2e_wall = time.perf_counter() - t0
    state_bytes = nx * ny * 5 * 8
    e2e = {"value": n_fluid * args.steps / e2e_wall, "unit": UNIT,
           "h2d_bytes_per_step": state_bytes / args.steps,
           "d2h_bytes_per_step": state_bytes / args.steps + 32 + 96,
           "api": "Simulation(q0 host) -> advance() x K -> sim.q (host)"}
    # ---- developed flow: the same K steps from a state 300 steps further on
    # (more solved x-faces, gas "dust" exercising the exact-replay path);
    # the state is advanced outside the timed region ----
    dev_line = None
    if not args.no_developed:
        sim.q = q_host                  # back to q0 (pinned host copy), t = 0
        sim.t, sim.step_count = 0.0, 0
        sim.run_steps(300, chunk=20)
        torch.cuda.synchronize()
        c0 = sim.work_counters()["replays"]
        e0.record(stream)
        sim.run_steps(args.steps, chunk=max(d for d in range(1, 17) if args.steps % d == 0))
        e1.record(stream)
        torch.cuda.synchronize()
        dms = e0.elapsed_time(e1)
        wcd = sim.work_counters()
        dev_line = {"start_step": sim.step_count - args.steps, "steps": args.steps,
                    "ms_per_step": dms / args.steps,
                    "value": n_fluid * args.steps / (dms * 1e-3), "unit": UNIT,
                    "counters_last_step": {k: wcd[k] for k in ("n_second_order", "x_faces",
                                                               "y_faces")},
                    "exact_replays": wcd["replays"] - c0}
    base = cpu_baseline(args, (nx, ny)) if not args.no_cpu else None
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": value / PUBLISHED,
            "dtype": "f64", "data": "synthetic",
            "config": bench_config(nx, ny, n_fluid, 1),
            "parallelism": f"x-slab dp{args.gpus}",
            "roofline": roof, "cpu_baseline": base, "e2e": e2e, "gpu_launches": launches,
            "developed": dev_line, "clocks": clk}
    print(json.dumps(line), flush=True)



def run_ours_distributed(args):
    """N > 1 ranks under torchrun, one GPU each: the wall-impact x-slab of
    4096 x 16384 cells per rank, global grid (4096 N) x 16384 (weak scaling).
    K steps of the multi-rank driver (NCCL halo send/recv + one MAX all-reduce
    per step), device time = max over ranks of the CUDA-event time on each
    rank's stream.  WB_DIST_BACKEND=gloo (host-staged collectives) exists only
    to exercise this path with several ranks on one GPU; it is not a
    benchmark configuration."""
    import ctypes
    import torch
    import torch.distributed as dist
    from paper_1806_04960_b200.distributed import (DeviceSlab, DistributedSimulation,
                                                   slab_bounds, stored_range)
    from paper_1806_04960_b200.scenarios import build_scenario
    rank = int(os.environ["RANK"])
    world = int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    dev = local % torch.cuda.device_count()
    torch.cuda.set_device(dev)
    backend = os.environ.get("WB_DIST_BACKEND", "nccl")
    if backend == "nccl":
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{dev}"))
    else:
        dist.init_process_group(backend)
    nx, ny = slab()[0] * world, slab()[1]
    i0, i1 = slab_bounds(nx, world, rank)
    lo, hi = stored_range(nx, i0, i1)
    sc = build_scenario("wall-impact", (nx, ny), columns=(lo, hi))
    # this rank's columns built on the device (bit-identical to sc.q0)
    be = DeviceSlab(sc.grid, sc.params, None, lo, sc.boundary, 0.45, i0, i1, dev, ic=sc.ic)
    sim = DistributedSimulation(be, sc.grid)
    sim.run_steps(args.warmup)
    # the timed loop replays a CUDA graph of `chunk` steps (NCCL); capture it
    # (and run those steps) before the timed region
    chunk = max(d for d in range(1, 17) if args.steps % d == 0)
    sim.enqueue_steps(chunk)
    clocks = ClockSampler(",".join(str(d) for d in range(min(world, torch.cuda.device_count())))
                          ) if rank == 0 else None
    if clocks:
        clocks.start()
    torch.cuda.synchronize()
    dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(be.stream)
    for _ in range(args.steps // chunk):
        sim.enqueue_steps(chunk)
    graphs_used = sim.use_graphs
    halo_mode, overlapped = sim.halo, sim.overlap
    e1.record(be.stream)
    torch.cuda.synchronize()
    dist.barrier()
    clk = clocks.stop() if clocks else None

    def allmax(x):
        t = torch.tensor([float(x)], dtype=torch.float64,
                         device=f"cuda:{dev}" if backend == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    ms = allmax(e0.elapsed_time(e1))
    s = sim._sync()
    sim._check(s)
    n_fluid = int(np.count_nonzero(np.asarray(sc.grid.mask)))
    value = n_fluid * args.steps / (ms * 1e-3)
    # kernel roofline on this rank's slab (k_step timed alone, after the timed region)
    n2, ex, ey = s["counters"]
    md, mst, mtot = ctypes.c_double(), ctypes.c_double(), ctypes.c_double()
    be._lib.check(be.L.wb_profile_steps(be.h, 5, ctypes.byref(md), ctypes.byref(mst),
                                        ctypes.byref(mtot)), "wb_profile_steps")
    tf = ctypes.c_double()
    be._lib.check(be.L.wb_fp64_peak(dev, ctypes.byref(tf)), "wb_fp64_peak")
    F = flops_per_step(be.n_fluid, n2, ex, ey)
    fp64 = F / (mst.value * 1e-3) / 1e12
    # end to end through the slab API with host buffers: upload each rank's
    # columns (pinned), K steps, download the owned columns; max over ranks
    q_host = torch.empty(sc.q0.shape, dtype=torch.float64, pin_memory=True).numpy()
    q_host[...] = sc.q0
    del sim, be
    torch.cuda.empty_cache()
    dist.barrier()
    t0 = time.perf_counter()
    be2 = DeviceSlab(sc.grid, sc.params, q_host, lo, sc.boundary, 0.45, i0, i1, dev)
    sim2 = DistributedSimulation(be2, sc.grid)
    sim2.run_steps(args.steps, check_every=args.steps)
    out = be2.owned_state()
    wall = allmax(time.perf_counter() - t0)
    if rank == 0:
        state_bytes = sc.q0.nbytes * world
        roof = {"bound": "fp64", "achieved": fp64, "peak": tf.value, "unit": "TFLOP/s",
                "frac": fp64 / tf.value, "traffic": committed_traffic(*slab())[0],
                "kernel": "k_step on rank 0's slab, timed alone (wb_profile_steps)",
                "kernel_ms": mst.value, "flop_per_step": F,
                "counters": {"n_second_order": n2, "x_faces": ex, "y_faces": ey,
                             "n_fluid": be2.n_fluid}}
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
                "higher_is_better": True, "scaling": "weak", "vs_baseline": value / PUBLISHED,
                "dtype": "f64", "data": "synthetic",
                "config": bench_config(nx, ny, n_fluid, world),
                "parallelism": f"x-slab dp{world}, "
                               + ("halo stored into the neighbours over peer memory (CUDA IPC)"
                                  if halo_mode == "peer" else f"{backend} halo send/recv")
                               + f" + one {backend} MAX all-reduce per step"
                               + (", edge strips overlapped" if overlapped else "")
                               + (", CUDA graph of the step sequence" if graphs_used else ""),
                # per overlapped step: set_run, reset_counters, the edge strips
                # (k_step_push, which stores the halo into the peers, or k_step),
                # k_detect_cols, k_step (interior), prefinalize, finalize, and for
                # the collective halo k_pack_halo + k_unpack_halo
                "gpu_launches": (7 if halo_mode == "peer" else 9) * args.steps,
                "roofline": roof, "cpu_baseline": None,
                "e2e": {"value": n_fluid * args.steps / wall, "unit": UNIT,
                        "h2d_bytes_per_step": state_bytes / args.steps,
                        "d2h_bytes_per_step": out.nbytes * world / args.steps,
                        "api": "DeviceSlab(q host) -> DistributedSimulation.run_steps(K) -> "
                               "owned_state() (host), max over ranks"},
                "clocks": clk}
        print(json.dumps(line), flush=True)
    dist.barrier()
    dist.destroy_process_group()

def ctypes_void(p):
    import ctypes
    return ctypes.c_void_p(p)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU baseline leg")
    ap.add_argument("--no-developed", action="store_true",
                    help="skip the developed-flow window (steps 300-K..300)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
