"""Benchmark of the batch 2D tree SWDFT hot path on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c4] [--impl ours|reference]

One "step" = one pass of the hot path over the whole workload: the 2D SWDFT of
the config's full input array, all P0 x P1 windows, output resident in HBM.
Default workload: config 4 (4096x4096 f32 image-like array, 16x16 windows,
4081x4081x16x16 complex64 = 34.2 GB), the config BASELINE.json quotes at
1/2/4/8 GPUs.  Prints ONE JSON line (rank 0).

  value      output coefficients / s, device-timed (CUDA events on the launching
             stream), input resident in HBM, output preallocated; L2 flushed
             (256 MiB write) between steps, outside the timed events
  e2e        the same metric through the public API (tree_swdft_2d) from a
             pinned host numpy-backed input to the full coefficient array in
             pinned host memory: H2D + compute + D2H of every coefficient, per step
  roofline   HBM bytes (algorithmic: output written + input read) / kernel time
             vs the measured copy bandwidth in MEASURED_PEAKS.json
  cpu_baseline  the C restatement of the reference (oracle/, all host threads)
             on the first window rows of the same config (rank 0, N=1 only)

N > 1 (torchrun, one process per GPU, NCCL), --scaling strong (default): ONE
workload partitioned into gr x gc blocks of window rows x window columns (gr = N,
gc = 1 are the north star's window-row strips; the split is measured once on rank 0
per shape and broadcast, partition.choose_split; --split forces one); rank 0 holds
the input in HBM and each step = pipelined scatter of the input blocks with their
halos (NCCL send/recv from rank 0, piece-major: every rank's first chunk first; a
receiver's pieces alternate between two streams) + every rank's block of the
transform; value = coefficients / (max over ranks of the step time).  The line's "strong" object adds the scatter alone, the
compute alone and an in-run N=1 time of the same workload on rank 0, with
E(N) = t(1) / (N t(N)).  --scaling weak: every rank transforms its own
config-sized workload (generated locally) with no data-path collective.

--impl reference: times the CPU reference path (the oracle's C restatement of
the reference's levels-outer tree, all host threads) on a bounded sample of the
same workload, rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "2D SWDFT output coeffs/sec & HBM write GB/s (% peak), 1/2/4/8 B200 vs CPU ref"
UNIT = "coef/s"
FALLBACK_HBM_GBS = 6650.0  # B200_PROFILING.md fallback, used only if MEASURED_PEAKS.json is absent


def env_int(name, default):
    v = os.environ.get(name)
    return int(v) if v not in (None, "") else default


def host_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def measured_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy test)"
    except (OSError, KeyError, ValueError):
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


def ncu_traffic(config: str, precision: str):
    """dram bytes (read + write) per full launch of the dominant kernel, from the committed
    ncu capture of this config AND precision (profiles/ncu_summary.json "<config>/<prec>");
    None when no such full-launch capture exists."""
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(p) as f:
            d = json.load(f)
        e = d.get(f"{config}/{precision}")
        return None if e is None else float(e["dram_bytes_per_launch"])
    except (OSError, KeyError, ValueError):
        return None


class ClockSampler:
    """Samples SM clock + throttle reasons with NVML while the timed region runs."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
        0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
        0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
        0x100: "display_clock_setting",
    }

    def __init__(self, index: int):
        self.samples, self.reasons, self.max_mhz = [], 0, None
        self._stop = threading.Event()
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:  # noqa: BLE001 - NVML is optional evidence
            self.nv = None
        self.t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                self.reasons |= int(self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h))
            except Exception:  # noqa: BLE001
                pass
            self._stop.wait(0.005)

    def __enter__(self):
        if self.nv is not None:
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.nv is not None:
            self.t.join()

    def summary(self):
        if self.nv is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml_unavailable"]}
        reasons = [n for bit, n in self.REASONS.items() if self.reasons & bit and n != "gpu_idle"]
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": reasons, "samples": len(self.samples)}


def cpu_reference_rate(cfg, rows: int, reps: int, threads: int):
    """Coefficients/s of the oracle's C restatement of the reference (levels-outer,
    complex128, `threads` host threads) on window rows [0, rows) of the config."""
    import oracle

    oracle.build()
    try:  # the reference keeps the whole lattice in memory; bound it by the host's RAM
        import psutil

        cap = min(1 << 36, psutil.virtual_memory().available // 3)
    except ImportError:
        cap = 1 << 33
    x = cfg.generate(rows=rows + cfg.n0 - 1)
    times = []
    for _ in range(reps):
        t0 = time.perf_counter()
        out = oracle.tree2d(x, cfg.m0, cfg.m1, threads=threads, max_lattice_bytes=cap)
        times.append(time.perf_counter() - t0)
    coefs = out.size
    del out
    return coefs / statistics.median(times), times, coefs


def numpy_reference_rate(cfg, rows: int, threads: int):
    """Coefficients/s of the UNMODIFIED reference (swdft.tree2d.tree_swdft_2d, numpy,
    staged into baseline/_ref by scripts/stage_reference.sh) on window rows [0, rows) of
    the config, `threads` as its own thread-pool argument.  None if it is not staged."""
    ref = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isfile(os.path.join(ref, "swdft", "tree2d.py")):
        return None
    if ref not in sys.path:
        sys.path.insert(0, ref)
    from swdft import core as rcore
    from swdft import tree2d as rtree

    x = cfg.generate(rows=rows + cfg.n0 - 1)
    spec = rcore.WindowSpec((cfg.m0, cfg.m1))
    t0 = time.perf_counter()
    r = rtree.tree_swdft_2d(x, spec, threads=threads, budget=1 << 42)
    t = time.perf_counter() - t0
    coefs = r.values.size
    del r
    return {"value": coefs / t, "unit": UNIT, "cores": threads, "seconds": t,
            "sample": f"window rows [0,{rows}) of {cfg.name} ({coefs} coefficients)"}


def cpu_context(cfg, rows_port: int, rows_numpy: int):
    """BASELINE.md's CPU plan as context next to cpu_baseline: the C port at T=1 and the
    reference's own numpy code at T=1 and T=all cores (smaller sample: it is ~15x slower)."""
    ctx = {"cpu_model": cpu_model(), "host_cores": host_cores()}
    rate, t, coefs = cpu_reference_rate(cfg, rows_port, 1, 1)
    ctx["port_1_thread"] = {"value": rate, "unit": UNIT, "cores": 1, "seconds": t[0],
                            "sample": f"window rows [0,{rows_port}) of {cfg.name} ({coefs} "
                                      "coefficients), oracle/swdft2d_oracle.c"}
    for name, th in (("numpy_reference_1_thread", 1), ("numpy_reference_all_cores", host_cores())):
        try:
            r = numpy_reference_rate(cfg, rows_numpy, th)
        except Exception as e:  # noqa: BLE001 - context only; say why it is missing
            r = {"unavailable": f"{type(e).__name__}: {e}"}
        ctx[name] = r if r is not None else {
            "unavailable": "reference not staged (scripts/stage_reference.sh)"}
    return ctx


def run_reference(args, cfg, rank):
    if rank != 0:
        return
    threads = host_cores()
    rows = args.ref_rows
    for _ in range(args.warmup):
        cpu_reference_rate(cfg, rows, 1, threads)
    times = []
    coefs = 0
    for _ in range(args.steps):
        rate, t, coefs = cpu_reference_rate(cfg, rows, 1, threads)
        times.append(t[0])
    tot = sum(times)
    value = coefs * len(times) / tot
    sample = (f"window rows [0,{rows}) of {cfg.name} ({coefs} coefficients, input rows "
              f"[0,{rows + cfg.n0 - 1})), complex128, C restatement of the reference's "
              f"levels-outer tree (oracle/swdft2d_oracle.c), {threads} threads on {cpu_model()}")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * tot / len(times), "higher_is_better": True,
        "scaling": args.scaling,
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded, BASELINE.json recipe)",
        "config": {"workload": cfg.name, "desc": cfg.desc, "sample_window_rows": rows},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": sample,
                         "numpy_reference_all_cores": numpy_reference_rate(
                             cfg, min(rows, 32), threads)},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def make_flush(dev):
    """Two 256 MiB buffers (> the 126 MB L2): one written, one read by every flush."""
    import torch

    return (torch.empty(64 << 20, dtype=torch.float32, device=dev),
            torch.ones(64 << 20, dtype=torch.float32, device=dev))


def flush_l2(buf):
    """Write 256 MiB (evicts the step's input and output from L2), then read another
    256 MiB, so the step starts with a clean L2: after the write alone L2 held ~126 MB
    of DIRTY flush lines whose write-back the next step's first stores paid for
    (config 2: 0.0922 -> 0.0881 ms, profiles/flush_effect_r02.jsonl)."""
    buf[0].fill_(1.0)
    buf[1].sum()
    # ... then ~0.2 ms of device-side spinning (no memory traffic: L2 stays as flushed), so
    # the host has certainly queued the start event and the step behind it before the device
    # gets there.  Without it a slow host (the flush takes only ~90 us) leaves the device idle
    # inside the interval: config 2 read 0.1065 ms instead of 0.086-0.088 on two boxes where
    # the bench followed the test suite (profiles/c2_timing_r02.jsonl, "sleep" rows).
    import torch

    if hasattr(torch.cuda, "_sleep"):
        torch.cuda._sleep(400000)


def run_ours(args, cfg, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    from paper_1707_08213_b200 import WindowSpec, tree_swdft_2d
    from paper_1707_08213_b200 import _lib
    from paper_1707_08213_b200.partition import (block_plan, choose_pieces, choose_split,
                                                  pipelined_block_forward)
    from paper_1707_08213_b200.tree2d import _OUT_DTYPES, _precision_code, forward_into

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    spec = WindowSpec((cfg.m0, cfg.m1))
    prec = _precision_code(args.precision or cfg.precision, None)
    odt = _OUT_DTYPES[prec]
    stream = torch.cuda.current_stream(dev)
    flush = make_flush(dev)  # 2 x 256 MiB > 126 MB L2

    # N > 1 modes: "weak" (default) — every rank transforms its own full workload (its
    # own share of window rows of an N-times taller array, generated locally): no
    # data-path collective, per-GPU work fixed.  "strong" — the north-star partition of
    # ONE workload: window-row strips scattered from rank 0 over NCCL (pipelined).
    strips = (world > 1 or args.strips) and args.scaling == "strong"
    x_np = cfg.generate() if (rank == 0 or not strips) else None
    xdt = {"float32": torch.float32, "float64": torch.float64, "complex64": torch.complex64,
           "complex128": torch.complex128}[cfg.dtype]
    P0, P1, n0, n1 = cfg.P0, cfg.P1, cfg.n0, cfg.n1
    x_full = torch.from_numpy(x_np).to(dev) if x_np is not None else None
    # strong: the partition (gr x gc blocks of window rows x window columns) and the
    # scatter's piece count are measured once on rank 0 and broadcast (choose_split);
    # --split GRxGC forces one
    split, pieces, lead, split_table = (1, 1), 1, 0, []
    if strips:
        if args.split:
            split = tuple(int(v) for v in args.split.split("x"))
            pieces = choose_pieces((cfg.N0, cfg.N1), cfg.m0, cfg.m1, np.dtype(cfg.dtype).itemsize,
                                   8 if prec == _lib.PREC_FP32 else 16, world)
        else:
            ch = choose_split(x_full, (cfg.N0, cfg.N1), cfg.m0, cfg.m1, prec, world,
                              np.dtype(cfg.dtype).itemsize)
            split, pieces, lead = tuple(ch["split"]), ch["pieces"], ch.get("lead", 0)
            split_table = ch["table"]
    a, b, c0, c1, rb, re, cb, ce = block_plan(P0, P1, cfg.m0, cfg.m1, *split,
                                              lead)[rank if strips else 0]
    out = torch.empty((b - a, c1 - c0, n0, n1), dtype=odt, device=dev)
    recv = torch.empty((re - rb, ce - cb), dtype=xdt, device=dev) if x_full is None else None

    def compute(local, w0, w1):
        # on torch's current stream: the receive path alternates pieces between streams
        forward_into(local, cfg.m0, cfg.m1, out[w0:w1], prec=prec, p0_begin=w0, p0_end=w1)

    def step():
        # strong: the partitioner's pipelined scatter — every block travels from rank 0 in
        # in-order chunks and each rank starts on its first chunk on arrival
        if strips:
            pipelined_block_forward(x_full if rank == 0 else None, (cfg.N0, cfg.N1), cfg.m0,
                                    cfg.m1, split, xdt, dev, compute, recv=recv, pieces=pieces,
                                    lead=lead)
        elif b > a:
            compute(x_full, 0, b - a)

    if world > 1:
        dist.barrier()
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    graph = None
    if not strips and not args.no_graph:
        # one step = one K1 launch; replaying it from a CUDA graph keeps host-side
        # launch overhead out of the device-timed region
        graph = torch.cuda.CUDAGraph()
        cap = torch.cuda.Stream(dev)  # graphs are captured on a side stream
        cap.wait_stream(stream)
        with torch.cuda.graph(graph, stream=cap):
            forward_into(x_full, cfg.m0, cfg.m1, out, prec=prec, stream=cap)
        stream.wait_stream(cap)
        for _ in range(2):
            graph.replay()
        torch.cuda.synchronize()
    run_step = graph.replay if graph is not None else step

    times = []
    with ClockSampler(local_rank) as clk:
        for _ in range(args.steps):
            if world > 1:
                dist.barrier()
            torch.cuda.synchronize()
            # the L2 flush is queued just ahead of the start event, so the device is still
            # busy with it while the step is submitted: the events time the step's device
            # work, not the host's submission latency
            flush_l2(flush)
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            run_step()
            e1.record(stream)
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1) / 1e3)
    t_local = sum(times)
    if world > 1:
        tt = torch.tensor([t_local], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_job = float(tt.item())
    else:
        t_job = t_local
    step_s = t_job / args.steps
    units = cfg.coefficients * (world if (world > 1 and not strips) else 1)
    value = units / step_s
    out_bpc = 8 if prec == _lib.PREC_FP32 else 16
    bytes_alg = cfg.coefficients * out_bpc + cfg.in_bytes

    # one step at N=1 is exactly one K1 launch (graph replay), so the kernel's average
    # launch duration over the timed region is the step time
    kern_s = step_s

    peak, peak_src = measured_peak()
    achieved = bytes_alg / kern_s / 1e9 if not strips else (
        ((b - a) * P1 * n0 * n1 * out_bpc + (re - rb) * cfg.N1 * np.dtype(cfg.dtype).itemsize)
        / (t_local / args.steps) / 1e9)

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": step_s * 1e3, "higher_is_better": True,
        "scaling": args.scaling, "vs_baseline": None,
        "dtype": "f32" if prec == _lib.PREC_FP32 else "f64",
        "data": "synthetic (seeded, BASELINE.json recipe; see paper_1707_08213_b200/workloads.py)",
        "config": {"workload": cfg.name, "desc": cfg.desc, "N0": cfg.N0, "N1": cfg.N1,
                   "window": [n0, n1], "coefficients": cfg.coefficients,
                   "output_bytes": cfg.coefficients * out_bpc,
                   "l2": "L2 flushed before every timed step (then a 0.2 ms device-side spin so host "
                         "submission stays outside the interval): 256 MiB written, then another "
                         "256 MiB read so L2 starts clean (queued ahead of the start event, "
                         "outside the timed interval); output >> L2 as well",
                   "parallelism": (f"blocks{split[0]}x{split[1]} (window rows x window "
                                   "columns, NCCL scatter from rank 0)" if strips else
                                   f"replicas{world} (each rank its own full workload, no "
                                   "data-path collective)" if world > 1 else "single"),
                   "scatter_pieces": pieces, "lead": lead,
                   **({"split_choice": [{k: (list(v) if isinstance(v, tuple) else v)
                                         for k, v in r.items()} for r in split_table]}
                      if split_table else {})},
        "hbm_write_gbs": units * out_bpc / step_s / 1e9,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak,
                     "traffic": ncu_traffic(cfg.name, "fp32" if prec == _lib.PREC_FP32 else "fp64"),
                     "peak_source": peak_src,
                     # BASELINE.md's target is quoted against the 8.0 TB/s nominal HBM peak
                     "nominal_peak": 8000.0, "frac_nominal": achieved / 8000.0,
                     "bytes_per_launch": bytes_alg, "kernel_ms": kern_s * 1e3},
        "kernel": dict(_lib.stream_kernel_info(cfg.m0, cfg.m1, prec), name="K1 k1_stream_kernel"),
        "clocks": clk.summary(),
        # K1 launches per step: one at N=1; up to `pieces` per rank under the pipelined scatter
        "gpu_launches": args.steps * pieces,
    }

    if strips and not args.no_strong_detail:
        line["strong"] = strong_detail(args, cfg, rank, world, dev, stream, x_full, recv, out,
                                       prec, pieces, step_s, split, lead, graph_free=True)

    # e2e through the public API from pinned host memory
    if not args.no_e2e:
        if not strips:
            line["e2e"] = e2e_host(args, cfg, x_np, dev, spec, odt, out, world)
        else:
            out = None
            torch.cuda.empty_cache()
            line["e2e"] = e2e_sharded(args, cfg, x_np, dev, spec, xdt, prec, rank, world, split,
                                      pieces, lead)
    if world == 1 and not args.no_others:
        graph = out = None
        torch.cuda.empty_cache()
        line["other_configs"] = other_configs(args, cfg, dev, flush, stream)
    if world == 1 and not args.no_cpu:
        rate, t, coefs = cpu_reference_rate(cfg, args.ref_rows, 3, host_cores())
        line["cpu_baseline"] = {
            "value": rate, "unit": UNIT, "cores": host_cores(), "kind": "port",
            "sample": f"window rows [0,{args.ref_rows}) of {cfg.name} ({coefs} coefficients), "
                      f"median of 3, C restatement of the reference levels-outer tree "
                      f"(oracle/swdft2d_oracle.c, complex128) on {cpu_model()}"}
        if not args.no_cpu_context:
            line["cpu_baseline"]["context"] = cpu_context(cfg, args.ref_rows,
                                                          min(args.ref_rows, 32))
    if rank == 0:
        print(json.dumps(line), flush=True)


def strong_detail(args, cfg, rank, world, dev, stream, x_full, recv, out, prec, pieces, step_s,
                  split, lead=0, graph_free=True):
    """Strong-scaling breakdown (max over ranks, device-timed, L2 flushed): the pipelined
    scatter alone (compute replaced by nothing), each rank's block transform alone (input
    already resident), and t(1) = the whole workload on rank 0 alone in the same run, so
    E(N) = t(1) / (N t(N)) needs no other run."""
    import torch
    import torch.distributed as dist

    from paper_1707_08213_b200.partition import block_plan, pipelined_block_forward
    from paper_1707_08213_b200.tree2d import _OUT_DTYPES, forward_into

    flush = make_flush(dev)
    a, b, c0, c1, rb, re, cb, ce = block_plan(cfg.P0, cfg.P1, cfg.m0, cfg.m1, *split, lead)[rank]
    xdt = x_full.dtype if x_full is not None else recv.dtype
    local = x_full[rb:re, cb:ce] if x_full is not None else recv

    def timed(fn, reps):
        ts = []
        for _ in range(reps):
            dist.barrier()
            torch.cuda.synchronize()
            flush_l2(flush)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            fn()
            e1.record(stream)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) / 1e3)
        t = torch.tensor([statistics.median(ts)], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def scatter_only():
        pipelined_block_forward(x_full if rank == 0 else None, (cfg.N0, cfg.N1), cfg.m0, cfg.m1,
                                split, xdt, dev, lambda *_: None, recv=recv, pieces=pieces, lead=lead)

    def compute_only():
        if b > a and c1 > c0:
            forward_into(local, cfg.m0, cfg.m1, out, prec=prec, p0_begin=0, p0_end=b - a,
                         stream=stream)

    reps = max(3, min(args.steps, 5))
    t_scatter = timed(scatter_only, reps)
    t_compute = timed(compute_only, reps)
    # t(1): rank 0 transforms the whole workload alone (the other ranks idle)
    full = None
    if rank == 0:
        full = torch.empty((cfg.P0, cfg.P1, cfg.n0, cfg.n1), dtype=_OUT_DTYPES[prec], device=dev)
        forward_into(x_full, cfg.m0, cfg.m1, full, prec=prec, stream=stream)

    def one_gpu():
        if rank == 0:
            forward_into(x_full, cfg.m0, cfg.m1, full, prec=prec, stream=stream)

    t1 = timed(one_gpu, reps)
    del full
    torch.cuda.empty_cache()
    return {"t1_ms": t1 * 1e3, "tN_ms": step_s * 1e3, "efficiency_in_run": t1 / (world * step_s),
            "scatter_only_ms": t_scatter * 1e3, "compute_only_ms": t_compute * 1e3,
            "scatter_pieces": pieces, "split": list(split), "lead": lead,
            "note": "max over ranks, median of %d; t1 = whole workload on rank 0 alone, same run" % reps}


def other_configs(args, main_cfg, dev, flush, stream):
    """The other BASELINE configs on the same GPU in the same run (kernel-only, device
    timed, L2 flushed between steps): value, write rate and roofline fraction each."""
    import torch

    from paper_1707_08213_b200 import _lib
    from paper_1707_08213_b200.tree2d import _OUT_DTYPES, _precision_code, forward_into
    from paper_1707_08213_b200.workloads import CONFIGS

    peak, _ = measured_peak()
    res = {}
    # every other config at its BASELINE precision, plus the headline config in fp64 — the
    # reference's own precision (complex128, bitwise equal to the reference)
    runs = [(name, c, c.precision) for name, c in CONFIGS.items() if name != main_cfg.name]
    if main_cfg.precision != "fp64":
        # first: measured after config 5 (18.8 ms steps at the 1000 W power cap) the fp64
        # line read 403 vs 430 Gcoef/s standalone on the same box
        runs.insert(0, (f"{main_cfg.name}_fp64", main_cfg, "fp64"))
    for name, c, pname in runs:
        prec = _precision_code(pname, None)
        x = torch.from_numpy(c.generate()).to(dev)
        out = torch.empty((c.P0, c.P1, c.n0, c.n1), dtype=_OUT_DTYPES[prec], device=dev)
        for _ in range(3):
            forward_into(x, c.m0, c.m1, out, prec=prec, stream=stream)
        g = torch.cuda.CUDAGraph()  # same timing method as the headline: one launch per replay
        cap = torch.cuda.Stream(dev)
        cap.wait_stream(stream)
        with torch.cuda.graph(g, stream=cap):
            forward_into(x, c.m0, c.m1, out, prec=prec, stream=cap)
        stream.wait_stream(cap)
        g.replay()
        ts = []
        # short steps take more samples: on a fresh box single config-2 samples read 0.099-
        # 0.115 ms against a 0.086-0.088 median (profiles/c2_timing_r02.jsonl), and a median
        # of 5 once landed on them
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        g.replay()
        e1.record(stream)
        torch.cuda.synchronize()
        reps = 5 if e0.elapsed_time(e1) > 2.0 else 25
        with ClockSampler(dev.index or 0) as clk:
            for _ in range(reps):
                torch.cuda.synchronize()
                flush_l2(flush)  # ahead of the start event (see run_ours)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                g.replay()
                e1.record(stream)
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1) / 1e3)
        t = statistics.median(ts)
        alg = c.algorithmic_bytes(precision=pname)
        traffic = ncu_traffic(c.name, pname)
        res[name] = {"desc": c.desc, "dtype": "f32" if prec == _lib.PREC_FP32 else "f64",
                     "value": c.coefficients / t, "unit": UNIT, "kernel_ms": t * 1e3,
                     "samples": reps, "clocks": clk.summary(),
                     "ms_min_max": [round(min(ts) * 1e3, 4), round(max(ts) * 1e3, 4)],
                     "hbm_write_gbs": c.coefficients * (16 if pname == "fp64" else 8) / t / 1e9,
                     "roofline": {"bound": "hbm", "achieved": alg / t / 1e9, "peak": peak,
                                  "unit": "GB/s", "frac": alg / t / 1e9 / peak,
                                  "frac_nominal": alg / t / 1e9 / 8000.0, "traffic": traffic,
                                  "traffic_over_alg": None if traffic is None else traffic / alg},
                     "roofline_frac": alg / t / 1e9 / peak,
                     "kernel": dict(_lib.stream_kernel_info(c.m0, c.m1, prec),
                                    schedule=_lib.k1_schedule(c.N0, c.N1, c.m0, c.m1, prec)["mode"])}
        del g, x, out
        torch.cuda.empty_cache()
    return res


def e2e_sharded(args, cfg, x_np, dev, spec, xdt, prec, rank, world, split, pieces, lead=0):
    """N > 1: rank 0's pinned host input -> H2D -> tree_swdft_2d_sharded (pipelined NCCL
    scatter + K1 per block) -> every rank copies its block of coefficients to its own
    pinned host buffer (each GPU's own PCIe link).  Time = max over ranks."""
    import torch
    import torch.distributed as dist

    from paper_1707_08213_b200.partition import block_plan, tree_swdft_2d_sharded

    a, b, c0, c1 = block_plan(cfg.P0, cfg.P1, cfg.m0, cfg.m1, *split, lead)[rank][:4]
    x_pin = torch.from_numpy(x_np).pin_memory() if rank == 0 else None
    from paper_1707_08213_b200.tree2d import _OUT_DTYPES

    host_out = torch.empty((b - a, c1 - c0, cfg.n0, cfg.n1), dtype=_OUT_DTYPES[prec],
                           pin_memory=True)
    stream = torch.cuda.current_stream(dev)
    times = []
    for i in range(args.warmup + args.e2e_steps):
        dist.barrier()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        xd = x_pin.to(dev, non_blocking=True) if rank == 0 else None
        sh = tree_swdft_2d_sharded(xd, spec, shape=(cfg.N0, cfg.N1), dtype=xdt,
                                   precision="fp32" if prec == 0 else "fp64", budget=1 << 62,
                                   split=split, pieces=pieces, lead=lead)
        host_out.copy_(sh.values, non_blocking=True)
        e1.record(stream)
        torch.cuda.synchronize()
        del sh, xd
        if i >= args.warmup:
            times.append(e0.elapsed_time(e1) / 1e3)
    t = torch.tensor([statistics.mean(times)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    d2h = torch.tensor([host_out.numel() * host_out.element_size()], dtype=torch.float64,
                       device=dev)
    dist.all_reduce(d2h)
    s = float(t.item())
    return {"value": cfg.coefficients / s, "unit": UNIT,
            "h2d_bytes_per_step": int(cfg.in_bytes), "d2h_bytes_per_step": int(d2h.item()),
            "ms_per_step": s * 1e3, "steps": len(times),
            "path": "rank 0 pinned host input -> tree_swdft_2d_sharded -> each rank's block "
                    "to its own pinned host buffer; max over ranks"}


def e2e_host(args, cfg, x_np, dev, spec, odt, out_dev, world=1):
    """tree_swdft_2d(host x) -> device -> full coefficient array back in pinned host memory
    (every rank its own workload when world > 1; time = max over ranks)."""
    import torch

    from paper_1707_08213_b200 import tree_swdft_2d

    need = out_dev.numel() * out_dev.element_size() + x_np.nbytes
    if world > 1:
        # every rank pins its own full output: make sure the host can hold N of them
        import psutil

        ok = torch.tensor([float(psutil.virtual_memory().available > 1.25 * world * need)],
                          dtype=torch.float64, device=dev)
        torch.distributed.all_reduce(ok, op=torch.distributed.ReduceOp.MIN)
        full = bool(ok.item())
    else:
        full = True
    if os.environ.get("SWDFT2D_BENCH_E2E_RESIDENT") == "1":  # exercise the fallback (tests)
        full = False
    x_pin = torch.from_numpy(x_np).pin_memory()
    host_out = torch.empty(out_dev.shape, dtype=odt, pin_memory=True) if full else None
    stream = torch.cuda.current_stream(dev)
    times = []
    for i in range(args.warmup + args.e2e_steps if full else 0):
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        tree_swdft_2d(x_pin, spec, budget=1 << 62, device=dev, host_out=host_out)
        e1.record(stream)
        torch.cuda.synchronize()
        if i >= args.warmup:
            times.append(e0.elapsed_time(e1) / 1e3)
    s = statistics.mean(times) if full else 0.0
    if world > 1 and full:
        tt = torch.tensor([s], dtype=torch.float64, device=dev)
        torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
        s = float(tt.item())
    # the same call with the coefficients left resident in HBM (a GPU consumer's view):
    # H2D of the input, the transform, and a D2H read of one window's coefficients
    win = torch.empty(out_dev.shape[2:], dtype=odt, pin_memory=True)
    rtimes = []
    for i in range(args.warmup + args.e2e_steps):
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        res = tree_swdft_2d(x_pin, spec, budget=1 << 62, device=dev, out=out_dev)
        win.copy_(res.values[-1, -1], non_blocking=True)
        e1.record(stream)
        torch.cuda.synchronize()
        if i >= args.warmup:
            rtimes.append(e0.elapsed_time(e1) / 1e3)
    r = statistics.mean(rtimes)
    if world > 1:
        tt = torch.tensor([r], dtype=torch.float64, device=dev)
        torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
        r = float(tt.item())
    resident = {"value": world * cfg.coefficients / r, "unit": UNIT, "ms_per_step": r * 1e3,
                "h2d_bytes_per_step": int(x_pin.numel() * x_pin.element_size()),
                "d2h_bytes_per_step": int(win.numel() * win.element_size()),
                "path": "same call, coefficients left in HBM, one window read back"}
    # the reference's own calling convention: numpy in, a FRESH numpy array out (allocation
    # and first-touch page faults inside the interval; host wall clock).  The pageable
    # destination is filled through the library's pinned staging ring and worker threads.
    fresh = None
    import psutil

    if full and world == 1 and psutil.virtual_memory().available > 1.25 * need:
        ftimes = []
        for _ in range(2):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            r_np = tree_swdft_2d(x_np, spec, budget=1 << 62, device=dev, to_host=True)
            ftimes.append(time.perf_counter() - t0)
            assert isinstance(r_np.values, np.ndarray)
            del r_np
        fresh = {"value": cfg.coefficients / min(ftimes), "unit": UNIT,
                 "ms_per_call": min(ftimes) * 1e3, "calls": len(ftimes),
                 "path": "tree_swdft_2d(numpy input, to_host=True): fresh pageable numpy result, "
                         "host wall clock incl. allocation and page faults"}
    if not full:
        # N full pinned outputs do not fit the host: report the resident variant (input
        # H2D + transform + a D2H read of one window per rank), saying so
        return dict(resident, steps=len(rtimes),
                    full_d2h_skipped=f"host RAM < 1.25 x {world} x {need / 1e9:.0f} GB "
                                     "pinned outputs; value is the resident variant")
    return {"value": world * cfg.coefficients / s, "unit": UNIT,
            "h2d_bytes_per_step": int(x_pin.numel() * x_pin.element_size()),
            "d2h_bytes_per_step": int(host_out.numel() * host_out.element_size()),
            "ms_per_step": s * 1e3, "steps": len(times),
            "ms_all": [round(t * 1e3, 2) for t in times],
            "path": "tree_swdft_2d(pinned host input, host_out=pinned) = ONE C-ABI call, "
                    "swdft2d_forward_host: input H2D, strips computed in a 4-slot device ring "
                    "and copied D2H on 2 copy streams while later strips compute",
            "fresh_output": fresh, "resident": resident}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c4", choices=["c1", "c2", "c3", "c4", "c5"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--ref-rows", type=int, default=None,
                    help="window rows of the CPU sample (default: 64 for c5 as BASELINE.json "
                         "says, else 128; c1/c2 are small enough to run whole)")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-cpu-context", action="store_true",
                    help="skip the T=1 port and numpy-reference timings next to cpu_baseline")
    ap.add_argument("--no-graph", action="store_true")
    ap.add_argument("--no-others", action="store_true", help="skip the other-configs summary")
    ap.add_argument("--strips", action="store_true",
                    help="run the strip path (pipelined scatter + per-strip K1) even at N=1 "
                         "(under torchrun; exercises the N>1 code on one GPU)")
    ap.add_argument("--split", default=None,
                    help="N>1 strong: force the GRxGC block partition (default: measured on "
                         "rank 0 per shape, partition.choose_split)")
    ap.add_argument("--no-strong-detail", action="store_true",
                    help="N>1 strong: skip the scatter-only / compute-only / t(1) breakdown")
    ap.add_argument("--scaling", default="strong", choices=["weak", "strong"],
                    help="N>1: strong = ONE workload in window-row strips scattered from rank 0 "
                         "over NCCL, the north-star partition (default); weak = every rank its "
                         "own workload, no data-path collective")
    ap.add_argument("--precision", default=None, choices=[None, "fp32", "fp64"],
                    help="override the config's precision (fp64 = DAG-exact complex128)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "ours" else args.warmup

    from paper_1707_08213_b200.workloads import CONFIGS

    cfg = CONFIGS[args.config]
    if args.ref_rows is None:
        args.ref_rows = cfg.P0 if cfg.name in ("c1", "c2") else 64 if cfg.name == "c5" else 128
    world = env_int("WORLD_SIZE", 1)
    rank = env_int("RANK", 0)
    local_rank = env_int("LOCAL_RANK", 0)
    if args.impl == "reference":
        run_reference(args, cfg, rank)
        return
    dist_on = world > 1 or (args.strips and "RANK" in os.environ)
    if args.strips and not dist_on:
        ap.error("--strips needs a torchrun launch")
    if dist_on:
        import torch
        import torch.distributed as dist

        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    try:
        run_ours(args, cfg, rank, world, local_rank)
    finally:
        if dist_on:
            import torch.distributed as dist

            dist.destroy_process_group()


if __name__ == "__main__":
    main()
