"""Single-GPU emulation of the strip partition (no NCCL, no second GPU): for G in
{1, 2, 4, 8}, time K1 on the largest strip rank g would own (input rows with halo,
its window rows), CUDA events, L2 flushed between launches.  t(1) / (G * t_max(G))
is the compute-only strong-scaling efficiency the partition allows; the scatter
(rank 0's NVLink egress) is estimated from the strip bytes at the measured 770 GB/s
peer-copy rate (B200_PROFILING.md) and reported separately."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1707_08213_b200.partition import strip_plan  # noqa: E402
from paper_1707_08213_b200.tree2d import _OUT_DTYPES, _precision_code, forward_into  # noqa: E402
from paper_1707_08213_b200.workloads import CONFIGS  # noqa: E402

PEER_GBS = 770.0

cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c4"]
prec = _precision_code(cfg.precision, None)
x = torch.from_numpy(cfg.generate()).cuda()
flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
out = torch.empty((cfg.P0, cfg.P1, cfg.n0, cfg.n1), dtype=_OUT_DTYPES[prec], device="cuda")
t1 = None
res = []
for G in (1, 2, 4, 8):
    plan = strip_plan(cfg.P0, cfg.m0, G)
    times = []
    for (a, b, rb, re) in plan:
        strip = x[rb:re]
        o = out[:b - a]
        forward_into(strip, cfg.m0, cfg.m1, o, prec=prec)
        ts = []
        for _ in range(3):
            flush.fill_(1.0)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            forward_into(strip, cfg.m0, cfg.m1, o, prec=prec)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) / 1e3)
        times.append(min(ts))
    tmax = max(times)
    # the pipelined receive splits each strip into a 1/8 piece and the rest (two launches)
    from paper_1707_08213_b200.partition import piece_bounds

    a, b, rb, re = max(plan, key=lambda p: p[1] - p[0])
    wb = piece_bounds(b - a, 0.125, 2)
    ts = []
    for _ in range(3):
        flush.fill_(1.0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for c in range(len(wb) - 1):
            forward_into(x[rb:re], cfg.m0, cfg.m1, out[wb[c]:wb[c + 1]], prec=prec,
                         p0_begin=wb[c], p0_end=wb[c + 1])
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) / 1e3)
    t_piece1 = None
    t1 = t1 or tmax
    scatter_bytes = sum((re - rb) * cfg.N1 * x.element_size() for g, (a, b, rb, re) in enumerate(plan) if g)
    t_scatter = scatter_bytes / (PEER_GBS * 1e9)
    t_two = min(ts)
    first_bytes = (wb[1] + cfg.n0 - 1) * cfg.N1 * x.element_size() * (G - 1)  # all peers' first chunks
    t_first = first_bytes / (PEER_GBS * 1e9) if G > 1 else 0.0
    res.append({"config": cfg.name, "G": G, "strip_kernel_ms_max": tmax * 1e3,
                "two_piece_ms": t_two * 1e3, "first_chunks_ms_at_770GBps": t_first * 1e3,
                "efficiency_pipelined": t1 / (G * (t_two + t_first)) if G > 1 else 1.0,
                "strip_kernel_ms_min": min(times) * 1e3,
                "compute_efficiency": t1 / (G * tmax),
                "scatter_bytes": scatter_bytes, "scatter_ms_at_770GBps": t_scatter * 1e3,
                "efficiency_with_serial_scatter": t1 / (G * (tmax + t_scatter))})
    print(json.dumps(res[-1]), flush=True)
