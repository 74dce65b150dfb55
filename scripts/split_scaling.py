"""Single-GPU emulation of the multi-GPU partition, row strips AND 2-D blocks.

    python scripts/split_scaling.py c5 [c4 c3 ...] [--gs 2,4,8]

For every G and every factorisation G = gr x gc, the largest block a rank would own
(window rows of P0/gr, window columns of P1/gc, plus n0 - 1 / n1 - 1 halo rows /
columns) is transformed by K1 from a strided view of the config's input (what rank 0
computes on; the other ranks compute on a packed copy of the same shape), CUDA
events, L2 flushed, best of 3.  Efficiency t(1) / (G t_block) is the compute-only
strong scaling; the scatter is modelled from the bytes rank 0 sends at the measured
770 GB/s peer rate (B200_PROFILING.md), serial and pipelined (compute starts on a
first piece of 1/8 of the block's window rows; that launch pair is timed too).
Environment overrides (SWDFT2D_K1_*) apply as usual; they are echoed in each line.
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1707_08213_b200.partition import block_plan, piece_bounds  # noqa: E402
from paper_1707_08213_b200.tree2d import _OUT_DTYPES, _precision_code, forward_into  # noqa: E402
from paper_1707_08213_b200.workloads import CONFIGS  # noqa: E402

PEER_GBS = 770.0


def timed(fn, flush, reps=3):
    ts = []
    for _ in range(reps):
        flush.fill_(1.0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) / 1e3)
    return min(ts)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="*", default=["c4"])
    ap.add_argument("--gs", default="2,4,8")
    a = ap.parse_args()
    env = {k: v for k, v in os.environ.items() if k.startswith("SWDFT2D_")}
    flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
    for name in a.configs:
        cfg = CONFIGS[name]
        prec = _precision_code(cfg.precision, None)
        x = torch.from_numpy(cfg.generate()).cuda()
        esz = x.element_size()
        out = torch.empty((cfg.P0, cfg.P1, cfg.n0, cfg.n1), dtype=_OUT_DTYPES[prec], device="cuda")
        forward_into(x, cfg.m0, cfg.m1, out, prec=prec)
        t1 = timed(lambda: forward_into(x, cfg.m0, cfg.m1, out, prec=prec), flush)
        print(json.dumps({"config": name, "G": 1, "t1_ms": t1 * 1e3, "env": env}), flush=True)
        for G in (int(g) for g in a.gs.split(",")):
            for gr in (d for d in range(1, G + 1) if G % d == 0):
                gc = G // gr
                plan = block_plan(cfg.P0, cfg.P1, cfg.m0, cfg.m1, gr, gc)
                big = max(plan, key=lambda p: (p[1] - p[0]) * (p[3] - p[2]))
                a0, b0, a1, b1, rb, re, cb, ce = big
                if b0 <= a0 or b1 <= a1:
                    continue
                view = x[rb:re, cb:ce]
                o = out.view(-1)[:(b0 - a0) * (b1 - a1) * cfg.n0 * cfg.n1].view(
                    b0 - a0, b1 - a1, cfg.n0, cfg.n1)
                run = lambda: forward_into(view, cfg.m0, cfg.m1, o, prec=prec)  # noqa: E731
                run()
                tb = timed(run, flush)
                wb = piece_bounds(b0 - a0, 0.125, 2)

                def two():
                    for c in range(len(wb) - 1):
                        forward_into(view, cfg.m0, cfg.m1, o[wb[c]:wb[c + 1]], prec=prec,
                                     p0_begin=wb[c], p0_end=wb[c + 1])

                two()
                t2 = timed(two, flush)
                send = sum((p[5] - p[4]) * (p[7] - p[6]) for g, p in enumerate(plan) if g) * esz
                first = sum((min(p[5] - p[4], piece_bounds(p[1] - p[0], 0.125, 2)[1] + cfg.n0 - 1))
                            * (p[7] - p[6]) for g, p in enumerate(plan) if g and p[1] > p[0]) * esz
                ts, tf = send / (PEER_GBS * 1e9), first / (PEER_GBS * 1e9)
                print(json.dumps({
                    "config": name, "G": G, "gr": gr, "gc": gc, "block": [b0 - a0, b1 - a1],
                    "block_ms": tb * 1e3, "two_piece_ms": t2 * 1e3,
                    "compute_efficiency": t1 / (G * tb),
                    "scatter_bytes": send, "scatter_ms_at_770GBps": ts * 1e3,
                    "efficiency_serial_scatter": t1 / (G * (tb + ts)),
                    "efficiency_pipelined": t1 / (G * (t2 + tf)),
                    "env": env}), flush=True)
        del x, out
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
