"""Single-GPU emulation of the multi-GPU partition: row strips AND 2-D blocks, with the
scatter's arrival times replayed on the device.

    python scripts/split_scaling.py c5 [c4 c3 ...] [--gs 2,4,8]

For every G and every factorisation G = gr x gc, the largest block a rank would own
(window rows of P0/gr, window columns of P1/gc, plus the n0 - 1 / n1 - 1 halo rows /
columns) is transformed by K1 from a strided view of the config's input.  The scatter
from rank 0 is replayed as a timeline: a "link" stream sleeps (torch.cuda._sleep,
calibrated) until the bytes rank 0 sends would have left its NVLink egress at the
measured 770 GB/s peer rate (B200_PROFILING.md) — every peer's first piece first
(piece-major, partition.py), then the remainders — and records an arrival event per
piece; the block's compute waits on those events.  Strategies:
  serial    one launch after the whole scatter;
  pipe1     2 pieces (1/8 of the window rows first), both launches on one stream;
  pipe2     2 pieces on two streams, so the second launch's CTAs fill SMs as the
            first's retire (partition.py's receive path);
  compute   the block alone (no transfer);
  protocol  what partition.py does: the source sends everything and then computes its own
            band shortened by tune_split's `lead`; the largest receiver runs pipe2 on the
            re-balanced plan; the step is the slower of the two (eff_protocol_serial: one
            piece, every rank ~ scatter + block).
Efficiency t(1) / (G t), t(1) = the whole config on one GPU, CUDA events, L2 flushed
(write + read) ahead of the start event, median of 5.
"""
import argparse
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1707_08213_b200.partition import NVLINK_PEER_BPS, block_plan, piece_bounds  # noqa: E402
from paper_1707_08213_b200.tree2d import _OUT_DTYPES, _precision_code, forward_into  # noqa: E402
from paper_1707_08213_b200.workloads import CONFIGS  # noqa: E402


def calibrate_sleep():
    """ns per torch.cuda._sleep cycle."""
    torch.cuda._sleep(1000)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    torch.cuda._sleep(2_000_000)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e6 / 2_000_000


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="*", default=["c4"])
    ap.add_argument("--gs", default="2,4,8")
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    env = {k: v for k, v in os.environ.items() if k.startswith("SWDFT2D_")}
    fa = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
    fb = torch.ones(64 << 20, dtype=torch.float32, device="cuda")
    ns_per_cycle = calibrate_sleep()
    main_s = torch.cuda.current_stream()
    side = torch.cuda.Stream()
    link = torch.cuda.Stream()

    def timed(fn):
        ts = []
        for _ in range(a.reps):
            torch.cuda.synchronize()
            fa.fill_(1.0)
            fb.sum()
            torch.cuda._sleep(200000)  # the host enqueues everything before e0 runs
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(main_s)
            fn(e0)
            e1.record(main_s)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) / 1e3)
        return statistics.median(ts)

    def arrivals(e0, times):
        """Events recorded on the link stream at the given seconds after e0."""
        link.wait_event(e0)
        evs, t = [], 0.0
        with torch.cuda.stream(link):
            for at in times:
                if at > t:
                    torch.cuda._sleep(int((at - t) * 1e9 / ns_per_cycle))
                    t = at
                ev = torch.cuda.Event()
                ev.record(link)
                evs.append(ev)
        return evs

    for name in a.configs:
        cfg = CONFIGS[name]
        prec = _precision_code(cfg.precision, None)
        x = torch.from_numpy(cfg.generate()).cuda()
        esz = x.element_size()
        out = torch.empty((cfg.P0, cfg.P1, cfg.n0, cfg.n1), dtype=_OUT_DTYPES[prec], device="cuda")
        forward_into(x, cfg.m0, cfg.m1, out, prec=prec)
        t1 = timed(lambda e0: forward_into(x, cfg.m0, cfg.m1, out, prec=prec))
        print(json.dumps({"config": name, "G": 1, "t1_ms": t1 * 1e3, "env": env}), flush=True)
        for G in (int(g) for g in a.gs.split(",")):
            for gr in (d for d in range(1, G + 1) if G % d == 0):
                gc = G // gr
                plan = block_plan(cfg.P0, cfg.P1, cfg.m0, cfg.m1, gr, gc)
                big = max(plan[1:], key=lambda p: (p[1] - p[0]) * (p[3] - p[2]))
                a0, b0, a1, b1, rb, re, cb, ce = big
                if b0 <= a0 or b1 <= a1:
                    continue
                view = x[rb:re, cb:ce]
                o = out.view(-1)[:(b0 - a0) * (b1 - a1) * cfg.n0 * cfg.n1].view(
                    b0 - a0, b1 - a1, cfg.n0, cfg.n1)
                wb = piece_bounds(b0 - a0, 0.125, 2)
                # bytes rank 0 sends: every peer's block; first pieces go out first
                send = first = 0
                for p in plan[1:]:
                    if p[1] <= p[0] or p[3] <= p[2]:
                        continue
                    rows_in, cols_in = p[5] - p[4], p[7] - p[6]
                    send += rows_in * cols_in * esz
                    f = piece_bounds(p[1] - p[0], 0.125, 2)
                    first += min(rows_in, f[1] + cfg.n0 - 1) * cols_in * esz
                ts, tf = send / NVLINK_PEER_BPS, first / NVLINK_PEER_BPS

                def piece(c, st):
                    with torch.cuda.stream(st):
                        forward_into(view, cfg.m0, cfg.m1, o[wb[c]:wb[c + 1]], prec=prec,
                                     p0_begin=wb[c], p0_end=wb[c + 1])

                def compute(e0):
                    forward_into(view, cfg.m0, cfg.m1, o, prec=prec)

                def serial(e0):
                    (ev,) = arrivals(e0, [ts])
                    main_s.wait_event(ev)
                    forward_into(view, cfg.m0, cfg.m1, o, prec=prec)

                def pipe1(e0):
                    e_first, e_all = arrivals(e0, [tf, ts])
                    main_s.wait_event(e_first)
                    piece(0, main_s)
                    main_s.wait_event(e_all)
                    piece(1, main_s)

                def pipe2(e0):
                    e_first, e_all = arrivals(e0, [tf, ts])
                    side.wait_event(e0)
                    main_s.wait_event(e_first)
                    piece(0, main_s)
                    side.wait_event(e_all)
                    piece(1, side)
                    main_s.wait_stream(side)

                compute(None)
                res = {"config": name, "G": G, "gr": gr, "gc": gc, "block": [b0 - a0, b1 - a1],
                       "scatter_bytes": send, "scatter_ms": ts * 1e3, "first_ms": tf * 1e3}
                for label, fn in (("compute", compute), ("serial", serial), ("pipe1", pipe1),
                                  ("pipe2", pipe2)):
                    t = timed(fn)
                    res[label + "_ms"] = t * 1e3
                    res["eff_" + label] = t1 / (G * t)
                # the library's protocol (partition.py): the source sends everything, then
                # computes its own band shortened by `lead` (tune_split's formula);
                # receivers run pipe2 on their (slightly larger) blocks
                tb = res["compute_ms"] / 1e3
                extra = 0.5 * (cfg.n0 - 1) / max(1, b0 - a0) * tb + 5e-6
                bands, blen = (gr, b0 - a0) if gr > 1 else (gc, b1 - a1)
                lam = max(0.0, (ts - tf - extra) / tb * (bands - 1) / bands)
                lead = int(round(lam * blen))
                plan_l = block_plan(cfg.P0, cfg.P1, cfg.m0, cfg.m1, gr, gc, lead)
                z = plan_l[0]
                v0 = x[z[4]:z[5], z[6]:z[7]]
                o0 = out.view(-1)[:(z[1] - z[0]) * (z[3] - z[2]) * cfg.n0 * cfg.n1].view(
                    z[1] - z[0], z[3] - z[2], cfg.n0, cfg.n1)

                def own(e0):
                    forward_into(v0, cfg.m0, cfg.m1, o0, prec=prec)

                own(None)
                t0 = timed(own) + ts
                rbig = max(plan_l[1:], key=lambda p: (p[1] - p[0]) * (p[3] - p[2]))
                view = x[rbig[4]:rbig[5], rbig[6]:rbig[7]]
                o = out.view(-1)[:(rbig[1] - rbig[0]) * (rbig[3] - rbig[2]) * cfg.n0 * cfg.n1].view(
                    rbig[1] - rbig[0], rbig[3] - rbig[2], cfg.n0, cfg.n1)
                wb = piece_bounds(rbig[1] - rbig[0], 0.125, 2)
                piece(0, main_s)
                piece(1, main_s)
                trv = timed(pipe2)
                res.update({"lead": lead, "src_ms": t0 * 1e3, "recv_ms": trv * 1e3,
                            "eff_protocol": t1 / (G * max(t0, trv)),
                            "eff_protocol_serial": t1 / (G * (ts + tb))})
                res["env"] = env
                print(json.dumps(res), flush=True)
        del x, out
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
