"""Probe: would column pieces pipeline the scatter better than row pieces?

    python scripts/colpiece_probe.py c3 c4 c5 [--gs 4,8]

Same timeline emulation as scripts/split_scaling.py (a link stream sleeps until rank 0's
egress at 770 GB/s would have delivered each piece), for the largest receiver block of the
split choose_split picks per config:
  rpipe2  two ROW pieces (1/8 of the window rows first), two streams — the library's
          receive path; the second piece re-runs up to n0 - 1 warm-up rows;
  cpipe2  two COLUMN pieces (1/8 of the window columns first), two streams: nothing is
          recomputed (K1 column blocks are independent), the second piece is the full-width
          block (the first piece's columns travel twice, no packing on the source).
Each piece writes its own temporary output (same bytes as an output with a row stride).
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

SPLITS = {("c3", 8): (8, 1), ("c4", 8): (4, 2), ("c5", 8): (4, 2),
          ("c3", 4): (4, 1), ("c4", 4): (2, 2), ("c5", 4): (2, 2)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="*", default=["c3"])
    ap.add_argument("--gs", default="8")
    ap.add_argument("--reps", type=int, default=7)
    a = ap.parse_args()
    fa = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
    fb = torch.ones(64 << 20, dtype=torch.float32, device="cuda")
    torch.cuda._sleep(1000)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    torch.cuda._sleep(2_000_000)
    e1.record()
    torch.cuda.synchronize()
    ns_per_cycle = e0.elapsed_time(e1) * 1e6 / 2_000_000
    main_s, side, link = torch.cuda.current_stream(), torch.cuda.Stream(), torch.cuda.Stream()

    def timed(fn):
        ts = []
        for _ in range(a.reps):
            torch.cuda.synchronize()
            fa.fill_(1.0)
            fb.sum()
            torch.cuda._sleep(200000)
            s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s0.record(main_s)
            fn(s0)
            s1.record(main_s)
            torch.cuda.synchronize()
            ts.append(s0.elapsed_time(s1) / 1e3)
        return statistics.median(ts)

    def arrivals(s0, times):
        link.wait_event(s0)
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
        n0, n1 = cfg.n0, cfg.n1
        out = torch.empty((cfg.P0, cfg.P1, n0, n1), dtype=_OUT_DTYPES[prec], device="cuda")
        forward_into(x, cfg.m0, cfg.m1, out, prec=prec)
        t1 = timed(lambda s0: forward_into(x, cfg.m0, cfg.m1, out, prec=prec))
        flat = out.view(-1)
        for G in (int(g) for g in a.gs.split(",")):
            gr, gc = SPLITS.get((name, G), (G, 1))
            plan = block_plan(cfg.P0, cfg.P1, cfg.m0, cfg.m1, gr, gc)
            big = max(plan[1:], key=lambda p: (p[1] - p[0]) * (p[3] - p[2]))
            a0, b0, a1, b1, rb, re, cb, ce = big
            R, Cw = b0 - a0, b1 - a1
            view = x[rb:re, cb:ce]
            wr = piece_bounds(R, 0.125, 2)
            wc = piece_bounds(Cw, 0.125, 2)

            def o(rows, cols, off=0):
                return flat[off:off + rows * cols * n0 * n1].view(rows, cols, n0, n1)

            send = rfirst = cfirst = 0
            for p in plan[1:]:
                rows_in, cols_in = p[5] - p[4], p[7] - p[6]
                send += rows_in * cols_in * esz
                fr = piece_bounds(p[1] - p[0], 0.125, 2)
                rfirst += min(rows_in, fr[1] + n0 - 1) * cols_in * esz
                fc = piece_bounds(p[3] - p[2], 0.125, 2)
                cfirst += rows_in * min(cols_in, fc[1] + n1 - 1) * esz
            ts, tfr = send / NVLINK_PEER_BPS, rfirst / NVLINK_PEER_BPS
            tfc, tsc = cfirst / NVLINK_PEER_BPS, (cfirst + send) / NVLINK_PEER_BPS
            o_full = o(R, Cw)
            o_c0 = o(R, wc[1])
            o_c1 = o(R, Cw - wc[1], R * wc[1] * n0 * n1)

            def compute(s0):
                forward_into(view, cfg.m0, cfg.m1, o_full, prec=prec)

            def rpipe2(s0):
                ef, ea = arrivals(s0, [tfr, ts])
                side.wait_event(s0)
                main_s.wait_event(ef)
                forward_into(view, cfg.m0, cfg.m1, o_full[wr[0]:wr[1]], prec=prec,
                             p0_begin=wr[0], p0_end=wr[1])
                side.wait_event(ea)
                with torch.cuda.stream(side):
                    forward_into(view, cfg.m0, cfg.m1, o_full[wr[1]:wr[2]], prec=prec,
                                 p0_begin=wr[1], p0_end=wr[2])
                main_s.wait_stream(side)

            v0 = view[:, :wc[1] + n1 - 1]
            v1 = view[:, wc[1]:]

            def cpipe2(s0):
                ef, ea = arrivals(s0, [tfc, tsc])
                side.wait_event(s0)
                main_s.wait_event(ef)
                forward_into(v0, cfg.m0, cfg.m1, o_c0, prec=prec)
                side.wait_event(ea)
                with torch.cuda.stream(side):
                    forward_into(v1, cfg.m0, cfg.m1, o_c1, prec=prec)
                main_s.wait_stream(side)

            def cboth(s0):  # column pieces, no transfer: the split's own compute cost
                forward_into(v0, cfg.m0, cfg.m1, o_c0, prec=prec)
                with torch.cuda.stream(side):
                    side.wait_stream(main_s)
                    forward_into(v1, cfg.m0, cfg.m1, o_c1, prec=prec)
                main_s.wait_stream(side)

            res = {"config": name, "G": G, "split": [gr, gc], "block": [R, Cw],
                   "t1_ms": t1 * 1e3, "scatter_ms": ts * 1e3, "rfirst_ms": tfr * 1e3,
                   "cfirst_ms": tfc * 1e3, "cscatter_ms": tsc * 1e3}
            for label, fn in (("compute", compute), ("rpipe2", rpipe2), ("cpipe2", cpipe2),
                              ("ccompute", cboth)):
                fn(None) if label in ("compute", "ccompute") else None
                t = timed(fn)
                res[label + "_ms"] = t * 1e3
                res["eff_" + label] = t1 / (G * t)
            print(json.dumps(res), flush=True)
        del x, out, flat
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
