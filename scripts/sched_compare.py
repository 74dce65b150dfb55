"""Time K1 under the current SWDFT2D_K1_* environment on whole configs and on the largest
block of gr x gc partitions (the block a rank would own), fp32 unless --fp64.

    SWDFT2D_K1_STREAMK=1 python scripts/sched_compare.py c2 c4 w64x32:2048x2048 --splits 1x1,8x1,4x2

One JSON line per (config, split): block shape, median ms of 7 (L2 flushed, CUDA events
behind a device sleep so host launch overhead stays outside the interval),
write TB/s, the schedule the library chose, and the env.  Run once per env setting and
compare lines (scripts/sched_sweep.sh).
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1707_08213_b200 import _lib  # noqa: E402
from paper_1707_08213_b200.partition import block_plan  # noqa: E402
from paper_1707_08213_b200.tree2d import _OUT_DTYPES, forward_into  # noqa: E402
from paper_1707_08213_b200.workloads import CONFIGS  # noqa: E402


class AdHoc:
    def __init__(self, n0, n1, N0, N1):
        self.n0, self.n1, self.N0, self.N1 = n0, n1, N0, N1
        self.m0, self.m1 = n0.bit_length() - 1, n1.bit_length() - 1
        self.P0, self.P1 = N0 - n0 + 1, N1 - n1 + 1


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="*", default=["c2"])
    ap.add_argument("--splits", default="1x1")
    ap.add_argument("--fp64", action="store_true")
    ap.add_argument("--reps", type=int, default=7)
    a = ap.parse_args()
    env = {k: v for k, v in os.environ.items() if k.startswith("SWDFT2D_")}
    prec = 1 if a.fp64 else 0
    flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
    for name in a.configs:
        if name.startswith("w"):  # w<n0>x<n1>:<N0>x<N1> — random f32 input of that shape
            win, shp = name[1:].split(":")
            cfg = AdHoc(*(int(v) for v in win.split("x")), *(int(v) for v in shp.split("x")))
            x = torch.randn((cfg.N0, cfg.N1), device="cuda")
        else:
            cfg = CONFIGS[name]
            x = torch.from_numpy(cfg.generate()).cuda()
        out = torch.empty((cfg.P0, cfg.P1, cfg.n0, cfg.n1), dtype=_OUT_DTYPES[prec], device="cuda")
        for sp in a.splits.split(","):
            gr, gc = (int(v) for v in sp.split("x"))
            plan = block_plan(cfg.P0, cfg.P1, cfg.m0, cfg.m1, gr, gc)
            a0, b0, a1, b1, rb, re, cb, ce = max(plan, key=lambda p: (p[1] - p[0]) * (p[3] - p[2]))
            view = x[rb:re, cb:ce]
            o = out.view(-1)[:(b0 - a0) * (b1 - a1) * cfg.n0 * cfg.n1].view(
                b0 - a0, b1 - a1, cfg.n0, cfg.n1)
            forward_into(view, cfg.m0, cfg.m1, o, prec=prec)
            ts = []
            for _ in range(a.reps):
                flush.fill_(1.0)
                torch.cuda._sleep(300000)  # ~150 us: the host enqueues the call before e0 runs
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                forward_into(view, cfg.m0, cfg.m1, o, prec=prec)
                e1.record()
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1) / 1e3)
            t = float(np.median(ts))
            info = _lib.k1_schedule(re - rb, ce - cb, cfg.m0, cfg.m1, prec, 0, b0 - a0)
            info.pop("bounds")
            print(json.dumps({"config": name, "split": sp, "block": [b0 - a0, b1 - a1],
                              "ms": t * 1e3, "min_ms": min(ts) * 1e3,
                              "write_tbs": o.numel() * o.element_size() / t / 1e12,
                              "schedule": info, "env": env}), flush=True)
        del x, out
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
