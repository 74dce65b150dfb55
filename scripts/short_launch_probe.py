"""K1 on short window-row ranges (push_rows blocks, scatter pieces, host-output strips):
device time per launch and the schedule the rule picks, per config and row count.

    [SWDFT2D_K1_GUIDED=0|1] [SWDFT2D_K1_ONESHOT=0|1] [SWDFT2D_K1_STREAMK=k] \
        python scripts/short_launch_probe.py [c2 c3 c4 c5] [--rows 16,32,64,128,256]

One JSON line per (config, rows): median of 7 CUDA-event timings (L2 flushed ahead of the
start event), the write rate, and the schedule (swdft2d_k1_schedule).
"""
import argparse
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1707_08213_b200 import _lib  # noqa: E402
from paper_1707_08213_b200.tree2d import _OUT_DTYPES, _precision_code, forward_into  # noqa: E402
from paper_1707_08213_b200.workloads import CONFIGS  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="*", default=["c2", "c3", "c4", "c5"])
    ap.add_argument("--rows", default="16,32,64,128,256")
    ap.add_argument("--precision", default=None)
    a = ap.parse_args()
    env = {k: v for k, v in os.environ.items() if k.startswith("SWDFT2D_")}
    fa = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
    fb = torch.ones(64 << 20, dtype=torch.float32, device="cuda")
    for name in a.configs:
        cfg = CONFIGS[name]
        prec = _precision_code(a.precision or cfg.precision, None)
        x = torch.from_numpy(cfg.generate()).cuda()
        rmax = max(int(r) for r in a.rows.split(","))
        out = torch.empty((min(rmax, cfg.P0), cfg.P1, cfg.n0, cfg.n1), dtype=_OUT_DTYPES[prec],
                          device="cuda")
        for R in (int(r) for r in a.rows.split(",")):
            R = min(R, cfg.P0)
            a0 = (cfg.P0 - R) // 2  # a range in the middle of the array
            o = out[:R]
            forward_into(x, cfg.m0, cfg.m1, o, prec=prec, p0_begin=a0, p0_end=a0 + R)
            ts = []
            for _ in range(7):
                torch.cuda.synchronize()
                fa.fill_(1.0)
                fb.sum()
                torch.cuda._sleep(100000)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                forward_into(x, cfg.m0, cfg.m1, o, prec=prec, p0_begin=a0, p0_end=a0 + R)
                e1.record()
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1) / 1e3)
            t = statistics.median(ts)
            sch = _lib.k1_schedule(cfg.N0, cfg.N1, cfg.m0, cfg.m1, prec, a0, a0 + R)
            sch.pop("bounds", None)
            print(json.dumps({"config": name, "rows": R, "us": t * 1e6,
                              "write_tbs": o.numel() * o.element_size() / t / 1e12,
                              "schedule": sch, "env": env}), flush=True)
        del x, out
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
