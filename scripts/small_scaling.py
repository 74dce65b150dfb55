"""Device time of K1 vs the number of window rows (full width), from CUDA-graph replays.

    python scripts/small_scaling.py [--config c2] [--rows 8,16,...]

The intercept of time vs rows is the fixed cost of one launch (launch latency, ramp,
warm-up rows, drain); the slope is the streaming rate.
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_1707_08213_b200.tree2d import _OUT_DTYPES, forward_into  # noqa: E402
from paper_1707_08213_b200.workloads import CONFIGS  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--rows", default="1,8,16,32,64,128,256,497")
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--precision", default=None)
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    s = torch.cuda.current_stream(dev)
    cfg = CONFIGS[a.config]
    prec = 1 if (a.precision or cfg.precision) == "fp64" else 0
    x = torch.from_numpy(cfg.generate()).to(dev)
    flush = torch.empty(64 << 20, dtype=torch.float32, device=dev)
    for rows in [int(r) for r in a.rows.split(",")]:
        rows = min(rows, cfg.P0)
        out = torch.empty((rows, cfg.P1, cfg.n0, cfg.n1), dtype=_OUT_DTYPES[prec], device=dev)
        forward_into(x, cfg.m0, cfg.m1, out, prec=prec, p0_end=rows, stream=s)
        g = torch.cuda.CUDAGraph()
        cap = torch.cuda.Stream(dev)
        cap.wait_stream(s)
        with torch.cuda.graph(g, stream=cap):
            forward_into(x, cfg.m0, cfg.m1, out, prec=prec, p0_end=rows, stream=cap)
        s.wait_stream(cap)
        g.replay()
        torch.cuda.synchronize()
        ts = []
        for _ in range(a.reps):
            flush.fill_(1.0)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            g.replay()
            e1.record(s)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        t = sorted(ts)[len(ts) // 2]
        coefs = rows * cfg.P1 * cfg.n0 * cfg.n1
        print(json.dumps({"config": a.config, "rows": rows, "ms": round(t, 4),
                          "gcoef_s": round(coefs / t / 1e6, 1),
                          "write_tbs": round(coefs * out.element_size() / t / 1e9, 3)}), flush=True)
        del out, g


if __name__ == "__main__":
    main()
