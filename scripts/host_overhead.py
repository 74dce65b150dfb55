"""Host-side cost of one forward call, outside CUDA graphs.

    python scripts/host_overhead.py [--configs c2,c3,c4]

Per config: (1) host submission time of forward_into (perf_counter around the call
while the device is busy, so the call never waits on the GPU); (2) device time of one
call timed with events, each call preceded by a synchronize (the path a user without a
graph takes); (3) the same launch replayed from a CUDA graph.  (2) - (3) is what the
host path adds to a synchronous user's step.
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_1707_08213_b200.tree2d import _OUT_DTYPES, forward_into  # noqa: E402
from paper_1707_08213_b200.workloads import CONFIGS  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="c2,c3,c4")
    ap.add_argument("--reps", type=int, default=10)
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    s = torch.cuda.current_stream(dev)
    for name in a.configs.split(","):
        cfg = CONFIGS[name]
        prec = 1 if cfg.precision == "fp64" else 0
        x = torch.from_numpy(cfg.generate()).to(dev)
        out = torch.empty((cfg.P0, cfg.P1, cfg.n0, cfg.n1), dtype=_OUT_DTYPES[prec], device=dev)
        call = lambda: forward_into(x, cfg.m0, cfg.m1, out, prec=prec, stream=s)  # noqa: E731
        for _ in range(3):
            call()
        torch.cuda.synchronize()
        host = []
        for _ in range(a.reps):
            torch.cuda._sleep(50_000_000)  # keep the device busy: the call must not block
            t0 = time.perf_counter()
            call()
            host.append(time.perf_counter() - t0)
            torch.cuda.synchronize()
        dev_sync = []
        for _ in range(a.reps):
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            call()
            e1.record(s)
            torch.cuda.synchronize()
            dev_sync.append(e0.elapsed_time(e1))
        g = torch.cuda.CUDAGraph()
        cap = torch.cuda.Stream(dev)
        cap.wait_stream(s)
        with torch.cuda.graph(g, stream=cap):
            forward_into(x, cfg.m0, cfg.m1, out, prec=prec, stream=cap)
        s.wait_stream(cap)
        g.replay()
        torch.cuda.synchronize()
        graph = []
        for _ in range(a.reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            g.replay()
            e1.record(s)
            torch.cuda.synchronize()
            graph.append(e0.elapsed_time(e1))
        med = lambda v: sorted(v)[len(v) // 2]  # noqa: E731
        print(json.dumps({"config": name, "host_submit_us": round(med(host) * 1e6, 1),
                          "sync_call_ms": round(med(dev_sync), 4), "graph_ms": round(med(graph), 4)}),
              flush=True)
        del x, out, g
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
