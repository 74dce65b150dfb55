"""Latency of K1 (stream) vs K0 (window) on small inputs (config 1 and friends), each
launch replayed from a CUDA graph, median of 200; decides the AUTO kernel for tiny work."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1707_08213_b200 import _lib  # noqa: E402
from paper_1707_08213_b200.tree2d import _OUT_DTYPES, forward_into  # noqa: E402

dev = torch.device("cuda", 0)
cases = [((64, 64), (3, 3), 1), ((64, 64), (3, 3), 0), ((32, 32), (2, 2), 1), ((128, 128), (4, 4), 1),
         ((128, 128), (4, 4), 0), ((256, 256), (3, 3), 1), ((100, 100), (6, 6), 0),
         ((100, 100), (2, 2), 1), ((512, 512), (4, 4), 0)]
for (N0, N1), (m0, m1), prec in cases:
    x = torch.from_numpy(np.random.default_rng(0).standard_normal((N0, N1))).to(dev)
    P0, P1 = N0 - (1 << m0) + 1, N1 - (1 << m1) + 1
    out = torch.empty((P0, P1, 1 << m0, 1 << m1), dtype=_OUT_DTYPES[prec], device=dev)
    res = {"shape": [N0, N1], "window": [1 << m0, 1 << m1], "prec": "fp64" if prec else "fp32"}
    for kern in ("stream", "window"):
        s = torch.cuda.Stream(dev)
        forward_into(x, m0, m1, out, prec=prec, kernel=kern, stream=s)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            forward_into(x, m0, m1, out, prec=prec, kernel=kern, stream=s)
        ts = []
        for _ in range(200):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            g.replay()
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e3)
        res[kern + "_us"] = float(np.median(ts))
    print(json.dumps(res), flush=True)
