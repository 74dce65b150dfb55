"""Time one window shape through each applicable kernel path (auto / stream / separable),
fp32 and fp64, CUDA-graph replay, median of 5, L2 flushed.

    python scripts/kernel_compare.py N0 N1 m0 m1
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1707_08213_b200.tree2d import _OUT_DTYPES, forward_into  # noqa: E402

N0, N1, m0, m1 = (int(v) for v in sys.argv[1:5])
dev = torch.device("cuda", 0)
flush = torch.empty(64 << 20, dtype=torch.float32, device=dev)
x = torch.from_numpy(np.random.default_rng(0).standard_normal((N0, N1)).astype(np.float32)).to(dev)
n0, n1 = 1 << m0, 1 << m1
P0, P1 = N0 - n0 + 1, N1 - n1 + 1
for prec in (0, 1):
    out = torch.empty((P0, P1, n0, n1), dtype=_OUT_DTYPES[prec], device=dev)
    for kern in (sys.argv[5].split(",") if len(sys.argv) > 5 else ("auto", "separable")):
        s = torch.cuda.Stream(dev)
        forward_into(x, m0, m1, out, prec=prec, kernel=kern, stream=s)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            forward_into(x, m0, m1, out, prec=prec, kernel=kern, stream=s)
        ts = []
        for _ in range(5):
            torch.cuda.synchronize()
            flush.fill_(1.0)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            g.replay()
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        t = sorted(ts)[2] / 1e3
        coefs = P0 * P1 * n0 * n1
        print(json.dumps({"N": [N0, N1], "window": [n0, n1], "prec": "fp64" if prec else "fp32",
                          "kernel": kern, "ms": t * 1e3,
                          "write_tbs": coefs * (16 if prec else 8) / t / 1e12}), flush=True)
        del g
    del out
    torch.cuda.empty_cache()
