"""1D tree rate by window size (the KR row-tree kernel, n = 16 .. 1024), fp32 and fp64,
CUDA-graph replay, median of 5, L2 flushed before each launch."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1707_08213_b200.tree2d import _OUT_DTYPES, forward_into  # noqa: E402

dev = torch.device("cuda", 0)
flush = torch.empty(64 << 20, dtype=torch.float32, device=dev)
N = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 20
for prec in (0, 1):
    for m in (4, 6, 7, 8, 10):
        n = 1 << m
        if N * n * (16 if prec else 8) > 150e9:  # output beyond one B200's memory
            continue
        x = torch.from_numpy(np.random.default_rng(m).standard_normal((1, N))).to(dev)
        P = N - n + 1
        out = torch.empty((1, P, 1, n), dtype=_OUT_DTYPES[prec], device=dev)
        s = torch.cuda.Stream(dev)
        forward_into(x, 0, m, out, prec=prec, stream=s)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            forward_into(x, 0, m, out, prec=prec, stream=s)
        ts = []
        for _ in range(5):
            torch.cuda.synchronize()
            flush.fill_(1.0)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            g.replay()
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) / 1e3)
        t = float(np.median(ts))
        print(json.dumps({"N": N, "n": n, "prec": "fp64" if prec else "fp32",
                          "ms": t * 1e3,
                          "gcoef_s": P * n / t / 1e9,
                          "write_tbs": P * n * (16 if prec else 8) / t / 1e12}), flush=True)
        del out, g
        torch.cuda.empty_cache()
