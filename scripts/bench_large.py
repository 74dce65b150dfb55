"""Large-window path (KR + KC) rates: windows beyond K1's 64, plus the separable path
forced on config 4's 16 x 16 for comparison with K1.  CUDA-graph replay, median of 5,
L2 flushed before each launch; float32 input, fp32 and fp64 precision."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1707_08213_b200.tree2d import _OUT_DTYPES, forward_into  # noqa: E402

dev = torch.device("cuda", 0)
flush = torch.empty(64 << 20, dtype=torch.float32, device=dev)
cases = [((512, 512), (7, 7), "auto"), ((1024, 1024), (8, 6), "auto"), ((1024, 1024), (6, 8), "auto"),
         ((4096, 1024), (7, 3), "auto"), ((640, 2048), (3, 10), "auto"), ((2048, 640), (10, 3), "auto"),
         ((4096, 4096), (4, 4), "separable"), ((4096, 4096), (4, 4), "auto")]
for (N0, N1), (m0, m1), kern in cases:
    for prec in (0, 1):
        n0, n1 = 1 << m0, 1 << m1
        P0, P1 = N0 - n0 + 1, N1 - n1 + 1
        coefs = P0 * P1 * n0 * n1
        if coefs * (16 if prec else 8) > 120e9:
            continue
        x = torch.from_numpy(np.random.default_rng(m0 + m1).standard_normal((N0, N1)).astype(np.float32)).to(dev)
        out = torch.empty((P0, P1, n0, n1), dtype=_OUT_DTYPES[prec], device=dev)
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
            ts.append(e0.elapsed_time(e1) / 1e3)
        t = float(np.median(ts))
        print(json.dumps({"N": [N0, N1], "window": [n0, n1], "kernel": kern,
                          "prec": "fp64" if prec else "fp32", "ms": t * 1e3,
                          "gcoef_s": coefs / t / 1e9,
                          "write_tbs": coefs * (16 if prec else 8) / t / 1e12}), flush=True)
        del out, g
        torch.cuda.empty_cache()
