"""Time the PRODUCT library's K1 for every window 4..64 x 4..64 (fp32, ~8 GB of output per
shape, median of 5, L2 flushed) — confirms the per-shape table the sweep produced."""
import json
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1707_08213_b200 import _lib  # noqa: E402
from paper_1707_08213_b200.tree2d import forward_into  # noqa: E402

dev = torch.device("cuda", 0)
flush = torch.empty(64 << 20, dtype=torch.float32, device=dev)
for m0 in range(2, 7):
    for m1 in range(2, 7):
        n0, n1 = 1 << m0, 1 << m1
        N = int(min(8192, max(4 * max(n0, n1), math.sqrt(8e9 / (8 * n0 * n1)))))
        x = torch.randn((N, N), device=dev, dtype=torch.float32)
        P0, P1 = N - n0 + 1, N - n1 + 1
        out = torch.empty((P0, P1, n0, n1), dtype=torch.complex64, device=dev)
        forward_into(x, m0, m1, out, prec=0)
        ts = []
        for _ in range(5):
            flush.fill_(1.0)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            forward_into(x, m0, m1, out, prec=0)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) / 1e3)
        t = float(np.median(ts))
        c = P0 * P1 * n0 * n1
        print(json.dumps({"n0": n0, "n1": n1, "N": N, "gcoef_s": c / t / 1e9,
                          "write_tbs": c * 8 / t / 1e12,
                          "kernel": _lib.stream_kernel_info(m0, m1, 0)}), flush=True)
        del x, out
        torch.cuda.empty_cache()
