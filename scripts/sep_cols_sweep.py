"""Large-window path: the column trees on K1's Z-column kernel vs KC, per window.

    SWDFT2D_SEP_COLS=kc python scripts/sep_cols_sweep.py > kc.jsonl
    SWDFT2D_SEP_COLS=k1 python scripts/sep_cols_sweep.py > k1.jsonl

Windows n0 x n1 that run on the separable path (KR + column trees), float32 input sized
for ~4 GB of complex64 output, fp32 and fp64, CUDA-graph replay, L2 flushed (write + read),
median of 5.  One JSON line per (window, precision) with the env echoed.
"""
import json
import math
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1707_08213_b200.tree2d import _OUT_DTYPES, forward_into  # noqa: E402

WINDOWS = [(2, 128), (4, 128), (8, 128), (16, 128), (32, 128), (64, 128), (8, 1024), (64, 1024),
           (128, 32), (128, 64), (128, 128), (256, 16), (256, 64), (512, 8), (512, 32),
           (512, 64)]


def main():
    dev = torch.device("cuda", 0)
    fa = torch.empty(64 << 20, dtype=torch.float32, device=dev)
    fb = torch.ones(64 << 20, dtype=torch.float32, device=dev)
    env = {k: v for k, v in os.environ.items() if k.startswith("SWDFT2D_")}
    for n0, n1 in WINDOWS:
        m0, m1 = n0.bit_length() - 1, n1.bit_length() - 1
        for prec in (0, 1):
            target = 4e9 / (16 if prec else 8)  # coefficients
            pos = target / (n0 * n1)  # window positions
            P1 = max(n1, int(math.sqrt(pos)))
            P0 = max(8, int(pos // P1))
            N0, N1 = P0 + n0 - 1, P1 + n1 - 1
            x = torch.randn((N0, N1), device=dev)
            out = torch.empty((P0, P1, n0, n1), dtype=_OUT_DTYPES[prec], device=dev)
            forward_into(x, m0, m1, out, prec=prec, kernel="separable")
            g = torch.cuda.CUDAGraph()
            cap = torch.cuda.Stream(dev)
            cap.wait_stream(torch.cuda.current_stream(dev))
            with torch.cuda.graph(g, stream=cap):
                forward_into(x, m0, m1, out, prec=prec, kernel="separable", stream=cap)
            torch.cuda.current_stream(dev).wait_stream(cap)
            ts = []
            for _ in range(5):
                torch.cuda.synchronize()
                fa.fill_(1.0)
                fb.sum()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                g.replay()
                e1.record()
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1) / 1e3)
            t = statistics.median(ts)
            print(json.dumps({"window": [n0, n1], "N": [N0, N1], "prec": "fp64" if prec else "fp32",
                              "ms": t * 1e3, "write_tbs": out.numel() * out.element_size() / t / 1e12,
                              "env": env}), flush=True)
            del g, x, out
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
