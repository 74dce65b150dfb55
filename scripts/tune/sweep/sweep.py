"""Sweep K1 shapes (Q, TP1) for every window (n0, n1) in {4..64}^2 on a float32 array
sized for ~8 GB of complex64 output; report each variant's coef/s and the product
rule's choice.  Tuning harness (scripts/tune/sweep/_build/libsweep.so), not product code.

    python scripts/tune/sweep/sweep.py > sweep.jsonl
"""
import ctypes
import json
import math
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(HERE)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1707_08213_b200 import _lib  # noqa: E402


def rule_q(M0, M1):
    q = M0 - 2 if M0 > 2 else 0
    while q > 0 and (1 << M1) * (1 << q) > 512:
        q -= 1
    return q


def main():
    prec = int(sys.argv[1]) if len(sys.argv) > 1 else 0  # 0: fp32 variants, 1: fp64-exact
    lib = ctypes.CDLL(os.path.join(HERE, "_build", "libsweep.so"))
    lib.tune_name.restype = ctypes.c_char_p
    for name, (res, args) in _lib.SIGNATURES.items():
        getattr(lib, name).restype = res
        getattr(lib, name).argtypes = args
    dev = torch.device("cuda", 0)
    flush = torch.empty(64 << 20, dtype=torch.float32, device=dev)
    s = torch.cuda.current_stream(dev)
    by_shape = {}
    for v in range(lib.tune_count()):
        if lib.tune_m(v, 4) == prec:
            by_shape.setdefault((lib.tune_m(v, 0), lib.tune_m(v, 1)), []).append(v)
    for (m0, m1), vs in sorted(by_shape.items()):
        n0, n1 = 1 << m0, 1 << m1
        ob = 16 if prec else 8
        N = int(min(8192, max(4 * max(n0, n1), math.sqrt(8e9 / (ob * n0 * n1)))))
        x = torch.randn((N, N), device=dev, dtype=torch.float32)
        P0, P1 = N - n0 + 1, N - n1 + 1
        out = torch.empty((P0, P1, n0, n1), dtype=torch.complex128 if prec else torch.complex64,
                          device=dev)
        coefs = P0 * P1 * n0 * n1
        for v in vs:
            lib.tune_select(v)

            def launch():
                rc = lib.swdft2d_forward(x.data_ptr(), 0, N, N, N, m0, m1, prec, 1.0, 0, P0,
                                         out.data_ptr(), 1, s.cuda_stream)
                assert rc == 0, lib.swdft2d_last_error()

            launch()
            torch.cuda.synchronize()
            ts = []
            for _ in range(5):
                flush.fill_(1.0)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(s)
                launch()
                e1.record(s)
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1) / 1e3)
            t = float(np.median(ts))
            name = lib.tune_name(v).decode()
            q = int(name.split("Q=")[1].split()[0])
            tp1 = int(name.split("TP1=")[1].split()[0])
            rule_tp1 = max(1, 128 // (n1 << rule_q(m0, m1)))
            print(json.dumps({"m0": m0, "m1": m1, "N": N, "Q": q, "TP1": tp1,
                              "threads": lib.tune_m(v, 2), "gcoef_s": coefs / t / 1e9,
                              "write_tbs": coefs * ob / t / 1e12, "prec": prec,
                              "is_rule": q == rule_q(m0, m1) and tp1 == rule_tp1}), flush=True)
        del x, out
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
