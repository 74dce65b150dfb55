"""Time Z-column K1 variants (scripts/tune/_build/libtune.so) on the large-window path.

    SWDFT2D_SEP_COLS=k1 python scripts/tune/tune_colz.py N0 N1 m0 m1

Selects each COLZ variant of the harness in turn (the registry's m1 = 0, variant 2 slot)
and times swdft2d_forward on an N0 x N1 float32 input (separable path: KR + the column
trees), fp32 variants in fp32 and fp64 variants in fp64; CUDA events, L2 flushed.
"""
import ctypes
import json
import os
import statistics
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
import torch  # noqa: E402

from paper_1707_08213_b200 import _lib  # noqa: E402


def main():
    N0, N1, m0, m1 = (int(v) for v in sys.argv[1:5])
    lib = ctypes.CDLL(os.path.join(HERE, "_build", "libtune.so"))
    lib.tune_name.restype = ctypes.c_char_p
    for name, (res, args) in _lib.SIGNATURES.items():
        getattr(lib, name).restype = res
        getattr(lib, name).argtypes = args
    dev = torch.device("cuda", 0)
    fa = torch.empty(64 << 20, dtype=torch.float32, device=dev)
    fb = torch.ones(64 << 20, dtype=torch.float32, device=dev)
    x = torch.randn((N0, N1), device=dev)
    P0, P1 = N0 - (1 << m0) + 1, N1 - (1 << m1) + 1
    s = torch.cuda.current_stream(dev)
    for v in range(lib.tune_count()):
        name = lib.tune_name(v).decode()
        prec = 1 if name.startswith("double") else 0
        out = torch.empty((P0, P1, 1 << m0, 1 << m1),
                          dtype=torch.complex128 if prec else torch.complex64, device=dev)
        lib.tune_select(v)

        def launch():
            rc = lib.swdft2d_forward(x.data_ptr(), _lib.IN_F32, N0, N1, N1, m0, m1, prec, 1.0, 0,
                                     P0, out.data_ptr(), 0, s.cuda_stream)
            assert rc == 0, lib.swdft2d_last_error()

        launch()
        ts = []
        for _ in range(5):
            torch.cuda.synchronize()
            fa.fill_(1.0)
            fb.sum()
            torch.cuda._sleep(200000)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            launch()
            e1.record(s)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) / 1e3)
        t = statistics.median(ts)
        print(json.dumps({"variant": name, "window": [1 << m0, 1 << m1], "N": [N0, N1],
                          "ms": t * 1e3, "write_tbs": out.numel() * out.element_size() / t / 1e12}),
              flush=True)
        del out
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
