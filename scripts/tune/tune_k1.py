"""Time K1 shape variants (scripts/tune/_build/libtune.so) on the BASELINE configs.

    python scripts/tune/tune_k1.py [--reps 5]

For every variant: select it, run the full config it matches ((m0, m1) ->
c4 / c3 / c5), report device time, coefficient rate and HBM write GB/s, and
check the output against the product library (max window-relative error).
"""
import argparse
import ctypes
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_1707_08213_b200 import _lib  # noqa: E402
from paper_1707_08213_b200.tree2d import forward_into  # noqa: E402
from paper_1707_08213_b200.workloads import CONFIGS  # noqa: E402

BY_M = {}
for c in CONFIGS.values():
    if c.precision == "fp32":
        BY_M.setdefault((c.m0, c.m1), []).append(c)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--only", default="")
    ap.add_argument("--configs", default="c2,c3,c4,c5")
    ap.add_argument("--prec", type=int, default=0, help="0 fp32 / 1 fp64 variants")
    a = ap.parse_args()
    lib = ctypes.CDLL(os.environ.get("TUNE_LIB", os.path.join(HERE, "_build", "libtune.so")))
    lib.tune_name.restype = ctypes.c_char_p
    for name, (res, args) in _lib.SIGNATURES.items():
        getattr(lib, name).restype = res
        getattr(lib, name).argtypes = args
    dev = torch.device("cuda", 0)
    flush = torch.empty(64 << 20, dtype=torch.float32, device=dev)
    cache = {}
    for cname in a.configs.split(","):
        for v in range(lib.tune_count()):
            name = lib.tune_name(v).decode()
            if a.only and a.only not in name:
                continue
            cfg = CONFIGS[cname]
            if (lib.tune_m(v, 0), lib.tune_m(v, 1)) == (cfg.m0, cfg.m1):
                run_variant(lib, v, name, cfg, cache, dev, flush, a)


def run_variant(lib, v, name, cfg, cache, dev, flush, a):
        m0, m1 = cfg.m0, cfg.m1
        if cfg.name not in cache:
            cache.clear()
            torch.cuda.empty_cache()
            x = torch.from_numpy(cfg.generate()).to(dev)
            odt = torch.complex128 if a.prec else torch.complex64
            out = torch.empty((cfg.P0, cfg.P1, cfg.n0, cfg.n1), dtype=odt, device=dev)
            # reference output of the product library: full if it fits, else the first rows
            rows = cfg.P0 if cfg.coefficients * 8 < 60e9 else 64
            ref = torch.empty((rows, cfg.P1, cfg.n0, cfg.n1), dtype=odt, device=dev)
            forward_into(x, m0, m1, ref, prec=a.prec, p0_end=rows)
            cache[cfg.name] = (x, ref, out)
            del x, ref, out
        x, ref, out = cache[cfg.name]
        lib.tune_select(v)
        s = torch.cuda.current_stream(dev)

        def launch():
            rc = lib.swdft2d_forward(x.data_ptr(), _lib.IN_F32 if x.dtype == torch.float32 else _lib.IN_C64,
                                     cfg.N0, cfg.N1, cfg.N1, m0, m1, a.prec, 1.0, 0, cfg.P0,
                                     out.data_ptr(), 1, s.cuda_stream)
            assert rc == 0, lib.swdft2d_last_error()

        launch()
        torch.cuda.synchronize()
        ts = []
        for _ in range(a.reps):
            flush.fill_(1.0)
            torch.cuda._sleep(300000)  # the host enqueues the launch before e0 runs
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            launch()
            e1.record(s)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) / 1e3)
        t = sorted(ts)[len(ts) // 2]  # median: single slow reps (clock dips) do not move it
        err = 0.0
        for a0 in range(0, ref.shape[0], 512):
            a1 = min(a0 + 512, ref.shape[0])
            d = (out[a0:a1] - ref[a0:a1]).abs().amax((-1, -2))
            nrm = ref[a0:a1].abs().pow(2).sum((-1, -2)).sqrt().clamp_min(1e-30)
            err = max(err, float((d / nrm).max()))
        print(json.dumps({"variant": name, "config": cfg.name, "ms": t * 1e3,
                          "ms_min": min(ts) * 1e3, "ms_max": max(ts) * 1e3,
                          "gcoef_s": cfg.coefficients / t / 1e9,
                          "write_gbs": cfg.coefficients * (16 if a.prec else 8) / t / 1e9,
                          "threads": lib.tune_m(v, 2), "smem": lib.tune_m(v, 3),
                          "max_rel_vs_product": err}), flush=True)


if __name__ == "__main__":
    main()
