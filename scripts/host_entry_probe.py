"""Host-to-host paths compared on one config (default c4): seconds and Gcoef/s.

    python scripts/host_entry_probe.py [c4] [--reps 3]

  ring    tree_swdft_2d(pinned host tensor, host_out=pinned): the Python-orchestrated ring;
  c_abi   ONE swdft2d_forward_host call, numpy input -> pinned numpy output (host_empty);
  pageable  the same call into a fresh np.empty (pageable) output;
  alloc   swdft2d_host_alloc of the output (what a fresh pinned result costs);
  device+cpu  the full output in HBM, then .cpu() (the binding's old route).
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1707_08213_b200 import WindowSpec, _lib, tree_swdft_2d  # noqa: E402
from paper_1707_08213_b200.tree2d import _precision_code  # noqa: E402
from paper_1707_08213_b200.workloads import CONFIGS  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config", nargs="?", default="c4")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--strip-mb", type=int, default=512)
    ap.add_argument("--skip-slow", action="store_true")
    a = ap.parse_args()
    c = CONFIGS[a.config]
    prec = _precision_code(c.precision, None)
    odt = np.complex64 if prec == _lib.PREC_FP32 else np.complex128
    x = c.generate()
    shape = (c.P0, c.P1, c.n0, c.n1)
    spec = WindowSpec((c.m0, c.m1))
    torch.cuda.init()
    res = {"config": a.config, "coefficients": c.coefficients, "strip_mb": a.strip_mb}

    t0 = time.perf_counter()
    out = _lib.host_empty(shape, odt)
    res["alloc_pinned_s"] = time.perf_counter() - t0

    def timeit(fn, reps):
        ts = []
        for _ in range(reps):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            fn()
            torch.cuda.synchronize()
            ts.append(time.perf_counter() - t0)
        return min(ts), ts

    strip = a.strip_mb << 20
    t, ts = timeit(lambda: _lib.forward_host(x, c.m0, c.m1, out, prec=prec, strip_bytes=strip),
                   a.reps + 1)
    res["c_abi"] = {"s": t, "gcoef_s": c.coefficients / t / 1e9, "all": ts}
    chk = out[c.P0 // 2, c.P1 // 3].copy()

    x_pin = torch.from_numpy(x).pin_memory()
    host_out = torch.from_numpy(out)  # the same pinned block
    t, ts = timeit(lambda: tree_swdft_2d(x_pin, spec, budget=1 << 62, host_out=host_out,
                                         precision=c.precision, strip_bytes=strip), a.reps + 1)
    res["ring"] = {"s": t, "gcoef_s": c.coefficients / t / 1e9, "all": ts}
    assert np.array_equal(chk, out[c.P0 // 2, c.P1 // 3])
    if not a.skip_slow:
        del host_out
        del out
        # fresh pageable outputs (what a numpy-returning call hands back): staging workers /
        # non-temporal stores in the workers' copy / chunk size
        res["pageable_fresh"] = []
        for threads, nt, chunk in ((16, 1, 4), (16, 0, 4), (16, 1, 4), (16, 0, 4), (16, 1, 8), (16, 1, 2),
                                  (8, 1, 4), (4, 1, 4)):
            os.environ["SWDFT2D_HOST_THREADS"] = str(threads)
            os.environ["SWDFT2D_HOST_NT"] = str(nt)
            os.environ["SWDFT2D_HOST_CHUNK_MB"] = str(chunk)
            t0 = time.perf_counter()
            pg = np.empty(shape, odt)
            _lib.forward_host(x, c.m0, c.m1, pg, prec=prec, strip_bytes=strip)
            t = time.perf_counter() - t0
            assert np.array_equal(chk, pg[c.P0 // 2, c.P1 // 3])
            t2, _ = timeit(lambda: _lib.forward_host(x, c.m0, c.m1, pg, prec=prec, strip_bytes=strip), 1)
            res["pageable_fresh"].append({"threads": threads, "nt": nt, "chunk_mb": chunk, "s": t,
                                          "gcoef_s": c.coefficients / t / 1e9, "touched_s": t2})
            del pg
        for k in ("SWDFT2D_HOST_THREADS", "SWDFT2D_HOST_NT", "SWDFT2D_HOST_CHUNK_MB"):
            os.environ.pop(k, None)
        t0 = time.perf_counter()
        r = tree_swdft_2d(x, spec, budget=1 << 62, precision=c.precision)
        v = r.values.cpu().numpy()
        t = time.perf_counter() - t0
        res["device+cpu"] = {"s": t, "gcoef_s": c.coefficients / t / 1e9}
        assert np.array_equal(chk, v[c.P0 // 2, c.P1 // 3])
        del v
        t0 = time.perf_counter()
        v = r.numpy()  # swdft2d_download: staged by worker threads
        t = time.perf_counter() - t0
        res["download_fresh"] = {"s": t, "gb_s": v.nbytes / t / 1e9}
        assert np.array_equal(chk, v[c.P0 // 2, c.P1 // 3])
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
