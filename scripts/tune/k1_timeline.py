"""Per-CTA timeline of one K1 launch (tuning build with -DK1_TIMELINE):

    TUNE_LIB=scripts/tune/_build/libtune_tl.so python scripts/tune/k1_timeline.py c2

Runs the config's first harness variant once (after a warm-up launch and an L2 flush) and
prints the kernel span, per-SM busy time, the start ramp (first to last CTA start of the
first wave) and the tail (first SM idle to kernel end), all from %globaltimer."""
import ctypes
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1707_08213_b200 import _lib  # noqa: E402
from paper_1707_08213_b200.workloads import CONFIGS  # noqa: E402


def main():
    cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
    lib = ctypes.CDLL(os.environ.get("TUNE_LIB", os.path.join(HERE, "_build", "libtune_tl.so")))
    for name, (res, args) in _lib.SIGNATURES.items():
        getattr(lib, name).restype = res
        getattr(lib, name).argtypes = args
    lib.tune_select(0)
    dev = torch.device("cuda", 0)
    x = torch.from_numpy(cfg.generate()).to(dev)
    out = torch.empty((cfg.P0, cfg.P1, cfg.n0, cfg.n1), dtype=torch.complex64, device=dev)
    fa = torch.empty(64 << 20, dtype=torch.float32, device=dev)
    s = torch.cuda.current_stream(dev)
    info = _lib.k1_schedule(cfg.N0, cfg.N1, cfg.m0, cfg.m1, 0)
    grid = info["grid"]
    res = []
    for rep in range(4):
        fa.fill_(1.0)
        rc = lib.swdft2d_forward(x.data_ptr(), _lib.IN_F32, cfg.N0, cfg.N1, cfg.N1, cfg.m0, cfg.m1, 0,
                                 1.0, 0, cfg.P0, out.data_ptr(), 1, s.cuda_stream)
        assert rc == 0
        torch.cuda.synchronize()
        buf = (ctypes.c_ulonglong * (3 * grid))()
        assert lib.tune_timeline(buf, grid) == 0
        a = np.frombuffer(buf, dtype=np.uint64).reshape(grid, 3).astype(np.float64)
        t0 = a[:, 0].min()
        st, en, sm = (a[:, 0] - t0) / 1e3, (a[:, 1] - t0) / 1e3, a[:, 2].astype(int)
        span = en.max()
        busy = np.zeros(sm.max() + 1)
        last_end = np.zeros(sm.max() + 1)
        for i in range(grid):
            busy[sm[i]] += en[i] - st[i]
            last_end[sm[i]] = max(last_end[sm[i]], en[i])
        slots = info["slots"]
        first_wave = np.sort(st)[:slots]
        res.append({"config": cfg.name, "grid": grid, "span_us": span,
                    "first_wave_start_spread_us": first_wave.max() - first_wave.min(),
                    "cta_us_mean": float((en - st).mean()), "cta_us_max": float((en - st).max()),
                    "cta_us_min": float((en - st).min()),
                    "sm_last_end_min_us": float(last_end[last_end > 0].min()),
                    "tail_us": span - float(last_end[last_end > 0].min()),
                    "mean_resident_ctas": float(busy.sum() / (len(busy) * span))})
    for r in res:
        print(json.dumps(r))


if __name__ == "__main__":
    main()
