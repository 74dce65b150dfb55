"""k-D tree rate (3-D): per-slice 2-D transforms (K1) + the column-tree pass (KC)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1707_08213_b200 import WindowSpec  # noqa: E402
from paper_1707_08213_b200.treekd import tree_swdft_kd  # noqa: E402

dev = torch.device("cuda", 0)
for shape, m in [((128, 128, 128), (3, 3, 3)), ((64, 256, 256), (2, 3, 3)), ((96, 96, 96), (4, 3, 2))]:
    for prec in ("fp32", "fp64"):
        x = torch.from_numpy(np.random.default_rng(0).standard_normal(shape).astype(np.float32)).to(dev)
        spec = WindowSpec(m)
        tree_swdft_kd(x, spec, budget=1 << 62, precision=prec)
        torch.cuda.synchronize()
        ts = []
        for _ in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            r = tree_swdft_kd(x, spec, budget=1 << 62, precision=prec)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) / 1e3)
            coefs = r.values.numel()
            del r
        t = float(np.median(ts))
        print(json.dumps({"shape": shape, "window": [1 << v for v in m], "prec": prec,
                          "ms": t * 1e3, "gcoef_s": coefs / t / 1e9,
                          "write_tbs": coefs * (16 if prec == "fp64" else 8) / t / 1e12}), flush=True)
