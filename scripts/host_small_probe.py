"""Latency of the host-output call on small problems (config 1 and a few sizes around the
16 MiB threshold below which pageable outputs skip the staging workers)."""
import json
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1707_08213_b200 import WindowSpec, tree_swdft_2d  # noqa: E402

torch.cuda.init()
rng = np.random.default_rng(0)
for N, m in ((64, 3), (128, 3), (256, 3), (256, 4), (512, 4)):
    x = rng.standard_normal((N, N))
    spec = WindowSpec((m, m))
    for _ in range(3):
        r = tree_swdft_2d(x, spec, to_host=True, budget=1 << 40)
    ts, td = [], []
    for _ in range(20):
        t0 = time.perf_counter()
        r = tree_swdft_2d(x, spec, to_host=True, budget=1 << 40)
        ts.append(time.perf_counter() - t0)
        t0 = time.perf_counter()
        v = tree_swdft_2d(x, spec, budget=1 << 40).values.cpu().numpy()
        td.append(time.perf_counter() - t0)
    print(json.dumps({"N": N, "n": 1 << m, "out_mb": r.values.nbytes / 2**20,
                      "to_host_ms": statistics.median(ts) * 1e3,
                      "device_then_cpu_ms": statistics.median(td) * 1e3}), flush=True)
