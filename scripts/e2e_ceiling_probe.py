"""Is swdft2d_forward_host at the device-to-host link's rate on THIS box?

    python scripts/e2e_ceiling_probe.py [c4]

Interleaves, 5 times: a plain D2H copy of the config's full output (resident in HBM) into a
pinned buffer — the link's ceiling for these bytes — and one swdft2d_forward_host call into
the same buffer.  Prints both times per repetition.
"""
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
    c = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c4"]
    prec = _precision_code(c.precision, None)
    x = c.generate()
    spec = WindowSpec((c.m0, c.m1))
    dev_out = tree_swdft_2d(x, spec, budget=1 << 62, precision=c.precision).values
    host = torch.empty(dev_out.shape, dtype=dev_out.dtype, pin_memory=True)
    x_pin = torch.from_numpy(x).pin_memory()
    rows = []
    for rep in range(5):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        host.copy_(dev_out, non_blocking=True)
        torch.cuda.synchronize()
        t_copy = time.perf_counter() - t0
        t0 = time.perf_counter()
        tree_swdft_2d(x_pin, spec, budget=1 << 62, host_out=host, precision=c.precision)
        torch.cuda.synchronize()
        t_call = time.perf_counter() - t0
        rows.append({"rep": rep, "plain_d2h_s": t_copy, "plain_gb_s": host.numel() * host.element_size() / t_copy / 1e9,
                     "forward_host_s": t_call, "ratio": t_call / t_copy})
    print(json.dumps({"config": c.name, "bytes": host.numel() * host.element_size(), "reps": rows}))


if __name__ == "__main__":
    main()
