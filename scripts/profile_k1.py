"""Launch the hot-path kernel a few times on one config for ncu captures.

    python scripts/profile_k1.py --config c4 --rows 1024 --launches 3 [--kernel stream]

Runs window rows [0, rows) of the config (the full width), so an `ncu --set full`
replay only has to save/restore that much output.  Per-launch metrics scale
with the rows; the per-CTA behaviour is that of the full run.
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1707_08213_b200.tree2d import _OUT_DTYPES, _precision_code, forward_into  # noqa: E402
from paper_1707_08213_b200.workloads import CONFIGS  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c4")
    ap.add_argument("--rows", type=int, default=0, help="window rows (0 = all)")
    ap.add_argument("--launches", type=int, default=3)
    ap.add_argument("--kernel", default="auto")
    ap.add_argument("--precision", default=None)
    a = ap.parse_args()
    cfg = CONFIGS[a.config]
    rows = a.rows or cfg.P0
    x = torch.from_numpy(cfg.generate(rows=rows + cfg.n0 - 1)).cuda()
    prec = _precision_code(a.precision or cfg.precision, None)
    out = torch.empty((rows, cfg.P1, cfg.n0, cfg.n1), dtype=_OUT_DTYPES[prec], device="cuda")
    for _ in range(a.launches):
        forward_into(x, cfg.m0, cfg.m1, out, prec=prec, kernel=a.kernel)
    torch.cuda.synchronize()
    print(f"ok {a.config} rows={rows} launches={a.launches}")


if __name__ == "__main__":
    main()
