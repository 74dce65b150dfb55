"""Row-push stream throughput: push the rows of a config one at a time (device-resident
rows), time pushes after warm-up with CUDA events; reports rows/s and coef/s."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1707_08213_b200 import WindowSpec  # noqa: E402
from paper_1707_08213_b200.stream import SlidingRowStream2D  # noqa: E402
from paper_1707_08213_b200.workloads import CONFIGS  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c4")
ap.add_argument("--rows", type=int, default=256)
ap.add_argument("--precision", default="fp32")
ap.add_argument("--block", type=int, default=1, help="rows per push (push_rows when > 1)")
a = ap.parse_args()
cfg = CONFIGS[a.config]
warm = cfg.n0 + a.block  # warm-up pushes: the window rows plus one block (allocations)
x = torch.from_numpy(cfg.generate(rows=min(cfg.N0, a.rows + warm))).cuda()
a.rows = min(a.rows, x.shape[0] - warm)
st = SlidingRowStream2D(WindowSpec((cfg.m0, cfg.m1)), cfg.N1, precision=a.precision)
for r in range(cfg.n0):
    st.push_row(x[r])
if a.block > 1:
    st.push_rows(x[cfg.n0:warm])
else:
    st.push_row(x[cfg.n0])
    warm = cfg.n0 + 1
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
if a.block == 1:
    for r in range(warm, warm + a.rows):
        st.push_row(x[r])
else:
    for r in range(warm, warm + a.rows, a.block):
        st.push_rows(x[r:min(r + a.block, warm + a.rows)])
e1.record()
torch.cuda.synchronize()
s = e0.elapsed_time(e1) / 1e3
coefs = a.rows * cfg.P1 * cfg.n0 * cfg.n1
print(json.dumps({"config": cfg.name, "precision": a.precision, "pushes": a.rows, "block": a.block,
                  "us_per_push": s / a.rows * 1e6, "rows_per_s": a.rows / s,
                  "gcoef_s": coefs / s / 1e9}))
