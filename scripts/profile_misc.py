"""One launch of a non-K1 kernel for ncu captures.

    python scripts/profile_misc.py kr  N n      # KR, 1D tree of N float64 samples, window n (fp32)
    python scripts/profile_misc.py kc  N0 N1 m0 m1   # KR + KC, separable large window (fp32)
    python scripts/profile_misc.py k2  config   # K2 stream pushes of a config (fp32), after warm-up
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1707_08213_b200 import WindowSpec  # noqa: E402
from paper_1707_08213_b200.tree2d import _OUT_DTYPES, forward_into  # noqa: E402

mode = sys.argv[1]
dev = torch.device("cuda", 0)
if mode == "kr":
    N, n = int(sys.argv[2]), int(sys.argv[3])
    m = n.bit_length() - 1
    x = torch.from_numpy(np.random.default_rng(0).standard_normal((1, N))).to(dev)
    out = torch.empty((1, N - n + 1, 1, n), dtype=_OUT_DTYPES[0], device=dev)
    forward_into(x, 0, m, out, prec=0)
elif mode == "kc":
    N0, N1, m0, m1 = (int(v) for v in sys.argv[2:6])
    x = torch.from_numpy(np.random.default_rng(0).standard_normal((N0, N1)).astype(np.float32)).to(dev)
    out = torch.empty((N0 - (1 << m0) + 1, N1 - (1 << m1) + 1, 1 << m0, 1 << m1),
                      dtype=_OUT_DTYPES[0], device=dev)
    forward_into(x, m0, m1, out, prec=0, kernel="separable")
else:
    from paper_1707_08213_b200.stream import SlidingRowStream2D
    from paper_1707_08213_b200.workloads import CONFIGS

    cfg = CONFIGS[sys.argv[2]]
    x = torch.from_numpy(cfg.generate(rows=cfg.n0 + 4)).to(dev)
    st = SlidingRowStream2D(WindowSpec((cfg.m0, cfg.m1)), cfg.N1, precision="fp32")
    for r in range(cfg.n0 + 4):
        st.push_row(x[r])
torch.cuda.synchronize()
print("ok", mode)
