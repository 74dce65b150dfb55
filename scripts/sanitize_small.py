"""Small launches of every kernel (K1 LDG/TMA, K0, KR, K2, ring store) for
compute-sanitizer memcheck / racecheck / synccheck runs:

    compute-sanitizer --tool memcheck python scripts/sanitize_small.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1707_08213_b200 import WindowSpec, tree_swdft_2d  # noqa: E402
from paper_1707_08213_b200.stream import SlidingRowStream2D  # noqa: E402

rng = np.random.default_rng(0)
x = rng.standard_normal((40, 37))
for m in [(3, 2), (2, 4), (0, 5), (0, 8), (1, 1), (6, 3), (7, 1)]:
    for prec in ("fp64", "fp32"):
        for kernel in ("auto", "stream", "window", "stream_tma", "rows"):
            if kernel == "rows" and m[0] != 0:
                continue
            if kernel in ("stream", "stream_tma") and max(m) > 6:
                continue
            xx = x if m[0] < 7 else rng.standard_normal((140, 12))
            tree_swdft_2d(xx, WindowSpec(m), precision=prec, kernel=kernel, budget=1 << 40)
st = SlidingRowStream2D(WindowSpec((3, 2)), 37)
for r in range(12):
    st.push_row(x[r])
st.push_rows(x[12:20])
st.push_row(x[20])
torch.cuda.synchronize()
print("sanitize_small ok")
