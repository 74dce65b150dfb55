"""Run one K1 launch per (input dtype, precision, shape) in a fresh process and report failures."""
import itertools
import subprocess
import sys

CODE = r'''
import sys, numpy as np, torch
sys.path.insert(0, ".")
from paper_1707_08213_b200 import WindowSpec, tree_swdft_2d
import oracle
dt, prec, N0, N1, m0, m1 = sys.argv[1], sys.argv[2], int(sys.argv[3]), int(sys.argv[4]), int(sys.argv[5]), int(sys.argv[6])
rng = np.random.default_rng(0)
x = rng.standard_normal((N0, N1)) + (1j * rng.standard_normal((N0, N1)) if dt.startswith("c") else 0)
x = x.astype(dt)
r = tree_swdft_2d(x, WindowSpec((m0, m1)), precision=prec, budget=1 << 62, kernel="stream").values.cpu().numpy()
ref = oracle.tree2d(x.astype(np.complex128), m0, m1)
print("err", oracle.window_rel_err(r, ref))
'''
cases = list(itertools.product(["float32", "float64", "complex64", "complex128"], ["fp32", "fp64"],
                               [(64, 64, 4, 4), (40, 512, 2, 3), (100, 128, 5, 3), (130, 130, 6, 6)]))
for dt, prec, (N0, N1, m0, m1) in cases:
    r = subprocess.run([sys.executable, "-c", CODE, dt, prec, str(N0), str(N1), str(m0), str(m1)],
                       capture_output=True, text=True, timeout=120)
    tail = (r.stdout.strip().splitlines() or [""])[-1] if r.returncode == 0 else \
        [l for l in r.stderr.splitlines() if "Error" in l or "error" in l][-1:]
    print(dt, prec, (N0, N1, m0, m1), "rc", r.returncode, tail, flush=True)
