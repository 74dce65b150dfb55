"""Randomised fp64 (bitwise) / fp32 (tolerance) parity fuzz of the product path against the C oracle (test
infrastructure; run on the GPU box, not part of the default suite).

    python scripts/fuzz_parity.py [--cases 400] [--seed 1] [--max-coefs 6e6]

Each case draws a window (n0, n1 in 1..1024, weighted to K1's 1..64), an array shape
(from the window size up to a few hundred extra rows/columns, including sizes that leave
partial tiles and single window rows/columns), an input dtype (f32, f64, c64, c128), a
row stride (padded or not), a window-row sub-range and a normalization, runs
forward_into in fp64 and requires bitwise equality with the oracle
(oracle/swdft2d_oracle.c, the restated reference), and in fp32 within BASELINE's
max|err| / ||window||_2 <= 1e-4.  Prints one JSON line per failure and a
summary line; exit code 1 on any mismatch.
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
from paper_1707_08213_b200 import _lib  # noqa: E402
from paper_1707_08213_b200.core import WindowSpec, normalization_factor  # noqa: E402
from paper_1707_08213_b200.tree2d import _OUT_DTYPES, forward_into  # noqa: E402


def bits_equal(a, b):
    a = np.ascontiguousarray(a).view(np.uint64)
    b = np.ascontiguousarray(b).view(np.uint64)
    return a.shape == b.shape and bool(np.array_equal(a, b))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cases", type=int, default=400)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--max-coefs", type=float, default=6e6)
    ap.add_argument("--k1-only", action="store_true",
                    help="windows 2..64 x 1..64 only (K1), e.g. under SWDFT2D_K1_* overrides")
    a = ap.parse_args()
    oracle.build()
    dev = torch.device("cuda", 0)
    rng = np.random.default_rng(a.seed)
    dtypes = [np.float32, np.float64, np.complex64, np.complex128]
    fails = 0
    t0 = time.time()
    kinds = {}
    worst32 = 0.0
    for case in range(a.cases):
        u = rng.random()
        big, tall = u < 0.15, 0.15 <= u < 0.25  # tall: K1's 128/256-row windows
        if a.k1_only:
            big = tall = False
        m0 = int(rng.integers(7, 10)) if tall else int(rng.integers(0, 11 if big else 7))
        m1 = int(rng.integers(0, 6)) if tall else int(rng.integers(0, 11 if big else 7))
        if a.k1_only and m0 == 0:
            m0 = int(rng.integers(1, 7))
        n0, n1 = 1 << m0, 1 << m1
        # shape: window + extra, bounded output size
        for _ in range(50):
            N0 = n0 + int(rng.integers(0, 300 if n0 <= 64 else 40))
            N1 = n1 + int(rng.integers(0, 300 if n1 <= 64 else 40))
            if (N0 - n0 + 1) * (N1 - n1 + 1) * n0 * n1 <= a.max_coefs:
                break
        else:
            continue
        dt = dtypes[int(rng.integers(0, 4))]
        x = rng.standard_normal((N0, N1))
        if np.issubdtype(dt, np.complexfloating):
            x = x + 1j * rng.standard_normal((N0, N1))
        x = x.astype(dt)
        pad = int(rng.integers(0, 3)) * int(rng.integers(1, 17))
        P0, P1 = N0 - n0 + 1, N1 - n1 + 1
        p0a = int(rng.integers(0, P0)) if rng.random() < 0.3 else 0
        p0b = int(rng.integers(p0a + 1, P0 + 1)) if rng.random() < 0.3 else P0
        norm = ["none", "unitary", "paper-2d"][int(rng.integers(0, 3))]
        scale = normalization_factor(WindowSpec((m0, m1), norm)) if norm != "none" else None
        ref = oracle.tree2d(x, m0, m1, p0_begin=p0a, p0_end=p0b, scale=scale)
        wide = torch.zeros((N0, N1 + pad), dtype=torch.from_numpy(x).dtype, device=dev)
        wide[:, :N1] = torch.from_numpy(x).to(dev)
        out = torch.empty((p0b - p0a, P1, n0, n1), dtype=_OUT_DTYPES[_lib.PREC_FP64], device=dev)
        forward_into(wide[:, :N1], m0, m1, out, prec=_lib.PREC_FP64, p0_begin=p0a, p0_end=p0b,
                     scale=1.0 if scale is None else scale)
        got = out.cpu().numpy()
        # fp32 mode on the same case: BASELINE's tolerance, max |err| / ||window||_2 <= 1e-4
        o32 = torch.empty((p0b - p0a, P1, n0, n1), dtype=_OUT_DTYPES[_lib.PREC_FP32], device=dev)
        forward_into(wide[:, :N1], m0, m1, o32, prec=_lib.PREC_FP32, p0_begin=p0a, p0_end=p0b,
                     scale=1.0 if scale is None else scale)
        g32 = o32.cpu().numpy().astype(np.complex128)
        nrm = np.sqrt((np.abs(ref) ** 2).sum(axis=(-1, -2)))
        err = np.abs(g32 - ref).max(axis=(-1, -2))
        rel32 = float(np.max(np.where(nrm > 0, err / np.where(nrm > 0, nrm, 1), err)))
        worst32 = max(worst32, rel32)
        k1_big = (m0 == 7 and m1 <= 5) or (m0 == 8 and m1 <= 2) or (m0 == 9 and m1 <= 1)
        kind = "KR" if m0 == 0 else ("K1" if max(m0, m1) <= 6 or k1_big else "KR+KC")
        kinds[kind] = kinds.get(kind, 0) + 1
        if not bits_equal(got, ref) or rel32 > 1e-4:
            fails += 1
            d = np.abs(got - ref)
            print(json.dumps({"case": case, "m": [m0, m1], "N": [N0, N1], "dtype": np.dtype(dt).name,
                              "pad": pad, "rows": [p0a, p0b], "norm": norm, "kernel": kind,
                              "max_abs_diff": float(d.max()), "fp32_rel": rel32}), flush=True)
    done = sum(kinds.values())
    print(json.dumps({"cases": done, "requested": a.cases, "fails": fails,
                      "env": {k: v for k, v in os.environ.items() if k.startswith("SWDFT2D_")}, "by_kernel": kinds,
                      "fp32_worst_window_rel_err": worst32,
                      "seconds": round(time.time() - t0, 1)}), flush=True)
    return 1 if fails else 0


if __name__ == "__main__":
    sys.exit(main())
