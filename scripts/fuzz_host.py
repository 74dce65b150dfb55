"""Randomised check of swdft2d_forward_host / swdft2d_download against the device path.

    python scripts/fuzz_host.py [--cases 200] [--seed 1]

Each case draws a window (K1, KR and large-window paths), an array, an input dtype, a
precision, a padded row stride, a window-row range, a strip size (from one window row to the
whole output), a destination kind (pinned / pageable), staging threads and chunk size, and
requires the host result to equal swdft2d_forward's device result bit for bit (the strips
run the same kernels; fp32 is bitwise too, except on the large-window path, whose column
kernel depends on the strip length: there fp32 is held to 1e-5 of the window norm).  Outputs range up to ~300 MB so that pageable
destinations cross the 16 MiB threshold into the staging workers.
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1707_08213_b200 import _lib  # noqa: E402
from paper_1707_08213_b200.tree2d import _OUT_DTYPES, forward_into  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cases", type=int, default=200)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--exp", type=float, nargs=2, default=(4.5, 7.3),
                    help="log10 range of the coefficient count per case")
    a = ap.parse_args()
    rng = np.random.default_rng(a.seed)
    dev = torch.device("cuda", 0)
    dts = [np.float32, np.float64, np.complex64, np.complex128]
    fails, staged, t0 = 0, 0, time.time()
    for case in range(a.cases):
        m0 = int(rng.integers(0, 8)) if rng.random() < 0.85 else int(rng.integers(7, 10))
        m1 = int(rng.integers(0, 7)) if m0 <= 7 else int(rng.integers(0, 3))
        n0, n1 = 1 << m0, 1 << m1
        target = 10 ** rng.uniform(*a.exp)  # coefficients
        P0 = int(max(1, min(3000, rng.integers(1, 400))))
        P1 = int(max(1, min(4000, target / (P0 * n0 * n1))))
        N0, N1 = P0 + n0 - 1, P1 + n1 - 1
        dt = dts[int(rng.integers(0, 4))]
        prec = int(rng.integers(0, 2))
        ld = N1 + int(rng.integers(0, 9)) * int(rng.integers(0, 2))
        buf = rng.standard_normal((N0, ld)).astype(dt)
        if np.iscomplexobj(buf):
            buf = buf + 1j * rng.standard_normal((N0, ld)).astype(dt)
            buf = buf.astype(dt)
        x = buf[:, :N1]
        a0 = int(rng.integers(0, P0))
        b0 = int(rng.integers(a0 + 1, P0 + 1))
        scale = [1.0, 1.0 / np.sqrt(n0 * n1)][int(rng.integers(0, 2))]
        osz = 8 if prec == 0 else 16
        row_bytes = P1 * n0 * n1 * osz
        total = (b0 - a0) * row_bytes
        strip = int([0, row_bytes, max(row_bytes, total // int(rng.integers(1, 12))),
                     int(rng.integers(1, total + 2))][int(rng.integers(0, 4))])
        pinned = bool(rng.integers(0, 2))
        os.environ["SWDFT2D_HOST_THREADS"] = str(int(rng.integers(1, 17)))
        os.environ["SWDFT2D_HOST_CHUNK_MB"] = str(int(rng.choice([1, 2, 4, 8])))
        os.environ["SWDFT2D_HOST_NT"] = str(int(rng.integers(0, 2)))
        odt = np.complex64 if prec == 0 else np.complex128
        shape = (b0 - a0, P1, n0, n1)
        out = (_lib.host_empty if pinned else np.empty)(shape, odt)
        out.view(np.float32 if prec == 0 else np.float64).fill(np.nan)
        try:
            _lib.forward_host(x, m0, m1, out, prec=prec, scale=scale, p0_begin=a0, p0_end=b0,
                              strip_bytes=strip)
            xd = torch.from_numpy(np.ascontiguousarray(x)).to(dev)
            ref = torch.empty(shape, dtype=_OUT_DTYPES[prec], device=dev)
            forward_into(xd, m0, m1, ref, prec=prec, scale=scale, p0_begin=a0, p0_end=b0)
            got2 = _lib.download(ref)  # and the download path on the same data
            ref = ref.cpu().numpy()
            iv = np.uint32 if prec == 0 else np.uint64
            ok = np.array_equal(got2.view(iv), ref.view(iv))
            if prec == 0 and max(m0, m1) > 6:
                # the large-window path picks its column kernel (K1's Z-column kernel or KC)
                # by strip length; the two differ in fp32 rounding (FMA order), not in fp64
                d = np.abs(out.astype(np.complex128) - ref.astype(np.complex128)).reshape(len(out), P1, -1)
                nrm = np.linalg.norm(ref.astype(np.complex128).reshape(len(out), P1, -1), axis=2)
                ok = ok and bool((d.max(axis=2) <= 1e-5 * np.maximum(nrm, 1e-30)).all())
            else:
                ok = ok and np.array_equal(out.view(iv), ref.view(iv))
        except Exception as e:  # noqa: BLE001
            ok = False
            print(json.dumps({"case": case, "error": repr(e)}), flush=True)
        staged += (not pinned) and total > (16 << 20)
        if not ok:
            fails += 1
            print(json.dumps({"case": case, "m": [m0, m1], "N": [N0, N1], "dtype": np.dtype(dt).name,
                              "prec": prec, "rows": [a0, b0], "strip": strip, "pinned": pinned,
                              "env": {k: os.environ[k] for k in os.environ if k.startswith("SWDFT2D_HOST")}}),
                  flush=True)
        del out
    print(json.dumps({"cases": a.cases, "fails": fails, "staged_pageable_cases": int(staged),
                      "seed": a.seed, "seconds": round(time.time() - t0, 1)}), flush=True)
    sys.exit(1 if fails else 0)


if __name__ == "__main__":
    main()
