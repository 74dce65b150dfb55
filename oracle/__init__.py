"""Oracle for the 2D tree SWDFT hot path — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
``--impl reference`` legs may import this package.  The product package
(``paper_1707_08213_b200``) never imports it and has no CPU fallback.

Contents
  swdft2d_oracle.c   C restatement of the reference's levels-outer tree
                     (tree2d.py:30-129, core.py:125-138,223-246), bitwise equal
                     to the reference; pthreads split along axis 0 like
                     tree2d._split/_run_chunks (tree2d.py:22-27,58-64).
  tree2d_np.py       numpy restatement of the same schedule (small cases).

Pinning: tests/test_oracle.py checks both against the golden vectors in
tests/golden/ that tests/golden/make_golden.py produced by running the
reference itself (/root/reference/pkg/src/swdft) in the build container.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "libswdft2d_oracle.so")
_lib = None


def build() -> str:
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        i64, dp, c_int = ctypes.c_int64, ctypes.c_void_p, ctypes.c_int
        L.swdft2d_oracle_forward.argtypes = [dp, i64, i64, c_int, c_int, i64, i64,
                                             ctypes.c_double, c_int, dp, c_int, i64]
        L.swdft2d_oracle_forward.restype = c_int
        L.swdft2d_oracle_window_fft.argtypes = [dp, i64, i64, c_int, c_int, i64, i64, dp]
        L.swdft2d_oracle_window_fft.restype = c_int
        L.swdft2d_oracle_twiddles.argtypes = [c_int, dp, dp]
        L.swdft2d_oracle_twiddles.restype = None
        _lib = L
    return _lib


def _as_c128(x) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(x), dtype=np.complex128)


def tree2d(x, m0: int, m1: int, p0_begin: int = 0, p0_end: int | None = None,
           scale: float | None = None, threads: int = 1,
           max_lattice_bytes: int = 1 << 31) -> np.ndarray:
    """Window rows [p0_begin, p0_end) of the reference output, complex128 [R, P1, n0, n1].

    ``scale`` None means normalization mode "none" (identity); otherwise every
    component is multiplied by float64(scale) (core.normalize, core.py:301).
    """
    xc = _as_c128(x)
    N0, N1 = xc.shape
    n0, n1 = 1 << m0, 1 << m1
    P0, P1 = N0 - n0 + 1, N1 - n1 + 1
    if p0_end is None:
        p0_end = P0
    out = np.empty((p0_end - p0_begin, P1, n0, n1), dtype=np.complex128)
    rc = lib().swdft2d_oracle_forward(
        xc.ctypes.data, N0, N1, m0, m1, p0_begin, p0_end,
        float(scale) if scale is not None else 1.0, 0 if scale is None else 1,
        out.ctypes.data, int(threads), int(max_lattice_bytes))
    if rc != 0:
        raise ValueError(f"oracle rejected arguments (rc={rc})")
    return out


def window_fft(x, m0: int, m1: int, p0: int, p1: int) -> np.ndarray:
    """One window by per-window DIT FFT (oracle.swfft_2d semantics, oracle.py:166-187)."""
    xc = _as_c128(x)
    out = np.empty((1 << m0, 1 << m1), dtype=np.complex128)
    rc = lib().swdft2d_oracle_window_fft(xc.ctypes.data, xc.shape[0], xc.shape[1], m0, m1,
                                         p0, p1, out.ctypes.data)
    if rc != 0:
        raise ValueError("window out of range")
    return out


def twiddles(n: int) -> np.ndarray:
    re = np.empty(n)
    im = np.empty(n)
    lib().swdft2d_oracle_twiddles(n, re.ctypes.data, im.ctypes.data)
    t = np.empty(n, dtype=np.complex128)
    t.real = re
    t.imag = im
    return t


def window_rel_err(got, ref) -> float:
    """BASELINE.json tolerance metric: max over windows of
    max_k |got - ref| / ||ref window||_2 (absolute error for an all-zero window)."""
    got = np.asarray(got)
    ref = np.asarray(ref)
    d = np.abs(got.astype(np.complex128) - ref).reshape(ref.shape[0], ref.shape[1], -1)
    nrm = np.sqrt((np.abs(ref.reshape(ref.shape[0], ref.shape[1], -1)) ** 2).sum(-1))
    num = d.max(-1)
    den = np.where(nrm > 0, nrm, 1.0)
    return float((num / den).max()) if num.size else 0.0
