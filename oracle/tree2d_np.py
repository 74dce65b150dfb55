"""numpy restatement of the reference 2D tree SWDFT (levels-outer schedule).

TEST INFRASTRUCTURE ONLY (parity checker / CPU-baseline context).  The product
path must never import this module.

Follows /root/reference/pkg/src/swdft:
  core.make_twiddles   core.py:125-138
  core.butterfly       core.py:223-246  (float64, every multiply/add separately rounded)
  TreeLattice2D        tree2d.py:30-69  (two [N0, N1, n0, n1] complex128 buffers)
  row_level_step       tree2d.py:72-93
  col_level_step       tree2d.py:96-120
  _levels_outer        tree2d.py:123-129
The slicing here is written independently (no fancy-index gathers); the
arithmetic per node is the same sequence of IEEE float64 operations, so the
output is bitwise identical to the reference.
"""
from __future__ import annotations

import numpy as np


def twiddles(n: int) -> np.ndarray:
    """core.py:134-137."""
    ang = np.arange(n, dtype=np.float64) * (2.0 * np.pi / n)
    t = np.empty(n, dtype=np.complex128)
    t.real = np.cos(ang)
    t.imag = -np.sin(ang)
    return t


def _combine(sh: np.ndarray, w: np.ndarray, cu: np.ndarray, out: np.ndarray) -> None:
    """out = sh + w*cu with the reference's rounding order (core.py:238-245)."""
    wr, wi = w.real, w.imag
    cr, ci = cu.real, cu.imag
    re = wr * cr
    re -= wi * ci
    im = wr * ci
    im += wi * cr
    np.add(sh.real, re, out=out.real)
    np.add(sh.imag, im, out=out.imag)


def tree2d_levels_outer(x, m0: int, m1: int) -> np.ndarray:
    """Full-array 2D tree SWDFT, unnormalized; returns [P0, P1, n0, n1] complex128."""
    x = np.asarray(x, dtype=np.complex128)
    N0, N1 = x.shape
    n0, n1 = 1 << m0, 1 << m1
    cur = np.zeros((N0, N1, n0, n1), dtype=np.complex128)
    nxt = np.zeros_like(cur)
    cur[:, :, 0, 0] = x
    tw1 = twiddles(n1)
    tw0 = twiddles(n0)
    for t in range(1, m1 + 1):
        s, L = 1 << (m1 - t), 1 << t
        H = L // 2
        lo = n1 - s
        for half in (0, 1):  # node i = half*H + i'
            w = tw1[(np.arange(H) + half * H) * s]
            _combine(cur[:, lo - s:N1 - s, 0, :H], w, cur[:, lo:, 0, :H],
                     nxt[:, lo:, 0, half * H:(half + 1) * H])
        cur, nxt = nxt, cur
    for q in range(1, m0 + 1):
        s, L = 1 << (m0 - q), 1 << q
        H = L // 2
        lo = n0 - s
        for half in (0, 1):
            w = tw0[(np.arange(H) + half * H) * s][:, None]
            _combine(cur[lo - s:N0 - s, n1 - 1:, :H, :], w, cur[lo:, n1 - 1:, :H, :],
                     nxt[lo:, n1 - 1:, half * H:(half + 1) * H, :])
        cur, nxt = nxt, cur
    return cur[n0 - 1:, n1 - 1:].copy()
