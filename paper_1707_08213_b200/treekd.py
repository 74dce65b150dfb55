"""k-dimensional tree sliding-window DFT by composition of the 2D kernel.

Drop-in for the reference's ``treekd.tree_swdft_kd`` (/root/reference/pkg/src/
swdft/treekd.py:102-121).  The reference's level plan gives dimension k-1 the
first block of levels and dimension 0 the last (core.py:150-161), and every level
combines positions along its own dimension only.  So for k >= 3:

  1. levels of dims k-1 .. 1 act on each slice x[i0] independently: they are the
     (k-1)-dimensional tree of that slice (computed recursively; k-1 = 2 is K1);
  2. levels of dim 0 are, for every (p_1.., k_1..) column of the stacked slice
     results, the 1D tree along i0 with window n0 — K1 with m1 = 0 on the
     [N0, prod(inner)] matrix of slice results;
  3. a transpose moves k0 from the last axis to axis k.

Each node is computed by the same butterfly with the same operands as in the
reference's lattice, so fp64 output is bit-identical (tests/test_next_rows.py).
The normalization factor is applied once, in the last (dim-0) pass.
"""
from __future__ import annotations

import math

import torch

from . import core
from .core import CoefficientArray
from .tree2d import _OUT_DTYPES, _precision_code, _to_tensor, forward_into


def level_regions_kd(shape, exponents):
    """(region, nodes_per_tree, positions) per level of the k-D plan, in order —
    the add_region calls of kd_level_step (treekd.py:95-97, core.py:197-215)."""
    k = len(exponents)
    sizes = [1 << m for m in exponents]
    out = []
    for c in range(k - 1, -1, -1):  # dimension k-1 owns the first block of levels
        for q in range(1, exponents[c] + 1):
            s = 1 << (exponents[c] - q)
            ext = [1 if i < c else (1 << q) if i == c else sizes[i] for i in range(k)]
            thr = [0 if i < c else sizes[c] - s if i == c else sizes[i] - 1 for i in range(k)]
            region = tuple(slice(t, N) for t, N in zip(thr, shape))
            out.append((region, math.prod(ext), math.prod(N - t for t, N in zip(thr, shape))))
    return out


def _kd_values(xt: torch.Tensor, exps, prec: int, scale: float) -> torch.Tensor:
    """Unnormalized-then-scaled coefficients of a k-D device array (k >= 1)."""
    k = len(exps)
    dev = xt.device
    odt = _OUT_DTYPES[prec]
    if k == 1:
        (m,) = exps
        N = xt.shape[0]
        out = torch.empty((1, N - (1 << m) + 1, 1, 1 << m), dtype=odt, device=dev)
        forward_into(xt.reshape(1, N), 0, m, out, prec=prec, scale=scale)
        return out.view(N - (1 << m) + 1, 1 << m)
    if k == 2:
        m0, m1 = exps
        out = torch.empty((xt.shape[0] - (1 << m0) + 1, xt.shape[1] - (1 << m1) + 1, 1 << m0,
                           1 << m1), dtype=odt, device=dev)
        forward_into(xt if xt.stride(-1) == 1 else xt.contiguous(), m0, m1, out, prec=prec,
                     scale=scale)
        return out
    m0 = exps[0]
    n0 = 1 << m0
    N0 = xt.shape[0]
    P0 = N0 - n0 + 1
    inner = torch.stack([_kd_values(xt[i], exps[1:], prec, 1.0) for i in range(N0)])
    inner_shape = inner.shape[1:]  # (P1 .. P_{k-1}, n1 .. n_{k-1})
    M = math.prod(inner_shape)
    col = torch.empty((P0, M, n0, 1), dtype=odt, device=dev)
    forward_into(inner.reshape(N0, M), m0, 0, col, prec=prec, scale=scale)
    kk = k - 1
    # [P0, P1.., n1.., n0] -> [P0, P1.., n0, n1..]
    v = col.view((P0,) + tuple(inner_shape) + (n0,))
    perm = [0] + [1 + i for i in range(kk)] + [1 + 2 * kk] + [1 + kk + i for i in range(kk)]
    return v.permute(perm).contiguous()


def tree_swdft_kd(x, spec, counter=None, budget=None, *, precision=None,
                  device=None) -> CoefficientArray:
    """k-dimensional sliding-window DFT on the GPU (treekd.py:102-121 interface)."""
    xt = _to_tensor(x)
    k = len(spec.exponents)
    if xt.dim() != k:
        raise core.ShapeError(f"{k}-dimensional window applied to {xt.dim()}-dimensional array")
    shape = tuple(int(s) for s in xt.shape)
    spec.check_fits(shape)
    required = 2 * math.prod(shape) * (1 << sum(spec.exponents)) * core.COMPLEX_BYTES + \
        core.output_bytes(shape, spec)
    core.check_budget(required, budget, what="level buffers + coefficient output")
    prec = _precision_code(precision, xt.dtype)
    if device is None:
        device = xt.device if xt.is_cuda else torch.device("cuda", torch.cuda.current_device())
    xt = xt.to(device)
    values = _kd_values(xt, tuple(int(m) for m in spec.exponents), prec,
                        core.normalization_factor(spec))
    if counter is not None:
        for region, nodes, positions in level_regions_kd(shape, spec.exponents):
            counter.add_region(region, nodes, positions)
    return CoefficientArray(values, shape, spec, spec.normalization)
