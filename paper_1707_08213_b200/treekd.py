"""k-dimensional tree sliding-window DFT by composition of the 2D kernel.

Drop-in for the reference's ``treekd.tree_swdft_kd`` (/root/reference/pkg/src/
swdft/treekd.py:102-121).  The reference's level plan gives dimension k-1 the
first block of levels and dimension 0 the last (core.py:150-161), and every level
combines positions along its own dimension only.  So for k >= 3:

  1. levels of dims k-1 .. 1 act on each slice x[i0] independently: they are the
     (k-1)-dimensional tree of that slice (computed recursively; for k = 3 all
     slices go through one K1 launch over the slices stacked as a 2-D array);
  2. levels of dim 0 are, for every (p_1.., k_1..) column of the stacked slice
     results, the 1D tree along i0 with window n0 — the column-tree kernel KC
     (swdft2d_forward_columns) on the [N0, prod(inner)] matrix of slice results,
     which writes k0 straight into axis k (no separate transpose pass).

Each node is computed by the same butterfly with the same operands as in the
reference's lattice, so fp64 output is bit-identical (tests/test_next_rows.py).
The normalization factor is applied once, in the last (dim-0) pass.
"""
from __future__ import annotations

import math

import torch

from . import _lib, core
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


def _kd_values(xt: torch.Tensor, exps, prec: int, scale: float, out=None) -> torch.Tensor:
    """Unnormalized-then-scaled coefficients of a k-D device array (k >= 1), written into
    ``out`` (shape (P_0.., n_0..)) when given."""
    k = len(exps)
    dev = xt.device
    odt = _OUT_DTYPES[prec]
    sizes = [1 << m for m in exps]
    P = [int(N) - n + 1 for N, n in zip(xt.shape, sizes)]
    if out is None:
        out = torch.empty(tuple(P) + tuple(sizes), dtype=odt, device=dev)
    if k == 1:
        (m,) = exps
        forward_into(xt.reshape(1, -1), 0, m, out.view(1, P[0], 1, sizes[0]), prec=prec,
                     scale=scale)
        return out
    if k == 2:
        forward_into(xt if xt.stride(-1) == 1 else xt.contiguous(), exps[0], exps[1], out,
                     prec=prec, scale=scale)
        return out
    # dims k-1 .. 1: the (k-1)-D tree of every slice x[i0], straight into the stacked
    # matrix of slice results; then dim 0 down its columns with k0 put in place (KC)
    m0, n0, N0, P0 = exps[0], sizes[0], int(xt.shape[0]), P[0]
    M = math.prod(P[1:]) * math.prod(sizes[1:])
    if k == 3:
        # every slice's 2-D transform in ONE K1 launch: the slices stacked as an
        # (N0 N1) x N2 array; window rows that straddle two slices are computed into
        # the gap rows (p1 >= P1 of each slice) and never read
        N1, N2 = int(xt.shape[1]), int(xt.shape[2])
        x2 = xt.contiguous().view(N0 * N1, N2)
        ld = N1 * P[2] * sizes[1] * sizes[2]
        stacked = torch.empty((N0 * N1, P[2], sizes[1], sizes[2]), dtype=odt, device=dev)
        forward_into(x2, exps[1], exps[2], stacked[:N0 * N1 - sizes[1] + 1], prec=prec)
        inner = stacked.view(N0, ld)[:, :M]
    else:
        inner = torch.empty((N0,) + tuple(P[1:]) + tuple(sizes[1:]), dtype=odt, device=dev)
        for i in range(N0):
            _kd_values(xt[i], exps[1:], prec, 1.0, out=inner[i])
        inner = inner.view(N0, M)
        ld = M
    if m0 == 0:
        v = inner.reshape(out.shape)
        return out.copy_(v * scale if scale != 1.0 else v)
    lib = _lib.load()
    with torch.cuda.device(dev):
        rc = lib.swdft2d_forward_columns(inner.data_ptr(), prec, N0, M, ld, m0, sum(exps[1:]),
                                         float(scale), 0, P0, out.data_ptr(),
                                         torch.cuda.current_stream(dev).cuda_stream)
    _lib.check(rc)
    return out


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
