"""1D tree sliding-window DFT through the 2D kernel (the m0 = 0 case).

Drop-in for the reference's ``tree1d.tree_swdft_1d`` (/root/reference/pkg/src/
swdft/tree1d.py:29-60): a length-N signal is a 1 x N array with a 1 x n window,
whose row-level tree (dim 1) is exactly the 1D tree's DAG (tree1d.py:49-56 vs
tree2d.py:72-93), so the fp64 output is bitwise the reference's.
"""
from __future__ import annotations

import torch

from . import core
from .core import CoefficientArray
from .tree2d import _OUT_DTYPES, _precision_code, _to_tensor, forward_into


def tree_swdft_1d(x, spec, counter=None, *, precision=None, device=None) -> CoefficientArray:
    xt = _to_tensor(x)
    if xt.dim() != 1 or len(spec.exponents) != 1:
        raise core.ShapeError("tree_swdft_1d expects a 1D signal and 1D window")
    spec.check_fits(tuple(xt.shape))
    (m,) = (int(v) for v in spec.exponents)
    n, N = 1 << m, int(xt.shape[0])
    prec = _precision_code(precision, xt.dtype)
    if device is None:
        device = xt.device if xt.is_cuda else torch.device("cuda", torch.cuda.current_device())
    xt = xt.to(device).reshape(1, N)
    out = torch.empty((1, N - n + 1, 1, n), dtype=_OUT_DTYPES[prec], device=device)
    forward_into(xt, 0, m, out, prec=prec, scale=core.normalization_factor(spec))
    if counter is not None:  # tree1d.py:54-55, one region per level
        for l in range(1, m + 1):
            s, L = 1 << (m - l), 1 << l
            counter.add_region((slice(n - s, N),), L, N - (n - s))
    return CoefficientArray(out.view(N - n + 1, n), (N,), spec, spec.normalization)
