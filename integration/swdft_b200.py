"""Reference-side binding: the reference package's own ``swdft.tree2d.tree_swdft_2d``
(and its 1D / kD siblings ``swdft.tree1d.tree_swdft_1d``, ``swdft.treekd.tree_swdft_kd``)
served by libswdft2d.so on a B200.

This is the module a ``swdft`` maintainer would add: it keeps the
reference's entry point, types and exceptions, and swaps only the compute.  After

    import swdft.tree2d
    import swdft_b200            # this file (integration/ on sys.path)
    swdft_b200.enable()

a caller of ``swdft.tree2d.tree_swdft_2d(x, spec, ...)`` (``/root/reference/pkg/src/
swdft/tree2d.py:175-202``) gets:
  * the reference's validation, in its order and with its exception classes
    (``swdft.core.ShapeError`` / ``WindowTooLargeError`` via ``spec.check_fits`` /
    ``ValueError`` for ``loop_order`` / ``swdft.core.BudgetError`` from the reference's
    own ``check_budget`` on the reference's own byte accounting), run by calling the
    reference's functions themselves (``tree2d.py:189-196``);
  * a ``swdft.core.CoefficientArray`` (``core.py:258-285``) whose ``values`` are
    complex128 ``[P0, P1, n0, n1]``, bitwise equal to the reference (the fp64 kernels
    compute every node with the reference's rounding, ``core.py:223-246``; the
    normalization factor is applied per component in the store epilogue, bitwise equal
    to ``core.normalize``, ``core.py:288-302``), recorded with ``spec.normalization``;
  * the same ``counter.add_region`` calls as ``_levels_outer`` (``tree2d.py:90-92,
    115-118``), replayed from the reference's own ``core.shift_schedule``.

The stream classes ``swdft.tree2d.SlidingRowStream2D`` (``tree2d.py:205-303``) and
``swdft.tree1d.SlidingStream1D`` (``tree1d.py:63-119``) are routed too: same constructors,
attributes, exceptions and per-push accounting, slabs / vectors bitwise equal to the batch
transform's rows.

``values`` is a numpy array, as the reference returns, unless ``enable(values="device")``
(then a CUDA tensor stays in HBM; ``CoefficientArray`` accepts it).  ``loop_order`` is
validated and then has no effect (the reference's two orders are bitwise identical);
``threads`` is accepted and ignored.  There is no CPU fallback: if libswdft2d.so
cannot be loaded, ``enable()`` raises ImportError.
"""
from __future__ import annotations

import functools
import importlib
import os
import sys

_ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if _ROOT not in sys.path:
    sys.path.insert(0, _ROOT)

_STATE = {"orig": None, "values": "numpy", "precision": "fp64", "device": None}


def _replay_counter(counter, core, shape, spec) -> None:
    """The add_region calls of the reference's levels-outer schedule (tree2d.py:90-92,
    115-118): one per level, region = the level's validity thresholds onward."""
    N0, N1 = shape
    for g in core.shift_schedule(spec)[1:]:
        t0, t1 = g.thresholds
        counter.add_region((slice(t0, N0), slice(t1, N1)), g.nodes_per_tree,
                           (N0 - t0) * (N1 - t1))


def tree_swdft_2d_b200(x, spec, loop_order: str = "levels-outer", counter=None,
                       budget: int | None = None, threads: int = 1):
    """swdft.tree2d.tree_swdft_2d (tree2d.py:175-202) with the compute on the B200."""
    import numpy as np
    import torch
    from swdft import core, tree2d

    from paper_1707_08213_b200 import _lib
    from paper_1707_08213_b200.tree2d import _IN_CODES, _precision_code, forward_into

    # tree2d.py:189-196, verbatim order, the reference's own checks and exceptions
    x = np.asarray(x, dtype=np.complex128)
    if x.ndim != 2 or spec.k != 2:
        raise core.ShapeError("tree_swdft_2d expects a 2D array and 2D window")
    spec.check_fits(x.shape)
    if loop_order not in tree2d.LOOP_ORDERS:
        raise ValueError(f"loop_order must be one of {tree2d.LOOP_ORDERS}")
    required = core.lattice_bytes(x.shape, spec) + core.output_bytes(x.shape, spec)
    core.check_budget(required, budget, what="level buffers + coefficient output")

    m0, m1 = (int(m) for m in spec.exponents)
    n0, n1 = spec.sizes
    N0, N1 = x.shape
    P0, P1 = N0 - n0 + 1, N1 - n1 + 1
    prec = _precision_code(_STATE["precision"], torch.complex128)
    dev = _STATE["device"] or torch.device("cuda", torch.cuda.current_device())
    odt = torch.complex128 if prec == _lib.PREC_FP64 else torch.complex64
    scale = float(core.normalization_factor(spec))
    if _STATE["values"] == "device":
        xd = torch.from_numpy(np.ascontiguousarray(x)).to(dev)
        assert xd.dtype in _IN_CODES
        values = torch.empty((P0, P1, n0, n1), dtype=odt, device=dev)
        forward_into(xd, m0, m1, values, prec=prec, scale=scale)
    else:
        # numpy in, a fresh numpy array out, as the reference returns: ONE C-ABI call
        # (swdft2d_forward_host); the device holds a ring of strips, never the whole output
        values = np.empty((P0, P1, n0, n1),
                          dtype=np.complex128 if prec == _lib.PREC_FP64 else np.complex64)
        di = torch.device(dev).index
        di = torch.cuda.current_device() if di is None else di
        with torch.cuda.device(di):
            _lib.forward_host(np.ascontiguousarray(x), m0, m1, values, prec=prec, scale=scale,
                              stream=_lib.raw_stream(di))
    if counter is not None:
        _replay_counter(counter, core, x.shape, spec)
    # normalize() would have produced this record: values scaled, mode recorded
    return core.CoefficientArray(values, x.shape, spec, spec.normalization)


def _host_or_device(values):
    if _STATE["values"] == "device":
        return values
    from paper_1707_08213_b200 import _lib

    return _lib.download(values)  # swdft2d_download: staged, not a pageable cudaMemcpy


def tree_swdft_1d_b200(x, spec, counter=None):
    """swdft.tree1d.tree_swdft_1d (tree1d.py:29-60) with the compute on the B200 (the 1D
    tree is the m0 = 0 case of the 2D kernels; bitwise in fp64)."""
    import numpy as np
    from swdft import core

    from paper_1707_08213_b200 import tree1d as b200_1d

    x = np.asarray(x, dtype=np.complex128)  # tree1d.py:36-39, the reference's own checks
    if x.ndim != 1 or spec.k != 1:
        raise core.ShapeError("tree_swdft_1d expects a 1D signal and 1D window")
    spec.check_fits(x.shape)
    r = b200_1d.tree_swdft_1d(x, spec, counter, precision=_STATE["precision"],
                              device=_STATE["device"])
    return core.CoefficientArray(_host_or_device(r.values), x.shape, spec, spec.normalization)


def tree_swdft_kd_b200(x, spec, counter=None, budget=None):
    """swdft.treekd.tree_swdft_kd (treekd.py:102-121) with the compute on the B200."""
    import numpy as np
    from swdft import core

    from paper_1707_08213_b200 import treekd as b200_kd

    x = np.asarray(x, dtype=np.complex128)  # treekd.py:109-116, the reference's own checks
    if x.ndim != spec.k:
        raise core.ShapeError(
            f"{spec.k}-dimensional window applied to {x.ndim}-dimensional array")
    spec.check_fits(x.shape)
    required = core.lattice_bytes(x.shape, spec) + core.output_bytes(x.shape, spec)
    core.check_budget(required, budget, what="level buffers + coefficient output")
    r = b200_kd.tree_swdft_kd(x, spec, counter, budget=1 << 62, precision=_STATE["precision"],
                              device=_STATE["device"])
    return core.CoefficientArray(_host_or_device(r.values), x.shape, spec, spec.normalization)


def _translate(exc):
    """This package's exception -> the reference's class of the same name (core.py:23-56)."""
    from swdft import core

    cls = getattr(core, type(exc).__name__, None)
    return cls(*exc.args) if isinstance(cls, type) and issubclass(cls, Exception) else exc


class SlidingRowStream2D_b200:
    """swdft.tree2d.SlidingRowStream2D (tree2d.py:205-303) on the B200: same constructor,
    attributes, exceptions, per-push operation accounting and counter calls; ``push_row``
    returns the (P1, n0, n1) slab (numpy, or a CUDA tensor with ``enable(values="device")``),
    bitwise equal to the batch transform's rows in fp64.  The reference's own
    class raises for every window larger than 1x1."""

    def __init__(self, spec, row_length: int, counter=None):
        from swdft import core

        from paper_1707_08213_b200 import stream as b200_stream

        if spec.k != 2:  # tree2d.py:217-226, the reference's own checks
            raise core.ShapeError("SlidingRowStream2D needs a 2D window spec")
        if spec.sizes[1] > int(row_length):
            raise core.WindowTooLargeError(
                f"window size {spec.sizes[1]} exceeds row length {int(row_length)}")
        self._s = b200_stream.SlidingRowStream2D(spec, row_length, counter,
                                                 precision=_STATE["precision"],
                                                 device=_STATE["device"])
        self.spec, self.counter = spec, counter
        self.m0, self.m1 = spec.exponents
        self.n0, self.n1 = spec.sizes
        self.N1 = int(row_length)

    rows_pushed = property(lambda self: self._s.rows_pushed)
    ops_last_push = property(lambda self: self._s.ops_last_push)
    last_push_position_ops = property(lambda self: self._s.last_push_position_ops)
    closed = property(lambda self: self._s.closed)

    def push_row(self, row):
        import numpy as np

        try:
            slab = self._s.push_row(np.asarray(row, dtype=np.complex128))
        except Exception as e:  # noqa: BLE001
            raise _translate(e) from None
        return None if slab is None else _host_or_device(slab)

    def close(self) -> None:
        self._s.close()


class SlidingStream1D_b200:
    """swdft.tree1d.SlidingStream1D (tree1d.py:63-119) on the B200."""

    def __init__(self, spec, counter=None):
        from swdft import core

        from paper_1707_08213_b200 import stream as b200_stream

        if spec.k != 1:
            raise core.ShapeError("SlidingStream1D needs a 1D window spec")
        self._s = b200_stream.SlidingStream1D(spec, counter, precision=_STATE["precision"],
                                              device=_STATE["device"])
        self.spec, self.counter = spec, counter
        (self.m,) = spec.exponents
        (self.n,) = spec.sizes

    pushed = property(lambda self: self._s.pushed)
    ops_last_push = property(lambda self: self._s.ops_last_push)
    closed = property(lambda self: self._s.closed)

    def push(self, sample):
        try:
            out = self._s.push(sample)
        except Exception as e:  # noqa: BLE001
            raise _translate(e) from None
        return None if out is None else _host_or_device(out)

    def close(self) -> None:
        self._s.close()


# (module, attribute, B200 function) the binding routes
_ROUTES = (("tree2d", "tree_swdft_2d", tree_swdft_2d_b200),
           ("tree1d", "tree_swdft_1d", tree_swdft_1d_b200),
           ("treekd", "tree_swdft_kd", tree_swdft_kd_b200),
           ("tree2d", "SlidingRowStream2D", SlidingRowStream2D_b200),
           ("tree1d", "SlidingStream1D", SlidingStream1D_b200))


def enable(values: str = "numpy", precision: str = "fp64", device=None) -> None:
    """Route swdft.tree2d.tree_swdft_2d, swdft.tree1d.tree_swdft_1d,
    swdft.treekd.tree_swdft_kd and the two stream classes (tree2d.SlidingRowStream2D,
    tree1d.SlidingStream1D) to libswdft2d.so (idempotent).

    values     "numpy" (the reference's return type) or "device" (a CUDA tensor)
    precision  "fp64" (complex128, bitwise equal to the reference) or "fp32"
               (complex64, within BASELINE.json's 1e-4 of each window's L2 norm)
    """
    if values not in ("numpy", "device"):
        raise ValueError("values must be 'numpy' or 'device'")
    if precision not in ("fp64", "fp32"):
        raise ValueError("precision must be 'fp64' or 'fp32'")
    from swdft import tree2d

    from paper_1707_08213_b200 import _lib

    _lib.load()  # no CPU fallback: fail here, loudly, if the library is missing
    _STATE.update(values=values, precision=precision, device=device)
    if _STATE["orig"] is None:
        _STATE["orig"] = tree2d.tree_swdft_2d
        _STATE["origs"] = {}
        for modname, attr, fn in _ROUTES:
            mod = importlib.import_module("swdft." + modname)
            orig = getattr(mod, attr)
            _STATE["origs"][(modname, attr)] = orig
            setattr(mod, attr, fn if isinstance(fn, type) else functools.wraps(orig)(fn))


def disable() -> None:
    """Restore the reference's numpy implementations."""
    if _STATE["orig"] is not None:
        for (modname, attr), orig in _STATE.pop("origs").items():
            setattr(importlib.import_module("swdft." + modname), attr, orig)
        _STATE["orig"] = None


def original(modname: str, attr: str):
    """The reference's own implementation behind a routed name (while enabled)."""
    return _STATE["origs"][(modname, attr)]


def enabled() -> bool:
    return _STATE["orig"] is not None
