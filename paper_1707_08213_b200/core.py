"""Host-side mirror of the reference's domain types for the 2D tree SWDFT path.

Same names, arguments, error classes and messages as the reference's
``swdft.core`` (/root/reference/pkg/src/swdft/core.py), restated for this
package so that the drop-in ``tree_swdft_2d`` behaves like the reference's on
the boundary (validation, budget accounting, normalization bookkeeping)
without importing it.  Only what the batch 2D path touches is here.
"""
from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Iterable, Sequence

COMPLEX_BYTES = 16  # the reference accounts every complex at 16 B (core.py:17)
DEFAULT_BUDGET_BYTES = 4 * 1024**3  # core.py:18
NORMALIZATION_MODES = ("none", "paper-1d", "paper-2d", "unitary")  # core.py:20


class SwdftError(Exception):
    """Base class for package errors (core.py:23)."""


class InvalidWindowError(SwdftError, ValueError):
    """Window size not a power of two, or an inconsistent window spec (core.py:27)."""


class WindowTooLargeError(SwdftError, ValueError):
    """Window exceeds the array extent in some dimension (core.py:31)."""


class ShapeError(SwdftError, ValueError):
    """Input shape does not match what the operation expects (core.py:35)."""


class StateError(SwdftError, RuntimeError):
    """Operation applied out of order (core.py:39)."""


class ContainerError(SwdftError, ValueError):
    """Malformed SWDF container, bad CSV, or non-finite payload (core.py:44)."""


class BudgetError(SwdftError):
    """Projected allocation exceeds the configured memory budget (core.py:48-56)."""

    def __init__(self, required_bytes: int, budget_bytes: int, what: str = "allocation"):
        self.required_bytes = int(required_bytes)
        self.budget_bytes = int(budget_bytes)
        super().__init__(
            f"{what} requires {self.required_bytes} bytes; budget is {self.budget_bytes} bytes")


class DeviceError(SwdftError, RuntimeError):
    """CUDA failure inside libswdft2d.so (no reference counterpart)."""


class UnsupportedError(SwdftError, ValueError):
    """Shape outside the CUDA paths of libswdft2d.so (no reference counterpart)."""


def is_power_of_two(n: int) -> bool:
    return n >= 1 and (n & (n - 1)) == 0


@dataclass(frozen=True)
class WindowSpec:
    """Per-dimension window exponents, sizes n_i = 2**m_i (core.py:63-122)."""

    exponents: tuple
    normalization: str = "none"

    def __post_init__(self):
        exps = tuple(int(m) for m in self.exponents)
        object.__setattr__(self, "exponents", exps)
        if len(exps) < 1:
            raise InvalidWindowError("a window needs at least one dimension")
        if any(m < 0 for m in exps):
            raise InvalidWindowError(f"window exponents must be non-negative, got {exps}")
        if self.normalization not in NORMALIZATION_MODES:
            raise InvalidWindowError(f"unknown normalization mode {self.normalization!r}")
        if self.normalization == "paper-1d" and len(exps) != 1:
            raise InvalidWindowError("paper-1d normalization applies to 1D windows only")
        if self.normalization == "paper-2d" and len(exps) < 2:
            raise InvalidWindowError("paper-2d normalization needs at least two dimensions")

    @classmethod
    def from_sizes(cls, sizes: Iterable[int], normalization: str = "none") -> "WindowSpec":
        exps = []
        for n in sizes:
            n = int(n)
            if not is_power_of_two(n):
                raise InvalidWindowError(f"window size {n} is not a power of two")
            exps.append(n.bit_length() - 1)
        return cls(tuple(exps), normalization)

    @property
    def k(self) -> int:
        return len(self.exponents)

    @property
    def sizes(self) -> tuple:
        return tuple(1 << m for m in self.exponents)

    @property
    def total_levels(self) -> int:
        return sum(self.exponents)

    @property
    def window_elements(self) -> int:
        return 1 << self.total_levels

    def check_fits(self, shape: Sequence[int]) -> None:
        if len(shape) != self.k:
            raise ShapeError(
                f"{self.k}-dimensional window applied to {len(shape)}-dimensional array")
        for d, (n, ext) in enumerate(zip(self.sizes, shape)):
            if n > ext:
                raise WindowTooLargeError(f"window size {n} exceeds extent {ext} in dimension {d}")


def normalization_factor(spec) -> float:
    """core.py:249-255."""
    mode = spec.normalization
    if mode == "none":
        return 1.0
    if mode == "paper-1d":
        return 1.0 / spec.sizes[0]
    return 1.0 / math.sqrt(float(1 << sum(spec.exponents)))


@dataclass
class CoefficientArray:
    """Windowed DFT coefficients (core.py:258-285).

    ``values`` has shape P_0 x P_1 x n_0 x n_1 (P_i = N_i - n_i + 1); here it is
    normally a device-resident ``torch.Tensor`` (complex64 or complex128).
    """

    values: object
    source_shape: tuple
    window: WindowSpec
    normalization: str = "none"

    def __post_init__(self):
        self.source_shape = tuple(int(e) for e in self.source_shape)
        k = len(self.window.exponents)
        if self.values.ndim != 2 * k:
            raise ShapeError(f"expected {2 * k} axes, got {self.values.ndim}")
        expected = self.positions + tuple(self.window.sizes)
        if tuple(self.values.shape) != expected:
            raise ShapeError(f"coefficient shape {tuple(self.values.shape)} != expected {expected}")
        if self.normalization not in NORMALIZATION_MODES:
            raise InvalidWindowError(f"unknown normalization mode {self.normalization!r}")

    @property
    def positions(self) -> tuple:
        return tuple(N - n + 1 for N, n in zip(self.source_shape, self.window.sizes))

    def numpy(self):
        """``values`` as a numpy array, the reference's own return type: a device tensor
        is copied out through swdft2d_download (pinned staging + worker threads)."""
        if hasattr(self.values, "is_cuda"):
            from . import _lib

            return _lib.download(self.values)
        return self.values


def output_elements(shape: Sequence[int], spec) -> int:
    spec.check_fits(shape)
    positions = math.prod(N - n + 1 for N, n in zip(shape, spec.sizes))
    return positions * (1 << sum(spec.exponents))


def output_bytes(shape: Sequence[int], spec) -> int:
    """core.py:370-371 (16 B per complex, the reference's accounting)."""
    return output_elements(shape, spec) * COMPLEX_BYTES


def lattice_bytes(shape: Sequence[int], spec) -> int:
    """core.py:374-381: the reference's double-buffered lattice, 2*prod(N)*prod(n)."""
    spec.check_fits(shape)
    return 2 * math.prod(shape) * (1 << sum(spec.exponents)) * COMPLEX_BYTES


def check_budget(required_bytes: int, budget_bytes, what: str = "allocation") -> None:
    """core.py:384-388."""
    if budget_bytes is None:
        budget_bytes = DEFAULT_BUDGET_BYTES
    if required_bytes > budget_bytes:
        raise BudgetError(required_bytes, budget_bytes, what=what)


class OpCounter:
    """Mirror of the reference's bench.OpCounter (bench.py:25-44): tally of
    butterfly arms, optionally attributed per window position."""

    def __init__(self, position_shape=None):
        import numpy as np

        self.total = 0
        self.position_ops = (np.zeros(position_shape, dtype=np.int64)
                             if position_shape is not None else None)

    def add(self, count: int) -> None:
        self.total += int(count)

    def add_region(self, region, nodes_per_tree: int, positions: int) -> None:
        self.total += int(nodes_per_tree) * int(positions)
        if self.position_ops is not None:
            self.position_ops[region] += nodes_per_tree


def level_regions(shape: Sequence[int], spec):
    """Per tree level (1..m0+m1): the (region, nodes_per_tree, positions) the
    reference's levels-outer schedule reports (tree2d.py:90-92, 115-118),
    i.e. core.level_geometry's validity thresholds (core.py:197-215)."""
    N0, N1 = (int(s) for s in shape)
    m0, m1 = spec.exponents
    n0, n1 = 1 << m0, 1 << m1
    out = []
    for t in range(1, m1 + 1):  # row levels, dim 1
        s, L = 1 << (m1 - t), 1 << t
        lo = n1 - s
        out.append(((slice(0, N0), slice(lo, N1)), L, N0 * (N1 - lo)))
    for q in range(1, m0 + 1):  # column levels, dim 0
        s, L = 1 << (m0 - q), 1 << q
        lo = n0 - s
        out.append(((slice(lo, N0), slice(n1 - 1, N1)), L * n1, (N0 - lo) * (N1 - n1 + 1)))
    return out
