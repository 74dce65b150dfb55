"""B200-native 2D tree sliding-window DFT (Richardson & Eddy, arXiv:1707.08213).

Drop-in for the reference's batch path ``swdft.tree2d.tree_swdft_2d``
(/root/reference/pkg/src/swdft/tree2d.py:175-202).  The compute lives in
``libswdft2d.so`` (sm_100a CUDA kernels behind the C ABI in include/swdft2d.h);
this package is the host-side mirror of the reference's interface plus the
multi-GPU strip partitioner.
"""
from .core import (BudgetError, CoefficientArray, ContainerError, DeviceError, InvalidWindowError, OpCounter,
                   ShapeError, StateError, SwdftError, UnsupportedError, WindowSpec,
                   WindowTooLargeError, normalization_factor)
from .tree2d import LOOP_ORDERS, forward_into, tree_swdft_2d

__all__ = [
    "BudgetError", "CoefficientArray", "ContainerError", "DeviceError", "InvalidWindowError", "OpCounter",
    "ShapeError", "StateError", "SwdftError", "UnsupportedError", "WindowSpec",
    "WindowTooLargeError", "normalization_factor", "LOOP_ORDERS", "forward_into",
    "tree_swdft_2d",
]
