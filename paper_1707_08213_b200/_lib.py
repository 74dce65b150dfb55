"""ctypes binding of libswdft2d.so (include/swdft2d.h).

The library is built in-tree (``python -m paper_1707_08213_b200.build``).  There
is no CPU fallback: if the library is missing or cannot be loaded, importing
the compute entry points raises.
"""
from __future__ import annotations

import ctypes
import os

from . import core

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SWDFT2D_LIB", os.path.join(_HERE, "libswdft2d.so"))

ABI_VERSION = 1

OK = 0
E_INVALID_ARG = -1
E_SHAPE = -2
E_WINDOW_TOO_LARGE = -3
E_INVALID_WINDOW = -4
E_UNSUPPORTED = -6
E_CUDA = -7
E_NOMEM = -8

IN_F32, IN_F64, IN_C64, IN_C128 = 0, 1, 2, 3
K1_MAX_M, K0_MAX_M = 6, 10  # SWDFT2D_K1_MAX_M / SWDFT2D_K0_MAX_M
PREC_FP32, PREC_FP64 = 0, 1
KERNEL_AUTO, KERNEL_STREAM, KERNEL_WINDOW, KERNEL_STREAM_TMA, KERNEL_ROWS = 0, 1, 2, 3, 4
KERNEL_SEPARABLE = 5
KERNELS = {"auto": KERNEL_AUTO, "stream": KERNEL_STREAM, "window": KERNEL_WINDOW,
           "stream_tma": KERNEL_STREAM_TMA, "rows": KERNEL_ROWS, "separable": KERNEL_SEPARABLE}

# every symbol include/swdft2d.h declares: name -> (restype, argtypes)
_i64, _int, _dbl, _vp = ctypes.c_int64, ctypes.c_int, ctypes.c_double, ctypes.c_void_p
_pi64 = ctypes.POINTER(ctypes.c_int64)
SIGNATURES = {
    "swdft2d_abi_version": (_int, []),
    "swdft2d_last_error": (ctypes.c_char_p, []),
    "swdft2d_output_shape": (_int, [_i64, _i64, _int, _int, _pi64, _pi64]),
    "swdft2d_reference_bytes": (_int, [_i64, _i64, _int, _int, _pi64, _pi64]),
    "swdft2d_twiddles": (_int, [_int, ctypes.POINTER(ctypes.c_double)]),
    "swdft2d_forward": (_int, [_vp, _int, _i64, _i64, _i64, _int, _int, _int, _dbl, _i64, _i64,
                               _vp, _int, _vp]),
    "swdft2d_forward_ws": (_int, [_vp, _int, _i64, _i64, _i64, _int, _int, _int, _dbl, _i64,
                                  _i64, _vp, _vp, _i64, _int, _vp]),
    "swdft2d_forward_host": (_int, [_vp, _int, _i64, _i64, _i64, _int, _int, _int, _dbl, _i64,
                                    _i64, _vp, _i64, _int, _vp]),
    "swdft2d_download": (_int, [_vp, _vp, _i64, _vp]),
    "swdft2d_host_alloc": (_vp, [_i64]),
    "swdft2d_host_free": (_int, [_vp]),
    "swdft2d_workspace_bytes": (_int, [_i64, _i64, _int, _int, _int, _i64, _i64, _int, _pi64]),
    "swdft2d_k1_schedule": (_int, [_i64, _i64, _int, _int, _int, _i64, _i64, _pi64, _pi64,
                                   _int]),
    "swdft2d_has_stream_kernel": (_int, [_int, _int, _int]),
    "swdft2d_stream_kernel_info": (_int, [_int, _int, _int, _pi64]),
    "swdft2d_strip_range": (_int, [_i64, _int, _int, _int, _pi64]),
    "swdft2d_forward_multi": (_int, [_vp, _int, _i64, _i64, _i64, _int, _int, _int, _dbl, _int,
                                     ctypes.POINTER(ctypes.c_int), ctypes.POINTER(_vp),
                                     ctypes.POINTER(_vp), ctypes.POINTER(_vp)]),
    "swdft2d_stream_push": (_int, [_vp, _int, _i64, _vp, _vp, _int, _int, _int, _dbl, _i64, _vp,
                                   _int, _vp]),
    "swdft2d_stream_state_bytes": (_int, [_i64, _int, _int, _int, _pi64]),
    "swdft2d_forward_columns": (_int, [_vp, _int, _i64, _i64, _i64, _int, _int, _dbl, _i64, _i64,
                                       _vp, _vp]),
    "swdft2d_shutdown": (_int, []),
}

_lib = None


def load() -> ctypes.CDLL:
    """Load libswdft2d.so (once).  Raises ImportError when it is absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} not found: build it with `python -m paper_1707_08213_b200.build` "
            "(there is no CPU fallback for the SWDFT path)")
    lib = ctypes.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    v = lib.swdft2d_abi_version()
    if v != ABI_VERSION:
        raise ImportError(f"libswdft2d.so ABI {v} != expected {ABI_VERSION}")
    _lib = lib
    return lib


def last_error() -> str:
    return load().swdft2d_last_error().decode(errors="replace")


def check(rc: int) -> None:
    """Map a status code onto the reference's exception classes (core.py:23-56)."""
    if rc == OK:
        return
    msg = last_error()
    if rc == E_SHAPE:
        raise core.ShapeError(msg)
    if rc == E_WINDOW_TOO_LARGE:
        raise core.WindowTooLargeError(msg)
    if rc == E_INVALID_WINDOW:
        raise core.InvalidWindowError(msg)
    if rc == E_INVALID_ARG:
        raise ValueError(msg)
    if rc == E_UNSUPPORTED:
        raise core.UnsupportedError(msg)
    if rc in (E_CUDA, E_NOMEM):
        raise core.DeviceError(msg)
    raise core.SwdftError(f"libswdft2d error {rc}: {msg}")


def strip_range(P0: int, m0: int, rank: int, world: int):
    """(p0_begin, p0_end, row_begin, row_end) of one rank (swdft2d_strip_range)."""
    buf = (ctypes.c_int64 * 4)()
    check(load().swdft2d_strip_range(P0, m0, rank, world, buf))
    return tuple(int(v) for v in buf)


def twiddles(n: int):
    import numpy as np

    out = np.empty(2 * n, dtype=np.float64)
    check(load().swdft2d_twiddles(n, out.ctypes.data_as(ctypes.POINTER(ctypes.c_double))))
    t = np.empty(n, dtype=np.complex128)
    t.real = out[0::2]
    t.imag = out[1::2]
    return t


def has_stream_kernel(m0: int, m1: int, prec: int) -> bool:
    return bool(load().swdft2d_has_stream_kernel(m0, m1, prec))


def stream_kernel_info(m0: int, m1: int, prec: int) -> dict:
    buf = (ctypes.c_int64 * 6)()
    check(load().swdft2d_stream_kernel_info(m0, m1, prec, buf))
    return {"Q": int(buf[0]), "J": 1 << int(buf[0]), "TP1": int(buf[1]), "threads": int(buf[2]),
            "smem_bytes_ldg": int(buf[3]), "NB": int(buf[4]), "tma_input_staging": bool(buf[5])}


def workspace_bytes(N0: int, N1: int, m0: int, m1: int, prec: int, p0_begin: int, p0_end: int,
                    kernel: int = KERNEL_AUTO) -> int:
    """Device workspace swdft2d_forward_ws uses for this call (0: the path needs none)."""
    v = ctypes.c_int64()
    check(load().swdft2d_workspace_bytes(N0, N1, m0, m1, prec, p0_begin, p0_end, kernel,
                                         ctypes.byref(v)))
    return int(v.value)


K1_MODES = {0: "uniform", 1: "guided", 2: "oneshot", 3: "streamk"}


def k1_schedule(N0: int, N1: int, m0: int, m1: int, prec: int, p0_begin: int = 0,
                p0_end: int | None = None) -> dict:
    """The K1 launch schedule swdft2d_forward picks on the current device
    (swdft2d_k1_schedule): mode, rows per tile, chunk row bounds (relative to p0_begin),
    tiles, grid, column blocks, CTA slots, CTAs per SM."""
    if p0_end is None:
        p0_end = N0 - (1 << m0) + 1
    info = (ctypes.c_int64 * 8)()
    rows = p0_end - p0_begin
    cap = rows + 2
    bounds = (ctypes.c_int64 * cap)()
    check(load().swdft2d_k1_schedule(N0, N1, m0, m1, prec, p0_begin, p0_end, info, bounds, cap))
    nch = int(info[2])
    return {"mode": K1_MODES[int(info[0])], "rows_per_tile": int(info[1]), "chunks": nch,
            "bounds": [int(bounds[c]) for c in range(nch + 1)], "tiles": int(info[3]),
            "grid": int(info[4]), "column_blocks": int(info[5]), "slots": int(info[6]),
            "ctas_per_sm": int(info[7])}


def raw_stream(device_index: int) -> int:
    """cudaStream_t (as an int) of torch's current stream on a device, without the
    Python-side overhead of torch.cuda.current_stream (which dominated a stream push)."""
    import torch

    get = getattr(torch._C, "_cuda_getCurrentRawStream", None)
    if get is not None:
        return get(device_index)
    return torch.cuda.current_stream(device_index).cuda_stream


def host_empty(shape, dtype):
    """numpy array over pinned host memory from swdft2d_host_alloc (freed with the array):
    the output buffer swdft2d_forward_host fills at the PCIe rate."""
    import weakref

    import numpy as np

    dtype = np.dtype(dtype)
    n = int(np.prod(shape, dtype=np.int64)) * dtype.itemsize
    if n == 0:
        return np.empty(shape, dtype=dtype)
    lib = load()
    ptr = lib.swdft2d_host_alloc(n)
    if not ptr:
        raise core.DeviceError(last_error())
    buf = (ctypes.c_char * n).from_address(ptr)
    weakref.finalize(buf, lib.swdft2d_host_free, ptr)  # buf lives as long as any view of it
    return np.frombuffer(buf, dtype=dtype).reshape(shape)


NP_IN_CODES = {"float32": IN_F32, "float64": IN_F64, "complex64": IN_C64, "complex128": IN_C128}


def forward_host(x, m0: int, m1: int, out, *, prec: int, scale: float = 1.0, p0_begin: int = 0,
                 p0_end: int | None = None, strip_bytes: int = 0, kernel: int = KERNEL_AUTO,
                 stream: int | None = None):
    """swdft2d_forward_host on numpy arrays: ``x`` a 2D float32/float64/complex64/complex128
    array whose rows are contiguous (any row stride), ``out`` a C-contiguous complex array of
    (p0_end - p0_begin, P1, n0, n1) of the precision (pinned — host_empty — for the PCIe
    rate).  Synchronous; ``stream`` (a cudaStream_t as int) orders the compute."""
    code = NP_IN_CODES.get(x.dtype.name)
    if code is None or x.ndim != 2:
        raise ValueError(f"forward_host needs a 2D f32/f64/c64/c128 array, got {x.dtype} {x.shape}")
    N0, N1 = x.shape
    ld = x.strides[0] // x.itemsize if N0 > 1 else N1
    if (N1 > 1 and x.strides[1] != x.itemsize) or \
            (N0 > 1 and (x.strides[0] % x.itemsize or ld < N1)):
        raise ValueError("forward_host needs contiguous rows at a row stride >= the width")
    n0, n1 = 1 << m0, 1 << m1
    if p0_end is None:
        p0_end = N0 - n0 + 1
    want = (p0_end - p0_begin, N1 - n1 + 1, n0, n1)
    odt = "complex64" if prec == PREC_FP32 else "complex128"
    if tuple(out.shape) != want or out.dtype.name != odt or not out.flags.c_contiguous or \
            not out.flags.writeable:
        raise ValueError(f"out must be a writable C-contiguous {odt} array of shape {want}")
    check(load().swdft2d_forward_host(x.ctypes.data, code, N0, N1, ld, m0,
                                      m1, prec, float(scale), p0_begin, p0_end, out.ctypes.data,
                                      strip_bytes, kernel, stream))
    return out


def download(t):
    """CUDA tensor -> fresh numpy array through swdft2d_download (staged by worker threads:
    several times the rate of ``t.cpu()`` into fresh pageable memory)."""
    import numpy as np
    import torch

    if not t.is_cuda:
        return t.numpy()
    t = t.contiguous()
    out = np.empty(tuple(t.shape), dtype=torch.empty((), dtype=t.dtype).numpy().dtype)
    if out.nbytes:
        with torch.cuda.device(t.device):
            check(load().swdft2d_download(t.data_ptr(), out.ctypes.data, out.nbytes,
                                          raw_stream(t.device.index)))
    return out
