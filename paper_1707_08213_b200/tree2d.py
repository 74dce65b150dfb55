"""Drop-in B200 replacement for the reference's batch 2D tree SWDFT.

    tree_swdft_2d(x, spec, loop_order="levels-outer", counter=None, budget=None,
                  threads=1, *, precision=None, device=None, out=None, kernel="auto",
                  devices=None)

mirrors /root/reference/pkg/src/swdft/tree2d.py:175-202: same arguments, the
same validation order and exceptions, the same [P0, P1, n0, n1] layout, twiddle
sign and index convention, the same budget accounting, the same OpCounter
calls, and the same normalization bookkeeping.  The compute runs in
libswdft2d.so on the current torch stream (K1, the fused streaming kernel, for
windows up to 64x64; KR for n0 = 1; KR + KC for larger windows up to 1024x1024);
``values`` of the returned CoefficientArray is a device-resident torch tensor
(complex128 for precision "fp64" — bitwise equal to the reference — or
complex64 for "fp32").  PyTorch only provides device buffers and the stream.

Differences a caller can observe, all deliberate:
  * ``loop_order`` is validated, then has no effect: the reference's two
    schedules are bitwise identical (tree2d.py:185-186), and so are the kernels'.
  * ``threads`` is accepted and ignored (there are no host threads).
  * ``precision`` defaults to "fp32" for float32/complex64 input and "fp64"
    otherwise; the reference always computes in complex128.
"""
from __future__ import annotations

import warnings

import numpy as np
import torch

from . import _lib, core
from .core import CoefficientArray

LOOP_ORDERS = ("levels-outer", "trees-outer")  # tree2d.py:19

_IN_CODES = {
    torch.float32: _lib.IN_F32,
    torch.float64: _lib.IN_F64,
    torch.complex64: _lib.IN_C64,
    torch.complex128: _lib.IN_C128,
}
_OUT_DTYPES = {_lib.PREC_FP32: torch.complex64, _lib.PREC_FP64: torch.complex128}


def _spec_exponents(spec):
    return tuple(int(m) for m in spec.exponents)


def _to_tensor(x):
    """numpy / torch / nested sequence -> torch tensor with a dtype the ABI reads.

    Integers and bools are widened to float64 exactly as np.asarray(x, complex128)
    would (tree2d.py:189); float32/complex64 are kept (fp32 precision path).
    """
    if isinstance(x, torch.Tensor):
        t = x
    else:
        a = np.asarray(x)
        if a.dtype.kind not in "biufc":
            a = np.asarray(x, dtype=np.complex128)  # raises like the reference does
        if a.ndim:
            with warnings.catch_warnings():  # read-only arrays: the tensor is only ever read
                warnings.simplefilter("ignore", UserWarning)
                t = torch.from_numpy(np.ascontiguousarray(a))
        else:
            t = torch.as_tensor(a)
    if t.dtype not in _IN_CODES:
        # everything else (ints, bools, half floats, complex32) widens exactly to the
        # reference's own working type, so the default precision is fp64 (bitwise)
        t = t.to(torch.complex128 if t.is_complex() else torch.float64)
    return t


def _default_precision(dtype) -> int:
    return _lib.PREC_FP32 if dtype in (torch.float32, torch.complex64) else _lib.PREC_FP64


def _precision_code(precision, dtype) -> int:
    if precision is None:
        return _default_precision(dtype)
    p = str(precision).lower()
    if p in ("fp32", "float32", "complex64", "single"):
        return _lib.PREC_FP32
    if p in ("fp64", "float64", "complex128", "double"):
        return _lib.PREC_FP64
    raise ValueError(f"precision must be 'fp32' or 'fp64', got {precision!r}")


def replay_counter(counter, shape, spec) -> None:
    """Report the reference's per-level node counts (tree2d.py:90-92,115-118)."""
    for region, nodes, positions in core.level_regions(shape, spec):
        counter.add_region(region, nodes, positions)


def forward_into(xt: torch.Tensor, m0: int, m1: int, out: torch.Tensor, *, prec: int,
                 scale: float = 1.0, p0_begin: int = 0, p0_end: int | None = None,
                 kernel: str = "auto", stream=None) -> torch.Tensor:
    """Low-level launch: window rows [p0_begin, p0_end) of device tensor ``xt`` into ``out``.

    ``xt`` is a 2D CUDA tensor (row stride may exceed its width); ``out`` a CUDA
    tensor of (p0_end - p0_begin, P1, n0, n1) complex of precision ``prec``.
    Stream-ordered on ``stream`` (default: torch's current stream of xt's device).
    """
    lib = _lib.load()
    if not xt.is_cuda:
        raise ValueError("forward_into needs a CUDA input tensor")
    if xt.dim() != 2:
        raise core.ShapeError("tree_swdft_2d expects a 2D array and 2D window")
    if xt.stride(1) != 1:
        xt = xt.contiguous()
    N0, N1 = xt.shape
    n0, n1 = 1 << m0, 1 << m1
    P0, P1 = N0 - n0 + 1, N1 - n1 + 1
    if p0_end is None:
        p0_end = P0
    want = (p0_end - p0_begin, P1, n0, n1)
    if tuple(out.shape) != want or out.dtype != _OUT_DTYPES[prec] or not out.is_contiguous():
        raise ValueError(f"out must be a contiguous {_OUT_DTYPES[prec]} tensor of shape {want}")
    if out.device != xt.device:
        raise ValueError("x and out must be on the same device")
    dev = xt.device.index
    sp = stream.cuda_stream if stream is not None else _lib.raw_stream(dev)
    kcode = _lib.KERNELS[kernel]
    # the large-window path's workspace comes from torch's allocator (PyTorch owns every
    # device buffer; the library allocates nothing per call when given one)
    wkey = (N0, N1, m0, m1, prec, p0_begin, p0_end, kcode)
    wbytes = _WS_BYTES.get(wkey)
    if wbytes is None:
        wbytes = _lib.workspace_bytes(N0, N1, m0, m1, prec, p0_begin, p0_end, kcode)
        if len(_WS_BYTES) > 4096:
            _WS_BYTES.clear()
        _WS_BYTES[wkey] = wbytes
    ws = None
    if wbytes:
        with torch.cuda.stream(stream) if stream is not None else _nullctx():
            ws = torch.empty(wbytes, dtype=torch.uint8, device=xt.device)
    args = (xt.data_ptr(), _IN_CODES[xt.dtype], N0, N1, xt.stride(0), m0, m1, prec, float(scale),
            p0_begin, p0_end, out.data_ptr(), ws.data_ptr() if ws is not None else None, wbytes,
            kcode, sp)
    if torch.cuda.current_device() == dev:
        rc = lib.swdft2d_forward_ws(*args)
    else:
        with torch.cuda.device(dev):
            rc = lib.swdft2d_forward_ws(*args)
    _lib.check(rc)
    return out


_WS_BYTES: dict = {}


class _nullctx:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        return False


def _forward_to_host(xt, m0, m1, host, prec, scale, kernel, strip_bytes, device):
    """Host output: ONE C-ABI call, swdft2d_forward_host (csrc/host_pipe.cu).  The input
    (host or device tensor) is copied to the device, window rows are computed in strips of
    ~strip_bytes into a ring of 4 device strips and copied out while later strips compute:
    straight into a pinned ``host`` (the PCIe rate), or through the library's pinned staging
    ring and worker threads into a pageable one (a fresh numpy array).  ``host`` is a torch
    host tensor or a numpy array of (P0, P1, n0, n1); returns it."""
    lib = _lib.load()
    if xt.stride(1) != 1 or (xt.shape[0] > 1 and xt.stride(0) < xt.shape[1]):
        xt = xt.contiguous()
    N0, N1 = xt.shape
    ld = xt.stride(0) if N0 > 1 else N1
    ptr = host.data_ptr() if isinstance(host, torch.Tensor) else host.ctypes.data
    dev = device.index if device.index is not None else torch.cuda.current_device()
    with torch.cuda.device(dev):
        rc = lib.swdft2d_forward_host(xt.data_ptr(), _IN_CODES[xt.dtype], N0, N1, ld, m0, m1, prec,
                                      float(scale), 0, N0 - (1 << m0) + 1, ptr, int(strip_bytes),
                                      _lib.KERNELS[kernel], _lib.raw_stream(dev))
    _lib.check(rc)
    return host


def tree_swdft_2d(x, spec, loop_order: str = "levels-outer", counter=None, budget=None,
                  threads: int = 1, *, precision=None, device=None, out=None,
                  kernel: str = "auto", to_host: bool = False, host_out=None,
                  strip_bytes: int = 1 << 29, devices=None):
    """Sliding-window 2D DFT via the shared-tree algorithm, on a B200.

    Equals the reference's tree_swdft_2d bit for bit with precision="fp64" and
    to <= 1e-4 of each window's L2 norm with precision="fp32".  The budget check
    uses the reference's own accounting (lattice + output at 16 B/complex,
    tree2d.py:195-196) and runs before anything is allocated.

    ``values`` is a device tensor by default; ``to_host=True`` (or a pinned
    ``host_out`` tensor) returns a numpy array as the reference does, streaming
    strips of ~``strip_bytes`` device->host while later strips compute, so the
    device holds only a few strips of output.

    ``devices=[d0, d1, ...]`` splits the window rows into one strip per device from
    this one process (partition.tree_swdft_2d_multi) and returns the
    list of per-device ShardedCoefficients with their [p0_begin, p0_end) ranges.
    """
    xt = _to_tensor(x)
    if xt.dim() != 2 or len(spec.exponents) != 2:
        raise core.ShapeError("tree_swdft_2d expects a 2D array and 2D window")
    shape = (int(xt.shape[0]), int(xt.shape[1]))
    spec.check_fits(shape)
    if loop_order not in LOOP_ORDERS:
        raise ValueError(f"loop_order must be one of {LOOP_ORDERS}")
    required = core.lattice_bytes(shape, spec) + core.output_bytes(shape, spec)
    core.check_budget(required, budget, what="level buffers + coefficient output")
    if devices is not None:
        from .partition import tree_swdft_2d_multi

        shards = tree_swdft_2d_multi(xt, spec, devices, precision=precision, budget=budget)
        if counter is not None:
            replay_counter(counter, shape, spec)
        return shards
    if kernel not in _lib.KERNELS:
        raise ValueError(f"kernel must be one of {tuple(_lib.KERNELS)}")
    m0, m1 = _spec_exponents(spec)
    prec = _precision_code(precision, xt.dtype)
    if device is None:
        device = xt.device if xt.is_cuda else torch.device("cuda", torch.cuda.current_device())
    device = torch.device(device)
    host_mode = to_host or host_out is not None
    n0, n1 = 1 << m0, 1 << m1
    P0, P1 = shape[0] - n0 + 1, shape[1] - n1 + 1
    scale = core.normalization_factor(spec)
    if host_mode:
        # host (numpy) output, as the reference returns: one swdft2d_forward_host call.
        # Without host_out the result is a fresh numpy array (pageable: pinning 34 GB takes
        # 14-16 s, filling a fresh pageable array through the staging workers 1.0 s)
        want = (P0, P1, n0, n1)
        odt = _OUT_DTYPES[prec]
        np_odt = np.complex64 if prec == _lib.PREC_FP32 else np.complex128
        if host_out is None:
            host_out = np.empty(want, dtype=np_odt)
        if isinstance(host_out, torch.Tensor):
            ok = not host_out.is_cuda and host_out.dtype == odt and host_out.is_contiguous()
        else:
            ok = isinstance(host_out, np.ndarray) and host_out.dtype == np_odt and \
                host_out.flags.c_contiguous and host_out.flags.writeable
        if not ok or tuple(host_out.shape) != want:
            raise ValueError(f"host_out must be a contiguous host {odt} tensor or numpy array "
                             f"of shape {want}")
        if xt.is_cuda and xt.device != device:
            xt = xt.to(device)
        _forward_to_host(xt, m0, m1, host_out, prec, scale, kernel, strip_bytes, device)
        if counter is not None:
            replay_counter(counter, shape, spec)
        values = host_out.numpy() if isinstance(host_out, torch.Tensor) else host_out
        return CoefficientArray(values, shape, spec, spec.normalization)
    if not xt.is_cuda or xt.device != device:
        # a call returning a device tensor must not leave a DMA reading the caller's buffer
        xt = xt.to(device)
    if out is None:
        out = torch.empty((P0, P1, n0, n1), dtype=_OUT_DTYPES[prec], device=device)
    forward_into(xt, m0, m1, out, prec=prec, scale=scale, kernel=kernel)
    if counter is not None:
        replay_counter(counter, shape, spec)
    return CoefficientArray(out, shape, spec, spec.normalization)
