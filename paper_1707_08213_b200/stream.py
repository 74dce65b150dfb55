"""Row-push streaming form of the 2D tree SWDFT on the GPU.

Mirror of the reference's ``tree2d.SlidingRowStream2D``
(/root/reference/pkg/src/swdft/tree2d.py:205-303): push one
length-N1 row at a time; once n0 rows have arrived every push returns the
(P1, n0, n1) coefficient slab of the newest window row, and the slab sequence
equals the batch transform's rows exactly.  The reference's
implementation raises for every window larger than 1x1;
this one implements the specified behaviour.

Device state, as the reference's stream keeps its tree levels between pushes:
the column levels of the dim-0 tree (m0 * n0/2 complex per output column, one
ring per level) advanced by one K2 launch per push (``swdft2d_stream_push``
with a state buffer: the pushed row's dim-1 nodes plus the dim-0 levels, O(n0 n1)
per window position, bitwise equal to the batch output in fp64).  Also the last
n0 input rows in a double-stored ring (row p at slots p mod n0 and p mod n0 + n0,
one contiguous [n0, N1] view): ``push_rows`` runs K1 over a block plus the n0 - 1
rows before it, and the next single push re-derives the level state from the
ring.  With an explicit ``kernel`` (or windows beyond 64) a push instead re-runs
that kernel over the ring view for the one window row.  Operation accounting (``ops_last_push``, ``last_push_position_ops``,
``counter.add_region``) follows tree2d.py:251-293 call for call.
"""
from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _lib, core
from .tree2d import _IN_CODES, _OUT_DTYPES, _precision_code, _to_tensor, forward_into

_RING_DTYPES = {_lib.PREC_FP32: torch.complex64, _lib.PREC_FP64: torch.complex128}


class SlidingRowStream2D:
    """Row-push streaming 2D tree SWDFT (tree2d.py:205-303 interface)."""

    def __init__(self, spec, row_length: int, counter=None, *, precision="fp64", device=None,
                 kernel: str = "auto"):
        if len(spec.exponents) != 2:
            raise core.ShapeError("SlidingRowStream2D needs a 2D window spec")
        self.spec = spec
        self.m0, self.m1 = (int(m) for m in spec.exponents)
        self.n0, self.n1 = 1 << self.m0, 1 << self.m1
        self.N1 = int(row_length)
        if self.n1 > self.N1:
            raise core.WindowTooLargeError(
                f"window size {self.n1} exceeds row length {self.N1}")
        self.counter = counter
        self.prec = _precision_code(precision, None)
        self.device = torch.device(device) if device is not None else torch.device(
            "cuda", torch.cuda.current_device())
        self.kernel = kernel
        if kernel not in _lib.KERNELS:
            raise ValueError(f"kernel must be one of {tuple(_lib.KERNELS)}")
        self._kernel_code = _lib.KERNELS[kernel]
        self._lib = _lib.load()
        self._factor = float(core.normalization_factor(spec))
        self._ring = torch.zeros((2 * self.n0, self.N1), dtype=_RING_DTYPES[self.prec],
                                 device=self.device)
        # incremental mode (K2): the tree's column-level state, advanced by every push
        self._state = None
        if kernel == "auto" and max(self.m0, self.m1) <= _lib.K1_MAX_M:
            nbytes = ctypes.c_int64()
            _lib.check(self._lib.swdft2d_stream_state_bytes(self.N1, self.m0, self.m1, self.prec,
                                                            ctypes.byref(nbytes)))
            self._state = torch.zeros(max(1, nbytes.value), dtype=torch.uint8, device=self.device)
        self._state_rows = 0  # rows the state has absorbed (== rows_pushed unless push_rows ran)
        self._pins = {}  # host-row upload ring per dtype (_upload)
        self._pin_next = 0
        self._ring_ptr = self._ring.data_ptr()
        self._dev_index = self.device.index if self.device.index is not None else \
            torch.cuda.current_device()
        self.P1 = self.N1 - self.n1 + 1
        self._levels = self._level_plan()
        self._profiles = self._push_profiles()
        self.rows_pushed = 0
        self.ops_last_push = 0
        self.last_push_position_ops = np.zeros(self.N1, dtype=np.int64)
        self._last_profile = -1
        self.closed = False

    def _level_plan(self):
        """(dim, shift, nodes) per tree level, core.shift_schedule order (core.py:197-220)."""
        plan = []
        for t in range(1, self.m1 + 1):
            plan.append((1, 1 << (self.m1 - t), 1 << t))
        for q in range(1, self.m0 + 1):
            plan.append((0, 1 << (self.m0 - q), (1 << q) * self.n1))
        return plan

    def _push_profiles(self):
        """(ops, per-position ops) of a push that runs the row levels and the first c
        column levels, c = 0..m0 (the per-push arithmetic of tree2d.py:251-293)."""
        n1, N1 = self.n1, self.N1
        vec = np.zeros(N1, dtype=np.int64)
        ops = 0
        out = []
        for dim, s, nodes in self._levels:
            if dim == 1:
                ops += (N1 - (n1 - s)) * nodes
                vec[n1 - s:] += nodes
        out.append((ops, vec.copy()))
        for dim, s, nodes in self._levels:
            if dim == 0:
                ops += (N1 - n1 + 1) * nodes
                vec[n1 - 1:] += nodes
                out.append((ops, vec.copy()))
        return out

    def _col_levels_run(self, p0: int) -> int:
        """Column levels a push of row p0 runs: those with p0 >= n0 - s (tree2d.py:273-274)."""
        c = 0
        for dim, s, _ in self._levels:
            if dim == 0:
                if p0 < self.n0 - s:
                    break
                c += 1
        return c

    def _account(self, p0: int, last: bool = True) -> None:
        """Operation accounting of pushing row p0 (tree2d.py:251-293): the counter's
        add_region calls level by level, and ops_last_push / last_push_position_ops."""
        n0, n1, N1 = self.n0, self.n1, self.N1
        if self.counter is not None:
            for dim, s, nodes in self._levels:
                if dim == 1:
                    self.counter.add_region((p0, slice(n1 - s, N1)), nodes, N1 - (n1 - s))
                else:
                    if p0 < n0 - s:
                        break  # deeper column levels need even more rows
                    self.counter.add_region((p0, slice(n1 - 1, N1)), nodes, N1 - n1 + 1)
        if last:
            k = self._col_levels_run(p0) if p0 < n0 - 1 else self.m0
            ops, vec = self._profiles[k]
            self.ops_last_push = ops
            if k != self._last_profile:  # the array only changes while warming up
                np.copyto(self.last_push_position_ops, vec)
                self._last_profile = k

    def push_row(self, row):
        """Ingest one length-N1 row; returns the (P1, n0, n1) slab (device tensor)
        once n0 rows have arrived, None while warming up.  One C-ABI call
        (swdft2d_stream_push: one K2 launch over the level state, or, with an explicit
        kernel, the ring store + that kernel over the ring view)."""
        if self.closed:
            raise core.StateError("push after close")
        r = _to_tensor(row)
        if tuple(r.shape) != (self.N1,):
            raise core.ShapeError(f"row shape {tuple(r.shape)} != ({self.N1},)")
        if not r.is_cuda:
            r = self._upload(r)
        elif r.device != self.device:
            r = r.to(self.device)
        if r.stride(0) != 1:
            r = r.contiguous()
        p0 = self.rows_pushed
        n0 = self.n0
        slab = None
        if p0 >= n0 - 1:
            slab = torch.empty((self.P1, n0, self.n1), dtype=_OUT_DTYPES[self.prec],
                               device=self.device)
        state = self._state.data_ptr() if self._state is not None else None
        if torch.cuda.current_device() == self._dev_index:
            rc = self._push(r, state, p0, slab)
        else:
            with torch.cuda.device(self.device):
                rc = self._push(r, state, p0, slab)
        if rc:
            _lib.check(rc)
        self._account(p0)
        self.rows_pushed += 1
        self._state_rows = self.rows_pushed
        return slab

    _UPLOAD_SLOTS = 4

    def _upload(self, r):
        """Host row -> device through a library-owned pinned ring: the caller's buffer is
        read synchronously here (so it may be refilled as soon as push_row returns) and the
        H2D copy of the pinned slot stays asynchronous; a slot is refilled only after its
        previous copy has completed (its event)."""
        slots = self._pins.get(r.dtype)
        if slots is None:
            slots = self._pins[r.dtype] = [
                (torch.empty(self.N1, dtype=r.dtype, pin_memory=True),
                 torch.empty(self.N1, dtype=r.dtype, device=self.device), torch.cuda.Event())
                for _ in range(self._UPLOAD_SLOTS)]
        host, dev, ev = slots[self._pin_next % self._UPLOAD_SLOTS]
        self._pin_next += 1
        ev.synchronize()  # no-op until the slot was used (an unrecorded event is complete)
        host.copy_(r.reshape(-1))
        with torch.cuda.device(self.device):
            dev.copy_(host, non_blocking=True)
            ev.record()
        return dev

    def _push(self, r, state, p0, slab) -> int:
        stream = _lib.raw_stream(self._dev_index)
        if state is not None and self._state_rows < p0:
            self._catch_up(p0, state, stream)
        return self._lib.swdft2d_stream_push(
            r.data_ptr(), _IN_CODES[r.dtype], self.N1, self._ring_ptr, state, self.m0, self.m1,
            self.prec, self._factor, p0, slab.data_ptr() if slab is not None else None,
            self._kernel_code, stream)

    def _catch_up(self, p0: int, state: int, stream: int) -> None:
        """Bring the level state up to row p0 - 1 after push_rows: replay the last
        n0 - 1 rows from the raw ring (no output).  A level-l value the next pushes read
        depends only on those rows, so the state's older content does not matter."""
        code = _lib.IN_C128 if self.prec == _lib.PREC_FP64 else _lib.IN_C64
        esz = self._ring.element_size()
        for q in range(max(self._state_rows, p0 - self.n0 + 1), p0):
            row = self._ring.data_ptr() + (q % self.n0) * self.N1 * esz
            _lib.check(self._lib.swdft2d_stream_push(row, code, self.N1, None, state, self.m0,
                                                     self.m1, self.prec, self._factor, q, None,
                                                     self._kernel_code, stream))
        self._state_rows = p0

    def push_rows(self, rows):
        """Ingest k rows at once (a [k, N1] block); returns the [k', P1, n0, n1] slabs
        of every window row completed by the block (k' <= k; None if none).  Equal to
        k push_row calls (same slabs, same accounting and counter calls), but one K1
        launch over the block plus the n0 - 1 rows before it."""
        if self.closed:
            raise core.StateError("push after close")
        blk = rows if isinstance(rows, torch.Tensor) else torch.from_numpy(
            np.asarray(rows, dtype=np.complex128))
        if blk.dim() != 2 or blk.shape[1] != self.N1:
            raise core.ShapeError(f"row block shape {tuple(blk.shape)} != (k, {self.N1})")
        k = int(blk.shape[0])
        if k == 0:
            return None
        n0 = self.n0
        blk = blk.to(device=self.device, dtype=self._ring.dtype)
        first = self.rows_pushed
        pre = min(first, n0 - 1)  # earlier rows the block's first windows need
        start = (first - pre) % n0
        work = torch.cat([self._ring[start:start + pre], blk]) if pre else blk.contiguous()
        if self.counter is not None:
            for i in range(k - 1):
                self._account(first + i, last=False)
        self._account(first + k - 1)
        keep = min(k, n0)  # keep the last n0 rows for later pushes (both ring copies)
        slots = torch.arange(first + k - keep, first + k, device=self.device) % n0
        self._ring.index_copy_(0, torch.cat([slots, slots + n0]), blk[k - keep:].repeat(2, 1))
        self.rows_pushed += k
        w_begin = max(0, first - n0 + 1)  # global window rows completed by this block
        w_end = first + k - n0 + 1
        if w_end <= w_begin:
            return None
        base = first - pre  # global row of work[0]
        out = torch.empty((w_end - w_begin, self.P1, n0, self.n1), dtype=_OUT_DTYPES[self.prec],
                          device=self.device)
        forward_into(work, self.m0, self.m1, out, prec=self.prec, scale=self._factor,
                     p0_begin=w_begin - base, p0_end=w_end - base, kernel=self.kernel)
        return out

    def close(self) -> None:
        self.closed = True


class SlidingStream1D:
    """Sample-push 1D stream (tree1d.py:63-119 interface) on the GPU.  For n <= 64 every
    push is one K2 launch over the tree's level state (the 1D tree is the dim-0 tree of a
    one-column 2D stream); larger windows keep a device ring of the last n samples
    (double-stored, so the window is one contiguous view) and run KR over it.  Once
    p >= n - 1 a push returns the n-point transform of the last n samples, bitwise equal
    to the batch 1D tree in fp64."""

    def __init__(self, spec, counter=None, *, precision="fp64", device=None):
        if len(spec.exponents) != 1:
            raise core.ShapeError("SlidingStream1D needs a 1D window spec")
        (self.m,) = (int(v) for v in spec.exponents)
        self.n = 1 << self.m
        self.spec = spec
        self.counter = counter
        self.prec = _precision_code(precision, None)
        self.device = torch.device(device) if device is not None else torch.device(
            "cuda", torch.cuda.current_device())
        self._factor = float(core.normalization_factor(spec))
        self._dev_index = self.device.index if self.device.index is not None else \
            torch.cuda.current_device()
        self._ring = torch.zeros(2 * self.n, dtype=_RING_DTYPES[self.prec], device=self.device)
        # n <= 64: K2 pushes (the 1D tree is the dim-0 tree of a 1-column 2D stream:
        # m0 = m, m1 = 0, N1 = 1), one launch per sample over the level state
        self._state = None
        if self.m <= _lib.K1_MAX_M:
            self._lib = _lib.load()
            nbytes = ctypes.c_int64()
            _lib.check(self._lib.swdft2d_stream_state_bytes(1, self.m, 0, self.prec,
                                                            ctypes.byref(nbytes)))
            self._state = torch.zeros(max(1, nbytes.value), dtype=torch.uint8, device=self.device)
            self._sample = torch.zeros(1, dtype=_RING_DTYPES[self.prec], device=self.device)
            self._code = _lib.IN_C128 if self.prec == _lib.PREC_FP64 else _lib.IN_C64
        self.pushed = 0
        self.ops_last_push = 0
        self.closed = False

    def push(self, sample):
        """Ingest one sample; returns the length-n coefficient vector (device tensor) once
        the window is full, None while warming up (tree1d.py:92-116)."""
        if self.closed:
            raise core.StateError("push after close")
        p = self.pushed
        n = self.n
        v = complex(sample) if not isinstance(sample, torch.Tensor) else sample
        if self._state is None:
            slot = p % n
            self._ring[slot] = v
            self._ring[slot + n] = v
        ops = 0
        for l in range(1, self.m + 1):  # tree1d.py:101-108
            s = 1 << (self.m - l)
            if p < n - s:
                break  # higher levels need even more history
            ops += 1 << l
            if self.counter is not None:
                self.counter.add_region((p,), 1 << l, 1)
        self.ops_last_push = ops
        self.pushed += 1
        if self._state is not None:
            self._sample.fill_(v) if not isinstance(v, torch.Tensor) else self._sample.copy_(
                v.reshape(1))
            out = torch.empty(n, dtype=_OUT_DTYPES[self.prec], device=self.device) \
                if p >= n - 1 else None
            with torch.cuda.device(self.device):
                _lib.check(self._lib.swdft2d_stream_push(
                    self._sample.data_ptr(), self._code, 1, None, self._state.data_ptr(), self.m,
                    0, self.prec, self._factor, p, out.data_ptr() if out is not None else None,
                    _lib.KERNEL_AUTO, _lib.raw_stream(self._dev_index)))
            return out
        if p < n - 1:
            return None
        first = (p + 1) % n
        out = torch.empty((1, 1, 1, n), dtype=_OUT_DTYPES[self.prec], device=self.device)
        forward_into(self._ring[first:first + n].view(1, n), 0, self.m, out, prec=self.prec,
                     scale=self._factor)
        return out.view(n)

    def close(self) -> None:
        self.closed = True
