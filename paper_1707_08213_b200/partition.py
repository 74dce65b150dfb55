"""Single-box window-row strip partitioner (one process per GPU, torch.distributed).

The batch 2D tree SWDFT shards exactly along window rows: window row p0 needs
only input rows [p0, p0 + n0) and a strip of rows computed alone is bitwise
identical to the same rows of a full run.  So the
only data movement is a scatter of input strips (each with its n0 - 1 halo
rows) from the rank that holds x; outputs stay resident on every rank and are
never gathered or reduced.

The reference has no multi-device path (its parallelism is a thread pool over
contiguous axis-0 chunks per level, tree2d.py:22-27,58-64); the split rule here
is the same "contiguous chunks of axis 0" idea applied once, across GPUs:
rank g of G owns window rows [floor(P0*g/G), floor(P0*(g+1)/G))
(swdft2d_strip_range in libswdft2d.so).

The scatter is one batched group of point-to-point sends from ``src`` over the
process group's backend (NCCL over NVLink/NVSwitch on the GPU box, gloo in the
CPU tests).
"""
from __future__ import annotations

from dataclasses import dataclass

import torch
import torch.distributed as dist

from . import _lib, core


def strip_plan(P0: int, m0: int, world: int):
    """[(p0_begin, p0_end, row_begin, row_end)] for every rank (via the C ABI)."""
    return [_lib.strip_range(P0, m0, g, world) for g in range(world)]


def block_plan(P0: int, P1: int, m0: int, m1: int, gr: int, gc: int):
    """2-D partition over gr x gc ranks (rank g = i * gc + j): window rows
    [floor(P0 i/gr), floor(P0 (i+1)/gr)) x window columns [floor(P1 j/gc),
    floor(P1 (j+1)/gc)), i.e. the strip rule on each axis, with the n0 - 1 halo input
    rows and n1 - 1 halo input columns.  Row strips are (G, 1).  Column blocks are
    bitwise exact like row strips.
    [(p0_begin, p0_end, p1_begin, p1_end, row_begin, row_end, col_begin, col_end)]."""
    rows = strip_plan(P0, m0, gr)
    cols = strip_plan(P1, m1, gc)
    return [(r[0], r[1], c[0], c[1], r[2], r[3], c[2], c[3]) for r in rows for c in cols]


def strip_plan_py(P0: int, m0: int, world: int):
    """Pure-Python statement of the same rule (used to cross-check the C ABI)."""
    n0 = 1 << m0
    out = []
    for g in range(world):
        a, b = (P0 * g) // world, (P0 * (g + 1)) // world
        out.append((a, b, a, b + n0 - 1 if b > a else a))
    return out


@dataclass
class ShardedCoefficients:
    """This rank's block of the [P0, P1, n0, n1] output (device resident): window rows
    [p0_begin, p0_end) x window columns [p1_begin, p1_end) (all columns for row strips)."""

    values: torch.Tensor
    p0_begin: int
    p0_end: int
    source_shape: tuple
    window: object
    normalization: str = "none"
    p1_begin: int = 0
    p1_end: int | None = None


def scatter_strips(x, shape, m0: int, dtype, device, group=None, src: int = 0, recv=None):
    """Scatter input row strips (with halos) from ``src``.

    ``x`` (a tensor on ``device``, rows contiguous) is only read on ``src``; the
    other ranks pass None (and may pass a preallocated ``recv`` buffer of their
    strip's shape).  Returns (local_rows_tensor, (p0_begin, p0_end, row_begin,
    row_end)).  Empty strips (P0 < world) come back as 0-row tensors.
    """
    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    N0, N1 = int(shape[0]), int(shape[1])
    P0 = N0 - (1 << m0) + 1
    plan = strip_plan(P0, m0, world)
    my = plan[rank]
    ops = []
    if rank == src:
        if x is None or tuple(x.shape) != (N0, N1):
            raise core.ShapeError(f"source rank needs the full {N0}x{N1} input")
        for g, (_, _, rb, re) in enumerate(plan):
            if g != src and re > rb:
                ops.append(dist.P2POp(dist.isend, x[rb:re].contiguous(), g, group))
        local = x[my[2]:my[3]]
    else:
        local = recv if recv is not None else torch.empty((my[3] - my[2], N1), dtype=dtype,
                                                          device=device)
        if tuple(local.shape) != (my[3] - my[2], N1):
            raise ValueError(f"recv buffer must have shape {(my[3] - my[2], N1)}")
        if my[3] > my[2]:
            ops.append(dist.P2POp(dist.irecv, local, src, group))
    if ops:
        for req in dist.batch_isend_irecv(ops):
            req.wait()
    return local, my


def piece_bounds(rows: int, first_fraction: float, pieces: int):
    """Window-row pieces [w_c, w_{c+1}) of a strip: a short first piece (so compute
    starts after a small part of the strip has arrived), the rest split evenly."""
    if rows <= 0:
        return [0, 0]
    if pieces <= 1 or rows < 2:
        return [0, rows]
    first = max(1, min(rows - 1, int(round(rows * first_fraction))))
    rest = pieces - 1
    bounds = [0, first]
    for c in range(1, rest + 1):
        bounds.append(first + ((rows - first) * c) // rest)
    return sorted(set(bounds))


NVLINK_PEER_BPS = 770e9  # measured peer-copy rate per direction (B200_PROFILING.md)
HBM_WRITE_BPS = 6.4e12   # K1's sustained coefficient write rate on one B200 (profiles/)


def choose_pieces(shape, m0: int, m1: int, in_bytes: int, out_bytes: int, world: int) -> int:
    """2 (pipelined: compute on a 1/8 first chunk while the rest arrives) when the scatter
    time it hides exceeds the extra launch's n0 - 1 halo rows of compute, else 1.
    Model: a window row costs P1*n0*n1*out_bytes / HBM_WRITE_BPS; rank 0's egress
    carries every other strip at NVLINK_PEER_BPS (single-GPU emulation in
    profiles/strip_scaling_r01.jsonl)."""
    if world <= 1:
        return 1
    N0, N1 = shape
    n0, n1 = 1 << m0, 1 << m1
    P0, P1 = N0 - n0 + 1, N1 - n1 + 1
    row_t = P1 * n0 * n1 * out_bytes / HBM_WRITE_BPS
    strip_rows = P0 / world
    send_all = (world - 1) * (strip_rows + n0 - 1) * N1 * in_bytes / NVLINK_PEER_BPS
    send_first = (world - 1) * (strip_rows / 8 + n0 - 1) * N1 * in_bytes / NVLINK_PEER_BPS
    return 2 if send_all - send_first > (n0 - 1) * row_t + 5e-6 else 1


def pipelined_block_forward(x, shape, m0: int, m1: int, split, dtype, device, compute,
                            group=None, src: int = 0, recv=None, pieces: int = 2,
                            first_fraction: float = 0.125):
    """Scatter + compute with overlap over the gr x gc block partition ``split``
    (block_plan): every rank's input block travels as ``pieces`` consecutive row chunks
    (separate point-to-point messages, in order), and ``compute(local, w_begin, w_end)``
    runs for the block's window rows [w_begin, w_end) (block-relative) as soon as the
    input rows they need, [w_begin, w_end + n0 - 1), have arrived — so rank g starts
    after its first (short) chunk instead of after its whole block.  The sends go out
    piece-major (one batched group per piece index: every peer's first chunk before any
    peer's remainder).  A block narrower than the input is packed into a contiguous copy
    per chunk on the source (row strips are sent as views).  The source rank computes
    its own block at once, from a strided view of x.
    Returns (local input block, (p0_begin, p0_end, p1_begin, p1_end, row_begin, row_end,
    col_begin, col_end))."""
    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    gr, gc = split
    if gr * gc != world:
        raise ValueError(f"split {gr}x{gc} does not cover {world} ranks")
    N0, N1 = int(shape[0]), int(shape[1])
    n0, n1 = 1 << m0, 1 << m1
    plan = block_plan(N0 - n0 + 1, N1 - n1 + 1, m0, m1, gr, gc)
    mine = plan[rank]
    a, b, _, _, rb, re, cb, ce = mine
    if rank == src:
        if x is None or tuple(x.shape) != (N0, N1):
            raise core.ShapeError(f"source rank needs the full {N0}x{N1} input")
        if x.stride(1) != 1 or (N0 > 1 and x.stride(0) != N1):
            raise ValueError("the source input must be C-contiguous (rows are sent as views)")
        per_peer = []  # (peer, [(first input row, end row) of each piece], cols)
        for g, (ga, gb, _, _, grb, gre, gcb, gce) in enumerate(plan):
            if g == src or gre <= grb or gce <= gcb:
                continue
            wb = piece_bounds(gb - ga, first_fraction, pieces)
            cuts = [0] + [w + n0 - 1 for w in wb[1:-1]] + [gre - grb]
            per_peer.append((g, [(grb + cuts[c], grb + cuts[c + 1]) for c in range(len(cuts) - 1)],
                             (gcb, gce)))
        # piece-major: one batched group per piece index, so every peer's (short) first
        # chunk leaves before any peer's remainder, whatever stream(s) the backend runs
        # its point-to-point operations on; within a peer, pieces arrive in order
        works = []
        for c in range(max((len(ps) for _, ps, _ in per_peer), default=0)):
            ops = []
            for g, ps, (gcb, gce) in per_peer:
                if c < len(ps):
                    t = x[ps[c][0]:ps[c][1], gcb:gce]
                    ops.append(dist.P2POp(dist.isend, t if gce - gcb == N1 else t.contiguous(),
                                          g, group))
            works += dist.batch_isend_irecv(ops)
        local = x[rb:re, cb:ce]
        if b > a and ce > cb:
            compute(local, 0, b - a)
        for w in works:
            w.wait()
        return local, mine
    local = recv if recv is not None else torch.empty((re - rb, ce - cb), dtype=dtype,
                                                      device=device)
    if tuple(local.shape) != (re - rb, ce - cb):
        raise ValueError(f"recv buffer must have shape {(re - rb, ce - cb)}")
    if b > a and ce > cb:
        wb = piece_bounds(b - a, first_fraction, pieces)
        cuts = [0] + [w + n0 - 1 for w in wb[1:-1]] + [re - rb]
        works = [dist.batch_isend_irecv([dist.P2POp(dist.irecv, local[cuts[c]:cuts[c + 1]], src,
                                                    group)])
                 for c in range(len(cuts) - 1)]
        for c in range(len(wb) - 1):
            for w in works[c]:
                w.wait()  # NCCL: the compute stream waits for this chunk only
            compute(local, wb[c], wb[c + 1])
    return local, mine


def pipelined_strip_forward(x, shape, m0: int, dtype, device, compute, group=None, src: int = 0,
                            recv=None, pieces: int = 2, first_fraction: float = 0.125):
    """Row-strip form of pipelined_block_forward (split (world, 1), every rank all
    columns).  Returns (local_rows_tensor, (p0_begin, p0_end, row_begin, row_end))."""
    world = dist.get_world_size(group)
    # m1 only sets the column halo, and a row strip has every column: pass m1 = 0
    local, p = pipelined_block_forward(x, shape, m0, 0, (world, 1), dtype, device, compute,
                                       group, src, recv, pieces, first_fraction)
    return local, (p[0], p[1], p[4], p[5])


def tree_swdft_2d_sharded(x, spec, *, shape=None, dtype=None, group=None, src: int = 0,
                          precision=None, budget=None, pieces=None) -> ShardedCoefficients:
    """Strip-sharded tree_swdft_2d: every rank returns its own window rows.

    On ``src`` pass the full input tensor (CUDA); elsewhere pass x=None plus
    ``shape`` and ``dtype``.  Budget accounting is the reference's, per strip.
    """
    from .tree2d import _OUT_DTYPES, _precision_code, forward_into

    rank = dist.get_rank(group)
    if rank == src:
        shape = tuple(int(s) for s in x.shape)
        dtype = x.dtype
        device = x.device
    else:
        device = torch.device("cuda", torch.cuda.current_device())
    if len(shape) != 2 or len(spec.exponents) != 2:
        raise core.ShapeError("tree_swdft_2d expects a 2D array and 2D window")
    spec.check_fits(shape)
    m0, m1 = (int(m) for m in spec.exponents)
    prec = _precision_code(precision, dtype)
    n0, n1 = 1 << m0, 1 << m1
    P0, P1 = shape[0] - n0 + 1, shape[1] - n1 + 1
    a, b, rb, re = strip_plan(P0, m0, dist.get_world_size(group))[dist.get_rank(group)]
    if b > a:
        sshape = (re - rb, shape[1])
        core.check_budget(core.lattice_bytes(sshape, spec) + core.output_bytes(sshape, spec),
                          budget, what="level buffers + coefficient output")
    out = torch.empty((b - a, P1, n0, n1), dtype=_OUT_DTYPES[prec], device=device)
    scale = core.normalization_factor(spec)
    if pieces is None:
        pieces = choose_pieces(shape, m0, m1, torch.empty((), dtype=dtype).element_size(),
                               out.element_size(), dist.get_world_size(group))

    def compute(local, w0, w1):
        forward_into(local, m0, m1, out[w0:w1], prec=prec, scale=scale, p0_begin=w0, p0_end=w1)

    pipelined_strip_forward(x, shape, m0, dtype, device, compute, group, src, pieces=pieces)
    return ShardedCoefficients(out, a, b, tuple(shape), spec, spec.normalization)


def tree_swdft_2d_multi(x, spec, devices, *, precision=None, budget=None):
    """Single-process multi-GPU tree_swdft_2d over ``devices`` (swdft2d_forward_multi).

    ``x`` is a CUDA tensor on devices[0] (or host data, copied there).  Device slot g
    gets strip g of len(devices) (swdft2d_strip_range): its input rows are copied over
    NVLink into a stage buffer on that device and transformed there; slot 0 computes
    straight from x.  Returns one ShardedCoefficients per slot, each resident on its
    device, in strip order — the same shards the torchrun path returns per rank.
    Stream-ordered on every device's current torch stream.  Budget accounting is the
    reference's, for the whole problem (tree2d.py:195-196).
    """
    import ctypes

    from .tree2d import _IN_CODES, _OUT_DTYPES, _precision_code, _to_tensor

    devs = [torch.device(d) if not isinstance(d, int) else torch.device("cuda", d)
            for d in devices]
    if not devs or any(d.type != "cuda" for d in devs):
        raise ValueError("devices must be a non-empty list of CUDA devices")
    devs = [torch.device("cuda", d.index if d.index is not None else torch.cuda.current_device())
            for d in devs]
    xt = _to_tensor(x)
    if xt.dim() != 2 or len(spec.exponents) != 2:
        raise core.ShapeError("tree_swdft_2d expects a 2D array and 2D window")
    shape = (int(xt.shape[0]), int(xt.shape[1]))
    spec.check_fits(shape)
    core.check_budget(core.lattice_bytes(shape, spec) + core.output_bytes(shape, spec), budget,
                      what="level buffers + coefficient output")
    if xt.device != devs[0]:
        xt = xt.to(devs[0])
    if xt.stride(1) != 1:
        xt = xt.contiguous()
    m0, m1 = (int(m) for m in spec.exponents)
    prec = _precision_code(precision, xt.dtype)
    n0, n1 = 1 << m0, 1 << m1
    P0, P1 = shape[0] - n0 + 1, shape[1] - n1 + 1
    G = len(devs)
    plan = strip_plan(P0, m0, G)
    outs, stages = [], []
    for g, (a, b, rb, re) in enumerate(plan):
        outs.append(torch.empty((b - a, P1, n0, n1), dtype=_OUT_DTYPES[prec], device=devs[g]))
        stages.append(torch.empty((re - rb, shape[1]), dtype=xt.dtype, device=devs[g])
                      if g > 0 else None)
    streams = [torch.cuda.current_stream(d) for d in devs]
    vp = ctypes.c_void_p
    c_devs = (ctypes.c_int * G)(*[d.index for d in devs])
    c_stage = (vp * G)(*[None if t is None or t.numel() == 0 else t.data_ptr() for t in stages])
    c_outs = (vp * G)(*[t.data_ptr() if t.numel() else None for t in outs])
    c_streams = (vp * G)(*[s.cuda_stream for s in streams])
    rc = _lib.load().swdft2d_forward_multi(xt.data_ptr(), _IN_CODES[xt.dtype], shape[0], shape[1],
                                           xt.stride(0), m0, m1, prec,
                                           float(core.normalization_factor(spec)), G, c_devs,
                                           c_stage, c_outs, c_streams)
    _lib.check(rc)
    return [ShardedCoefficients(outs[g], a, b, shape, spec, spec.normalization)
            for g, (a, b, _, _) in enumerate(plan)]
