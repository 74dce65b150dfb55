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


def _led_plan(P: int, m: int, parts: int, lead: int):
    """The strip rule on one axis with the first part ``lead`` units shorter and the rest
    spread over the others: part 0 = [0, floor(P/parts) - lead), part k >= 1 starts at
    e + floor((P - e)(k - 1)/(parts - 1)), e = part 0's end.  lead = 0 is the plain rule."""
    if lead <= 0 or parts < 2 or P < parts:
        return strip_plan(P, m, parts)
    n = 1 << m
    e = max(1, P // parts - lead)
    cuts = [0, e] + [e + ((P - e) * k) // (parts - 1) for k in range(1, parts)]
    return [(a, b, a, b + n - 1 if b > a else a) for a, b in zip(cuts, cuts[1:])]


def block_plan(P0: int, P1: int, m0: int, m1: int, gr: int, gc: int, lead: int = 0):
    """2-D partition over gr x gc ranks (rank g = i * gc + j): window rows
    [floor(P0 i/gr), floor(P0 (i+1)/gr)) x window columns [floor(P1 j/gc),
    floor(P1 (j+1)/gc)), i.e. the strip rule on each axis, with the n0 - 1 halo input
    rows and n1 - 1 halo input columns.  Row strips are (G, 1).  Column blocks are
    bitwise exact like row strips.
    ``lead`` > 0 makes the source rank's (rank 0's) band that many window rows shorter
    (window columns when gr = 1), spread over the other bands: rank 0 sends every other
    block before it computes its own (tune_split sizes it).
    [(p0_begin, p0_end, p1_begin, p1_end, row_begin, row_end, col_begin, col_end)]."""
    rows = _led_plan(P0, m0, gr, lead if gr > 1 else 0)
    cols = _led_plan(P1, m1, gc, lead if gr == 1 else 0)
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


def split_candidates(world: int):
    """Every gr x gc factorisation of ``world``, row strips (world x 1) first."""
    return [(gr, world // gr) for gr in range(world, 0, -1) if world % gr == 0]


_SPLITS: dict = {}


def _block_area(p):
    return max(0, p[1] - p[0]) * max(0, p[3] - p[2])


def tune_split(x, m0: int, m1: int, prec: int, world: int, reps: int = 2, src: int = 0):
    """Measure on x's device which gr x gc partition of ``world`` ranks finishes first.

    For every factorisation, K1 transforms the largest block a rank would own (from a
    strided view of x, as the source rank does) — the per-block time t includes its
    schedule's wave quantization, warm-up rows and launch.  The scatter is modelled from
    the bytes the source sends at NVLINK_PEER_BPS (all of it: t_all; the first pieces:
    t_first).  The source sends everything before it computes its own block (its NCCL
    kernel must not compete with its own K1 grid for SMs), so
      * one piece: every rank waits ~t_all, step ~ t_all + t;
      * two pieces: receivers start after t_first (+ the second piece's extra warm-up and
        launch), and the source's band is made `lead` window rows (columns when gr = 1)
        shorter, spread over the other bands, so that t_all + its block ~ t_first + a
        receiver's block: step ~ t_first + extra + t (1 + lambda / (b - 1)), lambda =
        (t_all - t_first - extra) / t * (b - 1) / b, b bands along that axis.
    The lower step time wins.  Measured on one GPU the same way in scripts/split_scaling.py
    (profiles/split_scaling_r02*.jsonl).  Returns {"split": (gr, gc), "pieces": p,
    "lead": window rows (or columns) taken off the source's band, "table": [...]}."""
    from .tree2d import _OUT_DTYPES, forward_into

    N0, N1 = int(x.shape[0]), int(x.shape[1])
    n0, n1 = 1 << m0, 1 << m1
    P0, P1 = N0 - n0 + 1, N1 - n1 + 1
    esz = x.element_size()
    cands = []
    for gr, gc in split_candidates(world):
        plan = block_plan(P0, P1, m0, m1, gr, gc)
        cands.append(((gr, gc), plan, max(plan, key=_block_area)))
    most = max(_block_area(big) for _, _, big in cands) * n0 * n1
    scratch = torch.empty(max(most, 1), dtype=_OUT_DTYPES[prec], device=x.device)
    table = []
    for split, plan, big in cands:
        a0, b0, a1, b1, rb, re, cb, ce = big
        if _block_area(big) == 0:
            continue
        view = x[rb:re, cb:ce]
        o = scratch[:_block_area(big) * n0 * n1].view(b0 - a0, b1 - a1, n0, n1)
        forward_into(view, m0, m1, o, prec=prec)
        ts_ = []
        for _ in range(reps):
            torch.cuda.synchronize(x.device)
            if hasattr(torch.cuda, "_sleep"):
                torch.cuda._sleep(100000)  # host submission stays outside the events
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            forward_into(view, m0, m1, o, prec=prec)
            e1.record()
            e1.synchronize()
            ts_.append(e0.elapsed_time(e1) / 1e3)
        t = min(ts_)
        send = first = 0
        for g, p in enumerate(plan):
            if g == src or _block_area(p) == 0:
                continue
            rows_in, cols_in = p[5] - p[4], p[7] - p[6]
            send += rows_in * cols_in * esz
            first += min(rows_in, piece_bounds(p[1] - p[0], 0.125, 2)[1] + n0 - 1) * cols_in * esz
        t_all, t_first = send / NVLINK_PEER_BPS, first / NVLINK_PEER_BPS
        # a second piece re-runs part of the n0 - 1 warm-up (about half of it: stage C is
        # skipped on most warm-up rows) and adds a launch
        extra = 0.5 * (n0 - 1) / max(1, b0 - a0) * t + 5e-6
        gr, gc = split
        bands, blen = (gr, b0 - a0) if gr > 1 else (gc, b1 - a1)
        lam = max(0.0, (t_all - t_first - extra) / t * (bands - 1) / bands)
        score1 = t_all + t
        score2 = t_first + extra + t * (1 + lam / (bands - 1))
        pieces = 2 if score2 < score1 else 1
        lead = int(round(lam * blen)) if pieces == 2 else 0
        table.append({"split": split, "block": [b0 - a0, b1 - a1], "compute_s": t,
                      "scatter_s": t_all, "first_s": t_first, "pieces": pieces, "lead": lead,
                      "score_s": min(score1, score2)})
    del scratch
    best = min(table, key=lambda r: r["score_s"])
    return {"split": best["split"], "pieces": best["pieces"], "lead": best["lead"],
            "table": table}


def choose_split(x, shape, m0: int, m1: int, prec: int, world: int, in_bytes: int,
                 group=None, src: int = 0) -> dict:
    """The partition every rank uses: measured once on ``src`` (tune_split), broadcast to
    the group, cached per (shape, window, precision, world, element size) on every rank.
    ``x`` is only read on ``src``."""
    key = (tuple(int(v) for v in shape), int(m0), int(m1), int(prec), int(world), int(in_bytes))
    hit = _SPLITS.get(key)
    if hit is not None:
        return hit
    if world == 1:
        res = {"split": (1, 1), "pieces": 1, "table": []}
    else:
        obj = [tune_split(x, m0, m1, prec, world, src=src) if dist.get_rank(group) == src
               else None]
        dist.broadcast_object_list(obj, src=dist.get_global_rank(group, src) if group else src,
                                   group=group)
        res = obj[0]
    _SPLITS[key] = res
    return res


def pipelined_block_forward(x, shape, m0: int, m1: int, split, dtype, device, compute,
                            group=None, src: int = 0, recv=None, pieces: int = 2,
                            first_fraction: float = 0.125, lead: int = 0):
    """Scatter + compute with overlap over the gr x gc block partition ``split``
    (block_plan): every rank's input block travels as ``pieces`` consecutive row chunks
    (separate point-to-point messages, in order), and ``compute(local, w_begin, w_end)``
    runs for the block's window rows [w_begin, w_end) (block-relative) as soon as the
    input rows they need, [w_begin, w_end + n0 - 1), have arrived — so rank g starts
    after its first (short) chunk instead of after its whole block.  The sends go out
    as one batched group, piece-major (every peer's first chunk ahead of its remainder).  A block narrower than the input is packed into a contiguous copy
    per chunk on the source (row strips are sent as views).  The source rank computes
    its own block from a strided view of x once its sends are done.
    Returns (local input block, (p0_begin, p0_end, p1_begin, p1_end, row_begin, row_end,
    col_begin, col_end))."""
    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    gr, gc = split
    if gr * gc != world:
        raise ValueError(f"split {gr}x{gc} does not cover {world} ranks")
    N0, N1 = int(shape[0]), int(shape[1])
    n0, n1 = 1 << m0, 1 << m1
    plan = block_plan(N0 - n0 + 1, N1 - n1 + 1, m0, m1, gr, gc, lead)
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
        # ONE batched group holding every send, piece-major (every peer's short first chunk,
        # then the remainders; within a peer, pieces go in order and the peers proceed in
        # parallel).  One group = one NCCL kernel, launched BEFORE this rank's own K1 below:
        # a second group's kernel would queue behind the first on the NCCL stream and then
        # find every SM held by the persistent K1 grid, i.e. the remainders would leave only
        # after this rank's whole compute.
        ops = []
        for c in range(max((len(ps) for _, ps, _ in per_peer), default=0)):
            for g, ps, (gcb, gce) in per_peer:
                if c < len(ps):
                    t = x[ps[c][0]:ps[c][1], gcb:gce]
                    ops.append(dist.P2POp(dist.isend, t if gce - gcb == N1 else t.contiguous(),
                                          g, group))
        works = dist.batch_isend_irecv(ops) if ops else []
        # ... and its own block only after the sends complete: launched alongside, a
        # persistent K1 grid that takes every SM first would hold the send kernel back
        # until the whole block is done (and every receiver with it).  tune_split shortens
        # this rank's band by `lead` to pay for the wait.
        for w in works:
            w.wait()
        local = x[rb:re, cb:ce]
        if b > a and ce > cb:
            compute(local, 0, b - a)
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
        # Every piece's receive is posted (one group each: a group completes as a whole, so
        # per-piece groups are what lets compute start on the first piece) before any
        # compute is launched.  On CUDA the pieces' computes alternate between the current
        # stream and a side stream, so a later piece's CTAs fill SMs as the previous
        # piece's retire instead of waiting for its last CTA (scripts/split_scaling.py:
        # "pipe2" vs "pipe1"); the current stream joins the side stream at the end.
        # compute() runs on torch's current stream.  (A later piece's receive kernel
        # queues behind the earlier one on the NCCL stream; if the first piece's K1 grid
        # takes every SM first, that receive waits for it: the step then degrades to the
        # serial schedule plus the first piece's transfer, never worse.)
        cur = torch.cuda.current_stream(device) if device.type == "cuda" else None
        side = _side_stream(device) if cur is not None and len(wb) > 2 else None
        if side is not None:
            side.wait_stream(cur)
        for c in range(len(wb) - 1):
            st = side if side is not None and c % 2 == 1 else cur
            with torch.cuda.stream(st) if st is not None else _nullctx():
                for w in works[c]:
                    w.wait()  # NCCL: the compute stream waits for this chunk only
                compute(local, wb[c], wb[c + 1])
        if side is not None:
            cur.wait_stream(side)
    return local, mine


_SIDE = {}


def _side_stream(device):
    """One side stream per device for the pipelined receive path."""
    idx = device.index if device.index is not None else torch.cuda.current_device()
    if idx not in _SIDE:
        _SIDE[idx] = torch.cuda.Stream(torch.device("cuda", idx))
    return _SIDE[idx]


class _nullctx:
    def __enter__(self):
        return None

    def __exit__(self, *exc):
        return False


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
                          precision=None, budget=None, pieces=None,
                          split="auto", lead: int = 0) -> ShardedCoefficients:
    """Sharded tree_swdft_2d: every rank returns its own block of the output.

    On ``src`` pass the full input tensor (CUDA); elsewhere pass x=None plus
    ``shape`` and ``dtype``.  ``split``: "auto" (measured on ``src`` once per shape and
    broadcast, choose_split), "strips" (window-row strips, world x 1) or an explicit
    (gr, gc).  Budget accounting is the reference's, per block.
    """
    from .tree2d import _OUT_DTYPES, _precision_code, forward_into

    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
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
    in_bytes = torch.empty((), dtype=dtype).element_size()
    if split == "auto":
        ch = choose_split(x if rank == src else None, shape, m0, m1, prec, world, in_bytes,
                          group, src)
        split = tuple(ch["split"])
        if pieces is None:
            # the lead shortens rank 0's band: the source's only when the source is rank 0
            pieces, lead = ch["pieces"], (ch.get("lead", 0) if src == 0 else 0)
    elif split in (None, "strips"):
        split = (world, 1)
    gr, gc = split
    a, b, c0, c1, rb, re, cb, ce = block_plan(P0, P1, m0, m1, gr, gc, lead)[rank]
    if b > a and c1 > c0:
        bshape = (re - rb, ce - cb)
        core.check_budget(core.lattice_bytes(bshape, spec) + core.output_bytes(bshape, spec),
                          budget, what="level buffers + coefficient output")
    out = torch.empty((b - a, c1 - c0, n0, n1), dtype=_OUT_DTYPES[prec], device=device)
    scale = core.normalization_factor(spec)
    if pieces is None:
        pieces = choose_pieces(shape, m0, m1, in_bytes, out.element_size(), world)

    def compute(local, w0, w1):
        forward_into(local, m0, m1, out[w0:w1], prec=prec, scale=scale, p0_begin=w0, p0_end=w1)

    pipelined_block_forward(x, shape, m0, m1, split, dtype, device, compute, group, src,
                            pieces=pieces, lead=lead)
    return ShardedCoefficients(out, a, b, tuple(shape), spec, spec.normalization, c0, c1)


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
