"""On-device tri-oracle verification and the Figure-4 benchmark CSV.

``verify`` mirrors the reference's ``swdft verify`` (/root/reference/pkg/src/swdft/
cli.py:142-155): the tree transform, the per-window FFT and the naive double sum
of the same input, passing iff max|tree - naive| <= 1e-10 and the tree equals the
per-window FFT exactly.  Here all three run on the GPU in float64: the tree is K1,
the per-window FFT is K0 (the reference DAG per window, oracle.swfft_2d), the naive
sum is the literal Eq. 2 contraction with exp-built DFT matrices (oracle.py:31-34,
60-72) as batched complex128 matrix products.  ``corrupt`` flips one bit of the
tree output first (the reference's hidden --corrupt detector test, cli.py:149-151).

``bench_records`` / ``to_csv`` mirror bench.run_bench / bench.to_csv
(bench.py:133-185): median-of-repetitions timings of tree / fft / naive on one
seeded complex input, in the reference's CSV format, timed on the device.
"""
from __future__ import annotations

import io
import math
import statistics
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib, core
from .tree2d import _to_tensor, forward_into

ALGORITHMS = ("tree", "fft", "naive")
CSV_HEADER = "algorithm,N0,N1,n0,n1,seconds,ops,peak_bytes"


def _dft_matrix(n: int, device) -> torch.Tensor:
    jk = np.outer(np.arange(n), np.arange(n))
    return torch.from_numpy(np.exp((-2j * np.pi / n) * jk)).to(device)


def naive_2d(xt: torch.Tensor, m0: int, m1: int) -> torch.Tensor:
    """Eq. 2 per window: F0 @ W @ F1^T over every window view (complex128)."""
    n0, n1 = 1 << m0, 1 << m1
    w = xt.to(torch.complex128).unfold(0, n0, 1).unfold(1, n1, 1)  # [P0, P1, n0, n1]
    f0 = _dft_matrix(n0, xt.device)
    f1 = _dft_matrix(n1, xt.device)
    return torch.einsum("kj,pqjl,ml->pqkm", f0, w, f1)


def _run(xt, m0, m1, algorithm):
    n0, n1 = 1 << m0, 1 << m1
    P0, P1 = xt.shape[0] - n0 + 1, xt.shape[1] - n1 + 1
    if algorithm == "naive":
        return naive_2d(xt, m0, m1)
    out = torch.empty((P0, P1, n0, n1), dtype=torch.complex128, device=xt.device)
    forward_into(xt, m0, m1, out, prec=_lib.PREC_FP64,
                 kernel="stream" if algorithm == "tree" and _lib.has_stream_kernel(m0, m1, 1)
                 else ("window" if algorithm == "fft" else "auto"))
    return out


def verify(x, window, budget=None, corrupt: bool = False, device=None):
    """Returns (max_err, exact_fft_match, ok) as cmd_verify prints / exits on."""
    spec = core.WindowSpec.from_sizes(window)
    xt = _to_tensor(x)
    if xt.dim() != 2 or spec.k != 2:
        raise core.ShapeError("verify supports 2D arrays and windows")
    shape = tuple(int(s) for s in xt.shape)
    spec.check_fits(shape)
    core.check_budget(core.lattice_bytes(shape, spec) + core.output_bytes(shape, spec), budget,
                      what="level buffers + coefficient output")
    dev = torch.device(device) if device is not None else torch.device(
        "cuda", torch.cuda.current_device())
    xt = xt.to(dev)
    m0, m1 = spec.exponents
    tree = _run(xt, m0, m1, "tree")
    fft = _run(xt, m0, m1, "fft")
    naive = _run(xt, m0, m1, "naive")
    if corrupt:
        tree = tree.clone()
        tree.view(torch.float64).view(torch.int64).view(-1)[0] ^= 1
    max_err = float((tree - naive).abs().max()) if tree.numel() else 0.0
    exact = bool(torch.equal(tree, fft))
    return max_err, exact, (max_err <= 1e-10 and exact)


@dataclass
class BenchRecord:
    algorithm: str
    shape: tuple
    window: tuple
    seconds: float
    ops: int
    peak_bytes: int


def tree_op_count(shape, sizes) -> int:
    """bench.tree_op_breakdown total (bench.py:47-62): enumerate the level geometry."""
    spec = core.WindowSpec.from_sizes(sizes)
    return sum(nodes * positions for _, nodes, positions in core.level_regions(shape, spec))


def predict_ops(algorithm, shape, sizes) -> int:
    """bench.predict_ops (bench.py:65-82)."""
    spec = core.WindowSpec.from_sizes(sizes)
    spec.check_fits(shape)
    positions = math.prod(N - n + 1 for N, n in zip(shape, spec.sizes))
    w = spec.window_elements
    if algorithm == "tree":
        return tree_op_count(shape, sizes)
    if algorithm == "naive":
        return positions * w * w
    return positions * (w // 2) * spec.total_levels


def bench_records(shape=(100, 100), windows=((4, 4), (8, 8), (16, 16), (32, 32), (64, 64)),
                  algorithms=ALGORITHMS, repetitions: int = 5, seed: int = 0, device=None,
                  naive_max_bytes: int = 8 << 30):
    """Device-timed median of ``repetitions`` runs per (algorithm, window) on the
    reference's seeded input (bench.py:140-141).  ``peak_bytes`` is this build's
    device footprint (input + complex128 output; naive adds its window views)."""
    rng = np.random.default_rng(seed)
    x = rng.standard_normal(shape) + 1j * rng.standard_normal(shape)
    dev = torch.device(device) if device is not None else torch.device(
        "cuda", torch.cuda.current_device())
    xt = torch.from_numpy(x).to(dev)
    recs = []
    for algorithm in algorithms:
        for sizes in windows:
            spec = core.WindowSpec.from_sizes(sizes)
            m0, m1 = spec.exponents
            out_bytes = core.output_bytes(shape, spec)
            peak = xt.numel() * 16 + out_bytes * (2 if algorithm == "naive" else 1)
            if algorithm == "naive" and peak > naive_max_bytes:
                continue
            _run(xt, m0, m1, algorithm)
            times = []
            for _ in range(max(1, repetitions)):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                _run(xt, m0, m1, algorithm)
                e1.record()
                torch.cuda.synchronize()
                times.append(e0.elapsed_time(e1) / 1e3)
            recs.append(BenchRecord(algorithm, tuple(shape), tuple(sizes), statistics.median(times),
                                    predict_ops(algorithm, shape, sizes), peak))
    return recs


def to_csv(records) -> str:
    """bench.to_csv (bench.py:175-185): ordered by algorithm then window size."""
    buf = io.StringIO()
    buf.write(CSV_HEADER + "\n")
    for r in sorted(records, key=lambda r: (r.algorithm, r.window[0] * r.window[1], r.window)):
        buf.write(f"{r.algorithm},{r.shape[0]},{r.shape[1]},{r.window[0]},{r.window[1]},"
                  f"{r.seconds!r},{r.ops},{r.peak_bytes}\n")
    return buf.getvalue()
