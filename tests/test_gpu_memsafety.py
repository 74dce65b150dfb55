"""Memory-safety checks of every device path, standing in for compute-sanitizer memcheck
(closed on this GPU pool) on the reference's disjoint-writer contract
(tree2d.py:22-27,58-64; core.py:309-312: every output element written once, nothing
outside the output written):

  * the output is a view into a larger buffer whose guard rows (one full output row,
    P1 x n0 x n1 coefficients, before and after) hold a sentinel bit pattern; after the
    launch the guards must still hold it bit for bit (no write outside the output) and no
    output element may still hold it (no element left unwritten);
  * the input is a view into a NaN-filled padded buffer (row stride > N1, rows and
    columns of NaN around it): a read outside the input that fed a node would turn that
    coefficient into NaN, and the output must be bitwise equal to the oracle (fp64) or
    within BASELINE's tolerance (fp32).

Covers K1 (register prefetch and TMA staging, every schedule its rule picks on these
shapes), K0, KR (n0 = 1), the large-window path (KR + K1's Z-column kernel or KC), window
row sub-ranges and normalization scales.
"""
import numpy as np
import pytest
import torch

import oracle
from paper_1707_08213_b200 import _lib
from paper_1707_08213_b200.tree2d import forward_into

pytestmark = pytest.mark.gpu

SENT64 = np.uint64(0x7FF4DEADBEEF0001)  # a signalling-NaN payload no kernel produces
SENT32 = np.uint32(0x7FA0DEAD)

CASES = [  # (N0, N1, m0, m1, kernel, precision, p0 range as fractions, scale)
    (40, 37, 3, 2, "stream", "fp64", (0.0, 1.0), None),
    (40, 37, 3, 2, "stream_tma", "fp64", (0.2, 0.7), 0.125),
    (70, 33, 4, 4, "auto", "fp32", (0.0, 1.0), None),
    (96, 80, 5, 3, "auto", "fp64", (0.1, 0.9), None),
    (130, 70, 6, 6, "auto", "fp32", (0.0, 1.0), 1 / 64),
    (70, 70, 6, 5, "stream", "fp64", (0.3, 1.0), None),
    (33, 29, 2, 3, "window", "fp64", (0.0, 1.0), None),
    (9, 300, 0, 6, "rows", "fp64", (0.0, 1.0), None),
    (5, 1100, 0, 10, "auto", "fp32", (0.0, 1.0), None),
    (300, 20, 7, 2, "auto", "fp32", (0.0, 1.0), None),
    (300, 20, 7, 2, "separable", "fp64", (0.25, 0.75), None),
    (130, 40, 7, 4, "auto", "fp64", (0.0, 1.0), None),
    (70, 300, 2, 8, "auto", "fp32", (0.0, 1.0), None),
    (600, 12, 9, 1, "auto", "fp32", (0.0, 1.0), None),
    (8, 8, 3, 3, "auto", "fp64", (0.0, 1.0), None),  # one window
]


def _sentinel_view(t: torch.Tensor):
    return t.view(torch.int64) if t.dtype == torch.complex128 else t.view(torch.int32)


def _fill_sentinel(t: torch.Tensor):
    v = _sentinel_view(t)
    s = SENT64 if t.dtype == torch.complex128 else SENT32
    v.fill_(int(np.array(s).view(np.int64 if t.dtype == torch.complex128 else np.int32)))


def _count_sentinel(t: torch.Tensor) -> int:
    a = _sentinel_view(t).cpu().numpy()
    s = SENT64.view(np.int64) if t.dtype == torch.complex128 else SENT32.view(np.int32)
    return int((a == s).sum())


@pytest.mark.parametrize("case", CASES, ids=lambda c: f"{c[0]}x{c[1]}_{1 << c[2]}x{1 << c[3]}_{c[4]}_{c[5]}")
def test_guard_bands_and_padded_input(cuda, case):
    N0, N1, m0, m1, kernel, prec, (fa, fb), scale = case
    n0, n1 = 1 << m0, 1 << m1
    P0, P1 = N0 - n0 + 1, N1 - n1 + 1
    a, b = int(P0 * fa), max(int(P0 * fa) + 1, int(round(P0 * fb)))
    rng = np.random.default_rng(N0 * 1000 + N1 + m0 * 7 + m1)
    x = rng.standard_normal((N0, N1))
    if prec == "fp32":
        x = x.astype(np.float32)
    xdt = torch.float64 if x.dtype == np.float64 else torch.float32
    pad = torch.full((N0 + 3, N1 + 9), float("nan"), dtype=xdt, device=cuda)
    xv = pad[1:N0 + 1, 4:N1 + 4]
    xv.copy_(torch.from_numpy(x))
    assert xv.stride(0) == N1 + 9
    odt = torch.complex128 if prec == "fp64" else torch.complex64
    big = torch.empty((b - a + 2, P1, n0, n1), dtype=odt, device=cuda)
    _fill_sentinel(big)
    out = big[1:b - a + 1]
    assert out.is_contiguous()
    forward_into(xv, m0, m1, out, prec=_lib.PREC_FP32 if prec == "fp32" else _lib.PREC_FP64,
                 scale=1.0 if scale is None else scale, p0_begin=a, p0_end=b, kernel=kernel)
    torch.cuda.synchronize()
    per_row = 2 * P1 * n0 * n1  # (re, im) words per output row
    assert _count_sentinel(big[:1]) == per_row, "write before the output"
    assert _count_sentinel(big[-1:]) == per_row, "write after the output"
    assert _count_sentinel(out) == 0, "output elements left unwritten"
    ref = oracle.tree2d(x, m0, m1, a, b, scale=scale)
    got = out.cpu().numpy()
    if prec == "fp64":
        assert np.array_equal(got.view(np.uint64), ref.view(np.uint64))
    else:
        assert np.isfinite(got.view(np.float32)).all()
        assert oracle.window_rel_err(got, ref) <= 1e-4


CONFIG_CASES = [  # (config, precision, window-row range or None = all, expected K1 schedule)
    ("c2", "fp32", None, "streamk"),
    ("c2", "fp64", None, "streamk"),
    ("c3", "fp32", (0, 700), "guided"),
    ("c4", "fp32", None, "guided"),
    ("c5", "fp32", (100, 420), "oneshot"),
]


@pytest.mark.parametrize("case", CONFIG_CASES, ids=lambda c: f"{c[0]}_{c[1]}")
def test_guard_bands_production_schedules(cuda, case):
    """The BASELINE configs on the schedules their launches use (stream-K, guided chunks
    with the tile counter, one-shot full-height tiles): guard rows untouched, every output
    element written, every coefficient finite."""
    from paper_1707_08213_b200.workloads import CONFIGS

    name, prec, rows, mode = case
    cfg = CONFIGS[name]
    pc = _lib.PREC_FP32 if prec == "fp32" else _lib.PREC_FP64
    a, b = rows if rows else (0, cfg.P0)
    assert _lib.k1_schedule(cfg.N0, cfg.N1, cfg.m0, cfg.m1, pc, a, b)["mode"] == mode
    x = torch.from_numpy(cfg.generate()).to(cuda)
    odt = torch.complex128 if prec == "fp64" else torch.complex64
    big = torch.empty((b - a + 2, cfg.P1, cfg.n0, cfg.n1), dtype=odt, device=cuda)
    _fill_sentinel(big)
    out = big[1:b - a + 1]
    forward_into(x, cfg.m0, cfg.m1, out, prec=pc, p0_begin=a, p0_end=b)
    torch.cuda.synchronize()
    per_row = 2 * cfg.P1 * cfg.n0 * cfg.n1
    assert _count_sentinel(big[:1]) == per_row, "write before the output"
    assert _count_sentinel(big[-1:]) == per_row, "write after the output"
    w = out.view(torch.float64 if prec == "fp64" else torch.float32)
    # every element written (no sentinel NaN left) and no NaN/inf produced: one pass
    assert bool(torch.isfinite(w).all().item()), "unwritten or non-finite coefficients"
    del big, out, w, x
    torch.cuda.empty_cache()
