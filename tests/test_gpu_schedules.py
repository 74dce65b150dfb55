"""GPU parity of the PRODUCTION K1 launch schedules at the BASELINE configs' full sizes.

K1 picks a schedule per launch (csrc/abi.cu k1_plan, queried through
swdft2d_k1_schedule): uniform row chunks on a persistent grid, guided big-first
chunks handed out by a tile counter (configs 3 and 4), or a one-shot grid of
full-height tiles (config 5).  The small-shape suites never reach the last two, so
here:
  * configs 3 and 4 run FULL SIZE in fp64 and are compared bit for bit with the
    oracle (the restated reference, tree2d.py:30-129) on full-width 128-row strips —
    the first rows, the rows straddling the first two guided chunk boundaries, the
    last rows — and over EVERY row with the independent on-device schedule KR + KC
    (the separable factorisation, bitwise equal to the tree);
  * config 5's one-shot grid runs in fp64 on a window-row range whose column blocks
    fill >= 3 waves, bitwise against KR + KC and oracle sub-blocks (row AND column
    strips of the input are exact, App. A #5);
  * the fp32 production schedules of configs 3-5 are bitwise equal to K1 re-run on
    short row ranges (other tiles, other warm-up rows: each node's arithmetic does
    not depend on the schedule);
  * the stream-K schedule (equal contiguous shares of the column-block-major row space;
    config 2, column blocks of config 4) in fp64, bitwise against KR + KC on every row
    and the oracle around the rows where shares start;
  * the guided tile counter (one slot per stream, zeroed by each launch's last fetch)
    survives back-to-back launches and concurrent streams;
  * the randomised fuzz runs with the schedule overrides forced, so small shapes go
    through every branch of k1_plan.
"""
import json
import os
import subprocess
import sys

import numpy as np
import pytest
import torch

from conftest import ROOT
from paper_1707_08213_b200 import WindowSpec, forward_into, tree_swdft_2d
from paper_1707_08213_b200 import _lib
from paper_1707_08213_b200.workloads import CONFIGS

pytestmark = pytest.mark.gpu

STRIP = 128  # window rows per oracle strip


def bits_equal_np(a, b):
    return a.shape == b.shape and np.array_equal(np.ascontiguousarray(a).view(np.uint64),
                                                 np.ascontiguousarray(b).view(np.uint64))


def bits_equal_dev(a, b):
    """Bitwise equality of two complex device tensors (-0.0 != +0.0, NaN payloads too)."""
    if a.shape != b.shape or a.dtype != b.dtype:
        return False
    ib = torch.int64 if a.dtype == torch.complex128 else torch.int32
    return torch.equal(torch.view_as_real(a).view(ib), torch.view_as_real(b).view(ib))


def strip_starts(sched, P0):
    """Oracle strips: the first rows, rows straddling chunk boundaries 1 and 2, the last rows."""
    starts = [0]
    for c in (1, 2):
        if c < len(sched["bounds"]) - 1:
            starts.append(max(0, min(P0 - STRIP, sched["bounds"][c] - STRIP // 2)))
    starts.append(P0 - STRIP)
    return sorted(set(starts))


def compare_with_separable(x, cfg, out, prec, p0_begin=0, chunk_bytes=2 << 30):
    """Every row of ``out`` (window rows [p0_begin, p0_begin + len(out))) bitwise against
    the KR + KC path computed strip by strip into a scratch buffer."""
    row_bytes = out[0].numel() * out.element_size()
    rows = max(1, chunk_bytes // row_bytes)
    scratch = torch.empty((rows,) + tuple(out.shape[1:]), dtype=out.dtype, device=out.device)
    bad = []
    for a in range(0, out.shape[0], rows):
        b = min(out.shape[0], a + rows)
        forward_into(x, cfg.m0, cfg.m1, scratch[:b - a], prec=prec, p0_begin=p0_begin + a,
                     p0_end=p0_begin + b, kernel="separable")
        if not bits_equal_dev(out[a:b], scratch[:b - a]):
            bad.append((a, b))
    del scratch
    return bad


@pytest.mark.parametrize("name", ["c3", "c4"])
def test_full_size_fp64_production_schedule_bitwise(cuda, oracle_lib, name):
    cfg = CONFIGS[name]
    x = cfg.generate()
    xd = torch.from_numpy(x).to(cuda)
    sched = _lib.k1_schedule(cfg.N0, cfg.N1, cfg.m0, cfg.m1, _lib.PREC_FP64)
    if name == "c4":
        assert sched["mode"] == "guided", sched
    assert sched["bounds"][0] == 0 and sched["bounds"][-1] == cfg.P0
    assert all(b > a for a, b in zip(sched["bounds"], sched["bounds"][1:]))
    res = tree_swdft_2d(xd, WindowSpec((cfg.m0, cfg.m1)), precision="fp64", budget=1 << 62)
    vals = res.values
    assert vals.dtype == torch.complex128 and tuple(vals.shape) == (cfg.P0, cfg.P1, cfg.n0, cfg.n1)
    threads = len(os.sched_getaffinity(0))
    for a in strip_starts(sched, cfg.P0):
        ref = oracle_lib.tree2d(x[a:a + STRIP + cfg.n0 - 1], cfg.m0, cfg.m1, threads=threads,
                                max_lattice_bytes=1 << 32)
        got = vals[a:a + STRIP].cpu().numpy()
        assert bits_equal_np(got, ref), (name, sched["mode"], a)
        del ref, got
    assert compare_with_separable(xd, cfg, vals, _lib.PREC_FP64) == []
    del vals, res
    torch.cuda.empty_cache()


def test_config5_oneshot_fp64_bitwise(cuda, oracle_lib):
    cfg = CONFIGS["c5"]
    x = cfg.generate()
    xd = torch.from_numpy(x).to(cuda)
    a0, a1 = 512, 512 + 160  # > 2 n0 rows: shorter launches take the short-launch rule
    sched = _lib.k1_schedule(cfg.N0, cfg.N1, cfg.m0, cfg.m1, _lib.PREC_FP64, a0, a1)
    assert sched["mode"] == "oneshot", sched
    assert sched["grid"] == sched["tiles"] == sched["column_blocks"]
    out = torch.empty((a1 - a0, cfg.P1, cfg.n0, cfg.n1), dtype=torch.complex128, device=cuda)
    forward_into(xd, cfg.m0, cfg.m1, out, prec=_lib.PREC_FP64, p0_begin=a0, p0_end=a1)
    assert compare_with_separable(xd, cfg, out, _lib.PREC_FP64, p0_begin=a0) == []
    # oracle sub-blocks: 4 window rows x 64 window columns at the range's ends and middle
    for r in (a0, (a0 + a1) // 2, a1 - 4):
        for c in (0, cfg.P1 // 2, cfg.P1 - 64):
            sub = x[r:r + 4 + cfg.n0 - 1, c:c + 64 + cfg.n1 - 1]
            ref = oracle_lib.tree2d(sub, cfg.m0, cfg.m1, threads=8)
            got = out[r - a0:r - a0 + 4, c:c + 64].cpu().numpy()
            assert bits_equal_np(got, ref), (r, c)
    del out
    torch.cuda.empty_cache()


def streamk_share_rows(sched, rows, n0, picks=(1, 2)):
    """Window rows where stream-K CTA shares begin inside a column block (CTA b's share
    starts at b * L // grid of the column-block-major cost space, each column block
    being n0 - 1 warm-up units followed by its rows; k1_stream.cuh)."""
    U = rows + n0 - 1
    L = sched["column_blocks"] * U
    return [max(0, (b * L // sched["grid"]) % U - (n0 - 1))
            for b in picks + (sched["grid"] // 2, sched["grid"] - 1)]


@pytest.mark.parametrize("case", ["c2", "c4cols"])
def test_streamk_production_schedule_fp64_bitwise(cuda, oracle_lib, case):
    """The stream-K schedule (abi.cu k1_plan: uniform-chunk shapes whose shares span
    >= 2 warm-ups — config 2 whole, and a column block of config 4 as a 1 x 8 partition
    rank owns it) in fp64: every row bitwise against KR + KC, and oracle strips around
    the rows where CTA shares start mid column block (each share starts its own warm-up)."""
    cfg = CONFIGS["c2" if case == "c2" else "c4"]
    x = cfg.generate()
    if case == "c4cols":  # the largest column block of a 1 x 8 split: 511 window columns
        x = np.ascontiguousarray(x[:, :511 + cfg.n1 - 1])
    N0, N1 = x.shape
    P0, P1 = N0 - cfg.n0 + 1, N1 - cfg.n1 + 1
    xd = torch.from_numpy(x).to(cuda)
    sched = _lib.k1_schedule(N0, N1, cfg.m0, cfg.m1, _lib.PREC_FP64)
    assert sched["mode"] == "streamk", sched
    out = torch.empty((P0, P1, cfg.n0, cfg.n1), dtype=torch.complex128, device=cuda)
    forward_into(xd, cfg.m0, cfg.m1, out, prec=_lib.PREC_FP64)
    assert compare_with_separable(xd, cfg, out, _lib.PREC_FP64) == []
    threads = len(os.sched_getaffinity(0))
    strip = 32
    for r in sorted(set(streamk_share_rows(sched, P0, cfg.n0)) | {0, P0 - strip}):
        a = max(0, min(P0 - strip, r - strip // 2))
        ref = oracle_lib.tree2d(x[a:a + strip + cfg.n0 - 1], cfg.m0, cfg.m1, threads=threads)
        assert bits_equal_np(out[a:a + strip].cpu().numpy(), ref), (case, a)
    del out
    torch.cuda.empty_cache()


@pytest.mark.parametrize("name", ["c3", "c4", "c5"])
def test_fp32_production_schedule_equals_short_launches(cuda, name):
    """fp32: the full-size production launch is bitwise equal to K1 over short row ranges
    (uniform chunks, other tile boundaries and warm-up rows)."""
    cfg = CONFIGS[name]
    xd = torch.from_numpy(cfg.generate()).to(cuda)
    sched = _lib.k1_schedule(cfg.N0, cfg.N1, cfg.m0, cfg.m1, _lib.PREC_FP32)
    expect = {"c3": "guided", "c4": "guided", "c5": "oneshot"}[name]
    assert sched["mode"] == expect, sched
    out = torch.empty((cfg.P0, cfg.P1, cfg.n0, cfg.n1), dtype=torch.complex64, device=cuda)
    forward_into(xd, cfg.m0, cfg.m1, out, prec=_lib.PREC_FP32)
    rows = 61  # prime-ish: no strip boundary coincides with a production chunk boundary
    scratch = torch.empty((rows,) + tuple(out.shape[1:]), dtype=out.dtype, device=cuda)
    bad = []
    # every row for c3 / c4, a third of c5 (129 GB): strips spaced over the whole range
    step = rows if name != "c5" else 3 * rows
    for a in range(0, cfg.P0, step):
        b = min(cfg.P0, a + rows)
        forward_into(xd, cfg.m0, cfg.m1, scratch[:b - a], prec=_lib.PREC_FP32, p0_begin=a,
                     p0_end=b)
        if not bits_equal_dev(out[a:b], scratch[:b - a]):
            bad.append(a)
    assert bad == []
    del out, scratch
    torch.cuda.empty_cache()


def test_guided_counter_reuse_and_concurrent_streams(cuda):
    """The guided schedule's tile counter is one slot per stream that each launch leaves
    zeroed: 6 back-to-back launches on one stream, then 2 streams at once, same bits."""
    N0, N1, m0, m1 = 600, 2400, 4, 4
    sched = _lib.k1_schedule(N0, N1, m0, m1, _lib.PREC_FP32)
    assert sched["mode"] == "guided" and sched["tiles"] > sched["grid"], sched
    g = torch.Generator().manual_seed(5)
    xd = torch.randn((N0, N1), generator=g).to(cuda)
    P0, P1 = N0 - 15, N1 - 15
    ref = torch.empty((P0, P1, 16, 16), dtype=torch.complex64, device=cuda)
    forward_into(xd, m0, m1, ref, prec=_lib.PREC_FP32, kernel="separable")
    outs = [torch.full_like(ref, float("nan")) for _ in range(3)]
    for k in range(6):
        forward_into(xd, m0, m1, outs[k % 3], prec=_lib.PREC_FP32)
    torch.cuda.synchronize()
    assert all(float((o - ref).abs().max()) <= 1e-3 for o in outs)
    assert bits_equal_dev(outs[0], outs[1]) and bits_equal_dev(outs[1], outs[2])
    s1, s2 = torch.cuda.Stream(cuda), torch.cuda.Stream(cuda)
    c1, c2 = torch.full_like(ref, float("nan")), torch.full_like(ref, float("nan"))
    torch.cuda.synchronize()
    for _ in range(3):
        forward_into(xd, m0, m1, c1, prec=_lib.PREC_FP32, stream=s1)
        forward_into(xd, m0, m1, c2, prec=_lib.PREC_FP32, stream=s2)
    torch.cuda.synchronize()
    assert bits_equal_dev(c1, outs[0]) and bits_equal_dev(c2, outs[0])
    # and inside a CUDA graph: replays reuse the same counter
    graph = torch.cuda.CUDAGraph()
    cap = torch.cuda.Stream(cuda)
    c3 = torch.full_like(ref, float("nan"))
    cap.wait_stream(torch.cuda.current_stream())
    with torch.cuda.graph(graph, stream=cap):
        forward_into(xd, m0, m1, c3, prec=_lib.PREC_FP32, stream=cap)
    for _ in range(4):
        c3.fill_(float("nan"))
        graph.replay()
        torch.cuda.synchronize()
        assert bits_equal_dev(c3, outs[0])


@pytest.mark.parametrize("env", [
    {"SWDFT2D_K1_GUIDED": "1"},
    {"SWDFT2D_K1_GUIDED": "0"},
    {"SWDFT2D_K1_ONESHOT": "1"},
    {"SWDFT2D_K1_ONESHOT": "1", "SWDFT2D_K1_GUIDED": "1"},
    {"SWDFT2D_K1_RCH": "3"},
    {"SWDFT2D_K1_RCH": "3", "SWDFT2D_K1_GUIDED": "0"},
    {"SWDFT2D_K1_STREAMK": "1"},
    {"SWDFT2D_K1_STREAMK": "3"},
    {"SWDFT2D_K1_STREAMK": "0"},
    {"SWDFT2D_K1_STREAMK": "2", "SWDFT2D_TMA": "1"},
    {"SWDFT2D_K1_GUIDED": "1", "SWDFT2D_TMA": "1"},
    {"SWDFT2D_SEP_COLS": "k1"},
    {"SWDFT2D_SEP_COLS": "kc"},
], ids=lambda e: ",".join(f"{k[8:]}={v}" for k, v in e.items()))
def test_fuzz_under_schedule_overrides(env):
    # the column-tree overrides act on the large-window path: full window range there
    k1_only = [] if "SWDFT2D_SEP_COLS" in env else ["--k1-only"]
    r = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "fuzz_parity.py"),
                        "--cases", "40", "--seed", "23"] + k1_only,
                       capture_output=True, text=True, timeout=900, env={**os.environ, **env})
    lines = [line for line in r.stdout.splitlines() if line.startswith("{")]
    assert lines, r.stdout + r.stderr
    summary = json.loads(lines[-1])
    assert r.returncode == 0 and summary["fails"] == 0, "\n".join(lines)
    assert summary["cases"] >= 30


@pytest.mark.parametrize("case", [("c2", 30, 100), ("c3", 40, 1000), ("c4", 32, 2000),
                                  ("c5", 100, 700)], ids=lambda c: c[0])
@pytest.mark.parametrize("precision", ["fp64", "fp32"])
def test_short_launch_streamk_bitwise(cuda, oracle_lib, case, precision):
    """Launches of at most 2 n0 window rows take one wave of stream-K shares (abi.cu
    k1_plan, short-launch rule): every row bitwise against KR + KC (fp64) and the oracle on
    sub-blocks at both ends and the middle of the range; fp32 bitwise against the
    production launch of the whole config (K1's fp32 results do not depend on tiling)."""
    name, rows, a0 = case
    cfg = CONFIGS[name]
    x = cfg.generate()
    xd = torch.from_numpy(x).to(cuda)
    prec = _lib.PREC_FP64 if precision == "fp64" else _lib.PREC_FP32
    a1 = a0 + rows
    sched = _lib.k1_schedule(cfg.N0, cfg.N1, cfg.m0, cfg.m1, prec, a0, a1)
    assert sched["mode"] == "streamk" and sched["grid"] <= sched["slots"], sched
    odt = torch.complex128 if precision == "fp64" else torch.complex64
    out = torch.empty((rows, cfg.P1, cfg.n0, cfg.n1), dtype=odt, device=cuda)
    forward_into(xd, cfg.m0, cfg.m1, out, prec=prec, p0_begin=a0, p0_end=a1)
    if precision == "fp64":
        assert compare_with_separable(xd, cfg, out, prec, p0_begin=a0) == []
        for r in (a0, a0 + rows // 2, a1 - 2):
            for c in (0, cfg.P1 // 2, cfg.P1 - 48):
                sub = x[r:r + 2 + cfg.n0 - 1, c:c + 48 + cfg.n1 - 1]
                ref = oracle_lib.tree2d(sub, cfg.m0, cfg.m1, threads=8)
                assert bits_equal_np(out[r - a0:r - a0 + 2, c:c + 48].cpu().numpy(), ref), (r, c)
    else:
        full = torch.empty((a1 + 1, cfg.P1, cfg.n0, cfg.n1), dtype=odt, device=cuda)
        forward_into(xd[:a1 + cfg.n0], cfg.m0, cfg.m1, full, prec=prec)
        assert bits_equal_dev(out, full[a0:a1])
        del full
    del out
    torch.cuda.empty_cache()
