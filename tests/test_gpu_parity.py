"""GPU parity: libswdft2d.so (through the C ABI / drop-in wrapper) vs the pinned oracle
and the reference's golden vectors.

fp64 ("DAG-exact") must be BITWISE equal to the reference.  fp32 must satisfy
BASELINE.json's tolerance: max_k |a_gpu - a_ref| / ||a_ref window||_2 <= 1e-4.
"""
import os

import numpy as np
import pytest
import torch

from conftest import sha
from golden_inputs import acc_input, kat6_input
from paper_1707_08213_b200 import (BudgetError, OpCounter, ShapeError, WindowSpec,
                                   WindowTooLargeError, forward_into, tree_swdft_2d)
from paper_1707_08213_b200 import _lib
from paper_1707_08213_b200.workloads import CONFIGS

pytestmark = pytest.mark.gpu

FP32_TOL = 1e-4  # BASELINE.json north_star, complex64 mode
FP64_TOL = 1e-10  # BASELINE.json north_star, fp64 mode (we require bitwise anyway)
KERNELS = ("stream", "window", "stream_tma")


def rel_err(got, ref):
    import oracle

    return oracle.window_rel_err(got, ref)


def run(x, m0, m1, precision, kernel="auto", normalization="none"):
    spec = WindowSpec((m0, m1), normalization)
    res = tree_swdft_2d(x, spec, precision=precision, kernel=kernel, budget=1 << 62)
    return res.values.cpu().numpy()


def bits_equal(a, b):
    return a.shape == b.shape and np.array_equal(a.view(np.uint64), b.view(np.uint64))


@pytest.mark.parametrize("kernel", KERNELS)
def test_kats_fp64_bitwise(golden, cuda, kernel):
    meta, arr = golden
    x = np.array(meta["kat"]["kat1"]["x"])
    assert bits_equal(run(x, 1, 1, "fp64", kernel), arr["kat1_out"])
    assert bits_equal(run(np.ones((8, 8)), 2, 2, "fp64", kernel), arr["kat2_out"])
    k6, nx = kat6_input()
    assert bits_equal(run(k6, 1, 2, "fp64", kernel), arr["kat6_out"])
    for mode in ("unitary", "paper-2d"):
        assert bits_equal(run(nx, 2, 1, "fp64", kernel, mode), arr[f"norm_{mode}_out"])


@pytest.mark.parametrize("kernel", KERNELS)
def test_acceptance_sweep_fp64_bitwise(golden, cuda, kernel):
    """SPEC.md acceptance 1+2 on the GPU: 800 (array, window) cases, SHA-256 equal to the reference."""
    meta, _ = golden
    bad = []
    for rec in meta["acc"]:
        x = acc_input(rec["case"])
        out = run(x, rec["m0"], rec["m1"], "fp64", kernel)
        if sha(out) != rec["sha"]:
            bad.append((rec["case"], rec["m0"], rec["m1"]))
    assert not bad, f"{len(bad)} mismatches, first {bad[:5]}"


def test_acceptance_sweep_fp32_tolerance(cuda, oracle_lib):
    for case in range(0, 50, 3):
        x = acc_input(case)
        for m0 in range(4):
            for m1 in range(4):
                if (1 << m0) > x.shape[0] or (1 << m1) > x.shape[1]:
                    continue
                ref = oracle_lib.tree2d(x, m0, m1)
                for kernel in KERNELS:
                    got = run(x.astype(np.complex64), m0, m1, "fp32", kernel)
                    assert rel_err(got, ref) <= FP32_TOL


@pytest.mark.parametrize("kernel", KERNELS)
def test_config1_full_bitwise(golden, cuda, kernel):
    meta, _ = golden
    cfg = CONFIGS["c1"]
    x = cfg.generate()
    out = run(x, cfg.m0, cfg.m1, "fp64", kernel)
    assert sha(out) == meta["configs"]["c1"]["full_sha"]


@pytest.mark.parametrize("name", ["c2", "c3", "c4", "c5"])
def test_config_strips_fp64_bitwise_and_fp32(golden, cuda, oracle_lib, name):
    """Small strips of configs 2-5: fp64 mode bitwise vs the reference's SHA-256;
    fp32 mode within tolerance of the (pinned) oracle."""
    meta, _ = golden
    cfg = CONFIGS[name]
    x = cfg.generate()
    assert sha(x) == meta["configs"][name]["in_sha"]
    for st in meta["configs"][name]["strips"]:
        sub = x[st["p0"]:st["p0"] + st["rows"] + cfg.n0 - 1, st["p1"]:st["p1"] + st["cols"] + cfg.n1 - 1]
        sub = np.ascontiguousarray(sub)
        for kernel in KERNELS:
            assert sha(run(sub, cfg.m0, cfg.m1, "fp64", kernel)) == st["sha"]
        ref = oracle_lib.tree2d(sub, cfg.m0, cfg.m1)
        for kernel in KERNELS:
            assert rel_err(run(sub, cfg.m0, cfg.m1, "fp32", kernel), ref) <= FP32_TOL


@pytest.mark.parametrize("name", ["c2", "c3", "c4", "c5"])
def test_config_full_size_fp32(golden, cuda, name):
    """The full BASELINE config on the GPU (complex64): sampled windows vs the
    reference's golden values and numpy fft2; size-independent properties over
    EVERY window: DC = window sum and Parseval, against fp64 box sums."""
    meta, arr = golden
    cfg = CONFIGS[name]
    x = cfg.generate()
    spec = WindowSpec((cfg.m0, cfg.m1))
    res = tree_swdft_2d(x, spec, budget=1 << 62)
    vals = res.values
    assert vals.dtype == torch.complex64 and tuple(vals.shape) == (cfg.P0, cfg.P1, cfg.n0, cfg.n1)
    for (p0, p1), ref in zip(arr[f"{name}_win_pos"], arr[f"{name}_win_out"]):
        got = vals[p0, p1].cpu().numpy()[None, None]
        assert rel_err(got, ref[None, None]) <= FP32_TOL
        f = np.fft.fft2(x[p0:p0 + cfg.n0, p1:p1 + cfg.n1].astype(np.complex128))
        assert rel_err(got, f[None, None]) <= FP32_TOL
    # independent check: numpy fft2 of 1024 windows per config —
    # the four corners, edge midpoints, and seeded random positions
    rng = np.random.default_rng(int(name[1:]) + 97)
    pts = [(0, 0), (0, cfg.P1 - 1), (cfg.P0 - 1, 0), (cfg.P0 - 1, cfg.P1 - 1),
           (cfg.P0 // 2, 0), (0, cfg.P1 // 2), (cfg.P0 - 1, cfg.P1 // 2), (cfg.P0 // 2, cfg.P1 - 1)]
    pts += list(zip(rng.integers(0, cfg.P0, 1024 - len(pts)), rng.integers(0, cfg.P1, 1024 - len(pts))))
    p0s = torch.tensor([p[0] for p in pts], device=vals.device)
    p1s = torch.tensor([p[1] for p in pts], device=vals.device)
    got = vals[p0s, p1s].cpu().numpy()
    xw = np.stack([x[a:a + cfg.n0, b:b + cfg.n1] for a, b in pts]).astype(np.complex128)
    ref_w = np.fft.fft2(xw)
    assert rel_err(got[None], ref_w[None]) <= FP32_TOL
    # every window: DC coefficient and Parseval, via fp64 summed-area tables on device
    xd = torch.from_numpy(np.ascontiguousarray(x)).to(cuda).to(torch.complex128)
    n0, n1 = cfg.n0, cfg.n1

    def box(t):
        s = torch.zeros((t.shape[0] + 1, t.shape[1] + 1), dtype=t.dtype, device=t.device)
        s[1:, 1:] = t.cumsum(0).cumsum(1)
        return s[n0:, n1:] - s[:-n0, n1:] - s[n0:, :-n1] + s[:-n0, :-n1]

    dc_ref = box(xd)
    en_ref = box(xd.abs() ** 2).real * (n0 * n1)
    chunk = max(1, (1 << 28) // (cfg.P1 * n0 * n1))
    worst_dc = worst_en = 0.0
    for a in range(0, cfg.P0, chunk):
        b = min(cfg.P0, a + chunk)
        v = vals[a:b]
        nrm = (v.abs().double() ** 2).sum((-1, -2))
        win_norm = torch.sqrt(en_ref[a:b]).clamp_min(1e-30)
        worst_dc = max(worst_dc, float(((v[..., 0, 0].to(torch.complex128) - dc_ref[a:b]).abs() / win_norm).max()))
        worst_en = max(worst_en, float(((nrm - en_ref[a:b]).abs() / en_ref[a:b].clamp_min(1e-30)).max()))
    assert worst_dc <= FP32_TOL, worst_dc
    assert worst_en <= 2e-4, worst_en
    del vals, res
    torch.cuda.empty_cache()


@pytest.mark.parametrize("shape,m", [
    ((8, 8), (3, 3)),      # n = N: a single window position
    ((9, 40), (0, 3)),     # n0 = 1
    ((40, 9), (3, 0)),     # n1 = 1
    ((5, 7), (0, 0)),      # 1x1 windows
    ((37, 29), (2, 4)),    # odd extents, non-square
    ((70, 130), (6, 6)),   # 64x64 windows (K1 V=2 path)
    ((100, 70), (5, 1)),   # n1 < 32, deep dim 0
    ((33, 300), (1, 6)),
    ((300, 20), (6, 2)),
])
def test_edge_shapes(cuda, oracle_lib, shape, m):
    rng = np.random.default_rng(sum(shape) + 7 * m[0] + m[1])
    x = rng.standard_normal(shape) + 1j * rng.standard_normal(shape)
    ref = oracle_lib.tree2d(x, *m)
    for kernel in KERNELS:
        assert bits_equal(run(x, *m, "fp64", kernel), ref), kernel
        assert rel_err(run(x.astype(np.complex64), *m, "fp32", kernel), ref) <= FP32_TOL


def test_input_dtypes_and_strides(cuda, oracle_lib):
    rng = np.random.default_rng(5)
    xr = rng.standard_normal((50, 45))
    ref = oracle_lib.tree2d(xr, 3, 2)
    assert bits_equal(run(xr, 3, 2, "fp64"), ref)                       # float64
    assert bits_equal(run(xr.astype(np.complex128), 3, 2, "fp64"), ref)  # complex128
    xi = rng.integers(-5, 5, (50, 45))
    assert bits_equal(run(xi, 3, 2, "fp64"), oracle_lib.tree2d(xi.astype(float), 3, 2))
    x32 = xr.astype(np.float32)
    assert bits_equal(run(x32, 3, 2, "fp64"), oracle_lib.tree2d(x32.astype(np.float64), 3, 2))
    assert rel_err(run(x32, 3, 2, None), ref) <= FP32_TOL                # default fp32 for f32
    # a strided device view (row stride > width) goes through ld_x
    big = torch.from_numpy(xr).to(cuda)
    pad = torch.zeros((50, 64), dtype=torch.float64, device=cuda)
    pad[:, :45] = big
    view = pad[:, :45]
    assert view.stride(0) == 64
    out = torch.empty((43, 42, 8, 4), dtype=torch.complex128, device=cuda)
    forward_into(view, 3, 2, out, prec=_lib.PREC_FP64)
    assert bits_equal(out.cpu().numpy(), ref)


def test_input_kinds_widen_like_the_reference(cuda, oracle_lib):
    """Whatever np.asarray(x, complex128) accepts (tree2d.py:189) is widened exactly and, with
    the default precision, transformed bitwise: nested lists, bools, small ints, half
    floats, Fortran order, negative strides, read-only arrays, torch host tensors."""
    rng = np.random.default_rng(9)
    xr = rng.standard_normal((21, 19))
    cases = {
        "list": xr.tolist(),
        "bool": rng.random((21, 19)) < 0.5,
        "int8": rng.integers(-100, 100, (21, 19)).astype(np.int8),
        "uint16": rng.integers(0, 60000, (21, 19)).astype(np.uint16),
        "int64": rng.integers(-2**40, 2**40, (21, 19)),
        "float16": xr.astype(np.float16),
        "fortran": np.asfortranarray(xr),
        "reversed": xr[::-1, ::-1],
        "every-other": rng.standard_normal((42, 38))[::2, ::2],
        "torch-host-bf16": torch.from_numpy(xr).to(torch.bfloat16),
        "complex-list": (xr + 1j * xr[::-1]).tolist(),
    }
    ro = xr.copy()
    ro.setflags(write=False)
    cases["read-only"] = ro
    for name, x in cases.items():
        wide = x.to(torch.float64).numpy() if isinstance(x, torch.Tensor) else \
            np.asarray(x, dtype=np.complex128)
        res = tree_swdft_2d(x, WindowSpec((2, 3)), budget=1 << 40)
        assert res.values.dtype == torch.complex128, name
        assert bits_equal(res.values.cpu().numpy(), oracle_lib.tree2d(wide, 2, 3)), name
    with pytest.raises((TypeError, ValueError)):
        tree_swdft_2d([["a", "b"], ["c", "d"]], WindowSpec((1, 1)))


def test_forward_host_c_abi(cuda, oracle_lib):
    """swdft2d_forward_host: host array in, host array out in one C-ABI call (the call the
    reference's numpy binding makes), strips through the 4-slot device ring."""
    import ctypes

    rng = np.random.default_rng(11)
    xr = rng.standard_normal((90, 70))
    ref = oracle_lib.tree2d(xr, 3, 2)                                   # (83, 67, 8, 4)
    row_bytes = 67 * 8 * 4 * 16
    for make in (_lib.host_empty, np.empty):                            # pinned, pageable
        for strip in (0, row_bytes, 3 * row_bytes + 5):                 # 1, 83 and 28 strips
            out = make(ref.shape, np.complex128)
            out.view(np.float64).fill(np.nan)
            _lib.forward_host(xr, 3, 2, out, prec=_lib.PREC_FP64, strip_bytes=strip)
            assert bits_equal(out, ref)
    # a row range of a padded view (row stride > width), scaled
    wide = np.full((90, 96), np.nan)
    wide[:, 5:75] = xr
    out = _lib.host_empty((20, 67, 8, 4), np.complex128)
    _lib.forward_host(wide[:, 5:75], 3, 2, out, prec=_lib.PREC_FP64, scale=0.125, p0_begin=31,
                      p0_end=51, strip_bytes=2 * row_bytes)
    assert bits_equal(out, oracle_lib.tree2d(xr, 3, 2, scale=0.125)[31:51])
    # complex64 in fp32, and the large-window path (its workspace comes from the pool)
    xc = (rng.standard_normal((140, 40)) + 1j * rng.standard_normal((140, 40))).astype(np.complex64)
    out32 = _lib.host_empty((140 - 127, 39, 128, 2), np.complex64)
    _lib.forward_host(xc, 7, 1, out32, prec=_lib.PREC_FP32, strip_bytes=4 * 39 * 256 * 8)
    assert rel_err(out32, oracle_lib.tree2d(xc.astype(np.complex128), 7, 1)) <= FP32_TOL
    out64 = np.empty((140 - 127, 39, 128, 2), np.complex128)
    _lib.forward_host(xc, 7, 1, out64, prec=_lib.PREC_FP64, kernel=_lib.KERNEL_SEPARABLE)
    assert bits_equal(out64, oracle_lib.tree2d(xc.astype(np.complex128), 7, 1))
    # x may also be a device pointer (copied device to device)
    xd = torch.from_numpy(xr).to(cuda)
    out = _lib.host_empty(ref.shape, np.complex128)
    lib = _lib.load()
    _lib.check(lib.swdft2d_forward_host(xd.data_ptr(), _lib.IN_F64, 90, 70, 70, 3, 2, _lib.PREC_FP64,
                                        1.0, 0, 83, out.ctypes.data, 0, _lib.KERNEL_AUTO, None))
    assert bits_equal(out, ref)
    # errors: null buffers, negative strip size, rows out of range; an empty range is a no-op
    assert lib.swdft2d_forward_host(None, _lib.IN_F64, 90, 70, 70, 3, 2, _lib.PREC_FP64, 1.0, 0, 83,
                                    out.ctypes.data, 0, 0, None) == _lib.E_INVALID_ARG
    assert lib.swdft2d_forward_host(xr.ctypes.data, _lib.IN_F64, 90, 70, 70, 3, 2, _lib.PREC_FP64,
                                    1.0, 0, 83, out.ctypes.data, -1, 0, None) == _lib.E_INVALID_ARG
    assert lib.swdft2d_forward_host(xr.ctypes.data, _lib.IN_F64, 90, 70, 70, 3, 2, _lib.PREC_FP64,
                                    1.0, 0, 84, out.ctypes.data, 0, 0, None) == _lib.E_INVALID_ARG
    assert lib.swdft2d_forward_host(xr.ctypes.data, _lib.IN_F64, 90, 70, 70, 3, 2, _lib.PREC_FP64,
                                    1.0, 5, 5, None, 0, 0, None) == _lib.OK
    dout = torch.empty(ref.shape, dtype=torch.complex128, device=cuda)   # a device pointer is refused
    assert lib.swdft2d_forward_host(xr.ctypes.data, _lib.IN_F64, 90, 70, 70, 3, 2, _lib.PREC_FP64,
                                    1.0, 0, 83, dout.data_ptr(), 0, 0, None) == _lib.E_INVALID_ARG
    with pytest.raises(ValueError):
        _lib.forward_host(xr[:, ::2], 3, 2, out, prec=_lib.PREC_FP64)
    assert lib.swdft2d_host_free(None) == _lib.OK and not lib.swdft2d_host_alloc(0)
    del out, out32
    import gc

    gc.collect()  # the pinned blocks are freed with their arrays (weakref.finalize)


def test_download_and_numpy_helper(cuda):
    """swdft2d_download: device tensor -> pinned or pageable host array (the latter through
    the staging workers, several chunks, an odd tail), ordered after the producing stream."""
    g = torch.Generator(device=cuda).manual_seed(3)
    t = torch.randn((9, 1237, 257), dtype=torch.float64, device=cuda, generator=g)
    c = torch.view_as_complex(t[..., :256].reshape(9, 1237, 128, 2).contiguous())   # 18 MB
    ref = c.cpu().numpy()
    got = _lib.download(c)
    assert got.dtype == np.complex128 and got.shape == ref.shape and bits_equal(got, ref)
    pinned = _lib.host_empty(ref.shape, np.complex128)
    _lib.check(_lib.load().swdft2d_download(c.data_ptr(), pinned.ctypes.data, pinned.nbytes, None))
    assert bits_equal(pinned, ref)
    assert _lib.download(c[:, ::3]).shape == (9, 413, 128)                # non-contiguous view
    assert _lib.download(torch.empty((0, 4), dtype=torch.complex64, device=cuda)).shape == (0, 4)
    s = torch.cuda.Stream(cuda)
    with torch.cuda.stream(s):                                            # stream ordering
        big = torch.zeros(1 << 24, dtype=torch.float32, device=cuda)
        for _ in range(20):
            big += 1.0
        assert float(_lib.download(big)[-1]) == 20.0
    res = tree_swdft_2d(np.ones((8, 8)), WindowSpec((2, 2)), budget=1 << 30)
    assert isinstance(res.numpy(), np.ndarray) and bits_equal(res.numpy(), res.values.cpu().numpy())
    assert _lib.load().swdft2d_download(None, pinned.ctypes.data, 8, None) == _lib.E_INVALID_ARG


def test_row_ranges(cuda, oracle_lib):
    """swdft2d_forward on window-row sub-ranges (the strip boundary) is bitwise exact."""
    rng = np.random.default_rng(9)
    x = rng.standard_normal((90, 60))
    ref = oracle_lib.tree2d(x, 4, 3)
    xt = torch.from_numpy(x).to(cuda)
    for (a, b) in [(0, 1), (5, 40), (74, 75), (30, 75)]:
        for kernel in KERNELS:
            out = torch.empty((b - a, 53, 16, 8), dtype=torch.complex128, device=cuda)
            forward_into(xt, 4, 3, out, prec=_lib.PREC_FP64, p0_begin=a, p0_end=b, kernel=kernel)
            assert bits_equal(out.cpu().numpy(), ref[a:b])


def test_wrapper_contract(cuda, golden):
    meta, _ = golden
    x = np.random.default_rng(1).standard_normal((20, 17))
    with pytest.raises(ShapeError):
        tree_swdft_2d(x[0], WindowSpec((1, 1)))
    with pytest.raises(WindowTooLargeError):
        tree_swdft_2d(x, WindowSpec((5, 1)))
    with pytest.raises(ValueError):
        tree_swdft_2d(x, WindowSpec((1, 1)), loop_order="bogus")
    with pytest.raises(BudgetError):
        tree_swdft_2d(np.ones((8, 8)), WindowSpec((1, 1)), budget=10)
    # OpCounter replay equals the reference's counts, both loop orders
    for rec in meta["opcount"]:
        xx = np.random.default_rng(rec["N0"] * 100 + rec["N1"]).standard_normal((rec["N0"], rec["N1"]))
        for order in ("levels-outer", "trees-outer"):
            c = OpCounter((rec["N0"], rec["N1"]))
            r = tree_swdft_2d(xx, WindowSpec((rec["m0"], rec["m1"])), loop_order=order, counter=c)
            assert c.total == rec[order]["total"]
            assert sha(c.position_ops) == rec[order]["pos_sha"]
            assert r.values.is_cuda
    # both loop orders give identical output
    a = tree_swdft_2d(x, WindowSpec((2, 2)), loop_order="levels-outer").values
    b = tree_swdft_2d(x, WindowSpec((2, 2)), loop_order="trees-outer").values
    assert torch.equal(a, b)


def test_linearity_and_transpose(cuda):
    """SPEC.md:350-351 properties on the device path (fp64)."""
    rng = np.random.default_rng(2)
    x = rng.standard_normal((24, 20)) + 1j * rng.standard_normal((24, 20))
    y = rng.standard_normal((24, 20)) + 1j * rng.standard_normal((24, 20))
    a, b = 0.7 - 0.2j, -1.3 + 0.5j
    lhs = run(a * x + b * y, 3, 2, "fp64")
    rhs = a * run(x, 3, 2, "fp64") + b * run(y, 3, 2, "fp64")
    assert np.abs(lhs - rhs).max() <= 1e-10 * max(1, np.abs(rhs).max())
    xt = run(np.ascontiguousarray(x.T), 2, 3, "fp64")
    assert np.abs(xt - run(x, 3, 2, "fp64").transpose(1, 0, 3, 2)).max() <= 1e-10


@pytest.mark.parametrize("world", [2, 3, 8])
def test_strip_partition_on_device(cuda, world):
    """Each rank's strip (window rows + n0-1 halo rows, swdft2d_strip_range) computed
    alone on the device reproduces its rows of the full output bitwise (fp64)."""
    from paper_1707_08213_b200.partition import strip_plan

    rng = np.random.default_rng(world)
    x = rng.standard_normal((75, 41))
    m0, m1 = 3, 2
    xt = torch.from_numpy(x).to(cuda)
    P0, P1 = 75 - 7, 41 - 3
    full = torch.empty((P0, P1, 8, 4), dtype=torch.complex128, device=cuda)
    forward_into(xt, m0, m1, full, prec=_lib.PREC_FP64)
    for (a, b, rb, re) in strip_plan(P0, m0, world):
        part = torch.empty((b - a, P1, 8, 4), dtype=torch.complex128, device=cuda)
        if b > a:
            forward_into(xt[rb:re].clone(), m0, m1, part, prec=_lib.PREC_FP64)
        assert torch.equal(part.view(torch.float64), full[a:b].view(torch.float64))


@pytest.mark.gpu
@pytest.mark.parametrize("split", [(2, 2), (1, 4), (4, 2), (1, 8), (3, 1)])
def test_block_partition_on_device(cuda, split):
    """Each rank's 2-D block (window rows x window columns + n0-1 halo rows and n1-1 halo
    columns, partition.block_plan) computed alone — from a strided view of x, as the
    source rank does, and from a packed copy, as a receiver does — reproduces its block
    of the full output bitwise (fp64); the blocks tile the output exactly."""
    from paper_1707_08213_b200.partition import block_plan

    rng = np.random.default_rng(sum(split))
    x = rng.standard_normal((75, 83))
    m0, m1 = 3, 2
    xt = torch.from_numpy(x).to(cuda)
    P0, P1 = 75 - 7, 83 - 3
    full = torch.empty((P0, P1, 8, 4), dtype=torch.complex128, device=cuda)
    forward_into(xt, m0, m1, full, prec=_lib.PREC_FP64)
    covered = np.zeros((P0, P1), dtype=int)
    for (a, b, c0, c1, rb, re, cb, ce) in block_plan(P0, P1, m0, m1, *split):
        covered[a:b, c0:c1] += 1
        if b <= a or c1 <= c0:
            continue
        assert (re - rb, ce - cb) == (b - a + 7, c1 - c0 + 3)
        for src in (xt[rb:re, cb:ce], xt[rb:re, cb:ce].clone()):
            part = torch.empty((b - a, c1 - c0, 8, 4), dtype=torch.complex128, device=cuda)
            forward_into(src, m0, m1, part, prec=_lib.PREC_FP64)
            assert torch.equal(part.view(torch.float64), full[a:b, c0:c1].view(torch.float64))
    assert (covered == 1).all()


@pytest.mark.gpu
def test_tune_split_measures_every_factorisation(cuda):
    """partition.tune_split times the largest block of every gr x gc factorisation and
    returns the lowest modelled step time."""
    from paper_1707_08213_b200.partition import split_candidates, tune_split

    x = torch.from_numpy(np.random.default_rng(3).standard_normal((300, 260))
                         .astype(np.float32)).to(cuda)
    res = tune_split(x, 4, 3, _lib.PREC_FP32, 4)
    assert [tuple(r["split"]) for r in res["table"]] == split_candidates(4)
    best = min(res["table"], key=lambda r: r["score_s"])
    assert tuple(res["split"]) == tuple(best["split"]) and res["pieces"] in (1, 2)
    assert all(r["compute_s"] > 0 and r["scatter_s"] > 0 for r in res["table"])


@pytest.mark.gpu
@pytest.mark.parametrize("slots,dtype", [(1, np.float64), (3, np.float64), (8, np.float32),
                                         (4, np.complex128)])
def test_forward_multi_slots(cuda, oracle_lib, slots, dtype):
    """swdft2d_forward_multi / tree_swdft_2d(devices=[...]): every device slot's shard
    equals its rows of the single-device output bitwise (fp64) and, for fp32, of the
    same K1 run; the union covers [0, P0) in order.  One GPU box: all slots on cuda:0
    (the strip copy is then a device-local cudaMemcpy2DAsync, the same call)."""
    from paper_1707_08213_b200 import OpCounter

    rng = np.random.default_rng(slots)
    x = rng.standard_normal((67, 45))
    if dtype is np.complex128:
        x = x + 1j * rng.standard_normal((67, 45))
    x = x.astype(dtype)
    spec = WindowSpec((3, 2), "unitary")
    xt = torch.from_numpy(x).to(cuda)
    # a strided row view exercises ld_x > N1 in the strip copies
    wide = torch.zeros((67, 53), dtype=xt.dtype, device=cuda)
    wide[:, :45] = xt
    full = tree_swdft_2d(xt, spec, budget=1 << 40).values
    c1, c2 = OpCounter((67, 45)), OpCounter((67, 45))
    shards = tree_swdft_2d(wide[:, :45], spec, budget=1 << 40, devices=[0] * slots, counter=c1)
    tree_swdft_2d(x, spec, budget=1 << 40, counter=c2)
    assert c1.total == c2.total
    torch.cuda.synchronize()
    assert len(shards) == slots
    assert shards[0].p0_begin == 0 and shards[-1].p0_end == full.shape[0]
    for g, sh in enumerate(shards):
        if g:
            assert sh.p0_begin == shards[g - 1].p0_end
        fl = torch.float64 if full.dtype == torch.complex128 else torch.float32
        assert torch.equal(sh.values.view(fl), full[sh.p0_begin:sh.p0_end].view(fl))
    if dtype is not np.float32:
        from paper_1707_08213_b200.core import normalization_factor

        ref = oracle_lib.tree2d(x, 3, 2, scale=normalization_factor(spec))
        got = torch.cat([sh.values for sh in shards]).cpu().numpy()
        assert np.array_equal(got.view(np.float64), ref.view(np.float64))


@pytest.mark.gpu
def test_forward_multi_errors(cuda):
    """Missing stage/out buffers and bad arguments fail loudly with the ABI's codes."""
    import ctypes

    lib = _lib.load()
    xt = torch.zeros((16, 16), dtype=torch.float32, device=cuda)
    out = torch.empty((5, 5, 4, 4), dtype=torch.complex64, device=cuda)
    s = torch.cuda.current_stream(cuda).cuda_stream
    vp = ctypes.c_void_p
    devs = (ctypes.c_int * 2)(0, 0)
    rc = lib.swdft2d_forward_multi(xt.data_ptr(), 0, 16, 16, 16, 2, 2, 0, 1.0, 2, devs,
                                   (vp * 2)(None, None), (vp * 2)(out.data_ptr(), None),
                                   (vp * 2)(s, s))
    assert rc == _lib.E_INVALID_ARG and b"stage" in lib.swdft2d_last_error()
    rc = lib.swdft2d_forward_multi(xt.data_ptr(), 0, 16, 16, 16, 2, 2, 0, 1.0, 0, devs,
                                   None, None, None)
    assert rc == _lib.E_INVALID_ARG
    rc = lib.swdft2d_forward_multi(xt.data_ptr(), 0, 16, 16, 16, 5, 2, 0, 1.0, 1, devs,
                                   None, (vp * 1)(out.data_ptr()), (vp * 1)(s))
    assert rc == _lib.E_WINDOW_TOO_LARGE
    torch.cuda.synchronize()


def test_sharded_api_world1(cuda):
    """tree_swdft_2d_sharded through a real NCCL process group of size 1 equals tree_swdft_2d."""
    import os
    import socket

    import torch.distributed as dist

    from paper_1707_08213_b200.partition import tree_swdft_2d_sharded

    with socket.socket() as sck:
        sck.bind(("127.0.0.1", 0))
        port = sck.getsockname()[1]
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=cuda)
    try:
        x = torch.from_numpy(np.random.default_rng(8).standard_normal((60, 50))).to(cuda)
        sh = tree_swdft_2d_sharded(x, WindowSpec((3, 2), "unitary"), precision="fp64")
        ref = tree_swdft_2d(x, WindowSpec((3, 2), "unitary"), precision="fp64").values
        assert (sh.p0_begin, sh.p0_end, sh.p1_begin, sh.p1_end) == (0, 53, 0, 47)
        assert torch.equal(sh.values.view(torch.float64), ref.view(torch.float64))
        for split in ("strips", (1, 1)):
            sh = tree_swdft_2d_sharded(x, WindowSpec((3, 2), "unitary"), precision="fp64",
                                       split=split, pieces=2)
            assert torch.equal(sh.values.view(torch.float64), ref.view(torch.float64))
    finally:
        dist.destroy_process_group()


def test_large_windows_k0_and_unsupported(cuda, oracle_lib):
    """Windows above K1's 2^6 run on the large-window path and on K0 (both bitwise);
    above 2^10 the ABI refuses loudly."""
    from paper_1707_08213_b200 import UnsupportedError

    rng = np.random.default_rng(12)
    x = rng.standard_normal((140, 12)) + 1j * rng.standard_normal((140, 12))
    ref = oracle_lib.tree2d(x, 7, 2)
    assert bits_equal(run(x, 7, 2, "fp64"), ref)                   # auto -> KR + KC (m0 = 7)
    assert bits_equal(run(x, 7, 2, "fp64", kernel="window"), ref)  # K0
    assert rel_err(run(x.astype(np.complex64), 7, 2, "fp32"), ref) <= FP32_TOL
    with pytest.raises(UnsupportedError):
        run(x, 7, 2, "fp64", kernel="stream")                     # K1 not instantiated
    y = np.zeros((2048, 2))
    with pytest.raises(UnsupportedError):
        run(y, 11, 0, "fp64")                                     # beyond K0's 2^10


@pytest.mark.parametrize("m1", list(range(0, 11)))
def test_row_kernel_windows(cuda, oracle_lib, m1):
    """KR (n0 = 1 windows, n1 = 1 .. 1024): bitwise vs the oracle in fp64 on a strided
    complex input with a ragged last tile, equal to K1 bitwise where K1 exists (n1 <= 64),
    window-row ranges, fp32 within tolerance, unitary scale fused."""
    rng = np.random.default_rng(100 + m1)
    n1 = 1 << m1
    N0, N1 = 3, n1 + 37 + (m1 * 13) % 29
    x = rng.standard_normal((N0, N1)) + 1j * rng.standard_normal((N0, N1))
    ref = oracle_lib.tree2d(x, 0, m1)
    got = run(x, 0, m1, "fp64")                               # auto -> KR
    assert bits_equal(got, ref)
    assert bits_equal(run(x, 0, m1, "fp64", kernel="rows"), ref)
    if m1 <= 6:
        assert bits_equal(run(x, 0, m1, "fp64", kernel="stream"), ref)
    assert rel_err(run(x.astype(np.complex64), 0, m1, "fp32"), ref) <= FP32_TOL
    # strided rows (ld_x > N1) and a window-row range, through the ABI directly
    wide = torch.zeros((N0, N1 + 5), dtype=torch.complex128, device=cuda)
    wide[:, :N1] = torch.from_numpy(x).to(cuda)
    P1 = N1 - n1 + 1
    part = torch.empty((2, P1, 1, n1), dtype=torch.complex128, device=cuda)
    forward_into(wide[:, :N1], 0, m1, part, prec=_lib.PREC_FP64, p0_begin=1, p0_end=3,
                 kernel="rows")
    assert bits_equal(part.cpu().numpy(), ref[1:3])
    from paper_1707_08213_b200.core import normalization_factor

    spec = WindowSpec((0, m1), "unitary")
    refu = oracle_lib.tree2d(x, 0, m1, scale=normalization_factor(spec))
    assert bits_equal(run(x, 0, m1, "fp64", normalization="unitary"), refu)


@pytest.mark.parametrize("m,rows", [((6, 7), 41), ((3, 7), 80), ((7, 6), 40), ((8, 4), 48),
                                    ((2, 8), 40)])
def test_large_windows_column_trees_on_k1(cuda, oracle_lib, m, rows):
    """Windows of the large-window path with enough window rows that the column trees run
    on K1's Z-column kernel by the library's rule (abi.cu use_k1_columns): bitwise vs the
    oracle in fp64 (where the fp64 kernel exists), fp32 in tolerance, and a window-row
    sub-range (a strip starting mid-array)."""
    m0, m1 = m
    n0, n1 = 1 << m0, 1 << m1
    rng = np.random.default_rng(3 * m0 + m1)
    N0, N1 = n0 - 1 + rows, n1 + 19
    x = rng.standard_normal((N0, N1)) + 1j * rng.standard_normal((N0, N1))
    ref = oracle_lib.tree2d(x, m0, m1, threads=8)
    got = run(x, m0, m1, "fp64")
    assert bits_equal(got, ref)
    assert rel_err(run(x.astype(np.complex64), m0, m1, "fp32"), ref) <= FP32_TOL
    xt = torch.from_numpy(x).to(cuda)
    a, b = 3, rows
    part = torch.empty((b - a, N1 - n1 + 1, n0, n1), dtype=torch.complex128, device=cuda)
    forward_into(xt, m0, m1, part, prec=_lib.PREC_FP64, p0_begin=a, p0_end=b)
    assert bits_equal(part.cpu().numpy(), ref[a:b])


@pytest.mark.parametrize("m", [(7, 2), (2, 7), (7, 7), (1, 8), (8, 1), (10, 3), (3, 10), (6, 9),
                               (3, 3), (4, 4), (1, 1), (5, 0)])
def test_separable_large_windows(cuda, oracle_lib, m):
    """KR + KC (the large-window path, also forced on small windows): bitwise vs the
    oracle in fp64 with unitary scale, strided rows, window-row ranges; fp32 in tolerance."""
    from paper_1707_08213_b200.core import normalization_factor

    m0, m1 = m
    n0, n1 = 1 << m0, 1 << m1
    rng = np.random.default_rng(7 * m0 + m1)
    N0, N1 = n0 + 5 + (m0 * 7) % 11, n1 + 9 + (m1 * 5) % 13
    x = rng.standard_normal((N0, N1)) + 1j * rng.standard_normal((N0, N1))
    spec = WindowSpec(m, "unitary")
    ref = oracle_lib.tree2d(x, m0, m1, scale=normalization_factor(spec))
    kern = "auto" if max(m) > 6 else "separable"
    got = run(x, m0, m1, "fp64", kernel=kern, normalization="unitary")
    assert bits_equal(got, ref)
    assert rel_err(run(x.astype(np.complex64), m0, m1, "fp32", kernel=kern,
                       normalization="unitary"), ref) <= FP32_TOL
    wide = torch.zeros((N0, N1 + 3), dtype=torch.complex128, device=cuda)
    wide[:, :N1] = torch.from_numpy(x).to(cuda)
    P0, P1 = N0 - n0 + 1, N1 - n1 + 1
    a, b = min(2, P0 - 1), P0
    part = torch.empty((b - a, P1, n0, n1), dtype=torch.complex128, device=cuda)
    forward_into(wide[:, :N1], m0, m1, part, prec=_lib.PREC_FP64, p0_begin=a, p0_end=b,
                 kernel="separable", scale=normalization_factor(spec))
    assert bits_equal(part.cpu().numpy(), ref[a:b])


def test_row_kernel_1d_large_and_errors(cuda, oracle_lib):
    """tree_swdft_1d with windows up to 1024 runs on KR (bitwise); kernel="rows" with
    n0 > 1 fails loudly."""
    from paper_1707_08213_b200 import UnsupportedError
    from paper_1707_08213_b200.tree1d import tree_swdft_1d

    rng = np.random.default_rng(21)
    s = rng.standard_normal(3000)
    for m in (7, 9, 10):
        ref = oracle_lib.tree2d(s.reshape(1, -1), 0, m)[0, :, 0, :]
        got = tree_swdft_1d(s, WindowSpec((m,))).values.cpu().numpy()
        assert bits_equal(got, ref)
    with pytest.raises(UnsupportedError):
        run(rng.standard_normal((10, 10)), 1, 2, "fp64", kernel="rows")


def test_host_output_pipeline(cuda, oracle_lib):
    """to_host / host_out (one swdft2d_forward_host call): strips computed in a device ring
    and streamed to host memory equal the oracle bit for bit (fp64), with many strips."""
    rng = np.random.default_rng(13)
    x = rng.standard_normal((70, 50)) + 1j * rng.standard_normal((70, 50))
    ref = oracle_lib.tree2d(x, 3, 2)
    res = tree_swdft_2d(x, WindowSpec((3, 2)), precision="fp64", to_host=True,
                        strip_bytes=3 * 47 * 32 * 16)  # 3 window rows per strip -> 21 strips
    assert isinstance(res.values, np.ndarray)
    assert bits_equal(res.values, ref)
    host = torch.empty((63, 47, 8, 4), dtype=torch.complex64, pin_memory=True)
    res32 = tree_swdft_2d(x.astype(np.complex64), WindowSpec((3, 2)), host_out=host,
                          strip_bytes=1 << 12)
    assert res32.values.base is not None or res32.values.ctypes.data == host.data_ptr()
    assert rel_err(res32.values, ref) <= FP32_TOL
    # a caller's numpy array (pageable), a device-resident input, a normalization
    mine = np.full((63, 47, 8, 4), np.nan, dtype=np.complex128)
    xd = torch.from_numpy(x).to(cuda)
    res = tree_swdft_2d(xd, WindowSpec((3, 2), "unitary"), host_out=mine, strip_bytes=5 * 47 * 32 * 16)
    assert res.values is mine and res.normalization == "unitary"
    assert bits_equal(mine, oracle_lib.tree2d(x, 3, 2, scale=1 / np.sqrt(32)))
    with pytest.raises(ValueError):
        tree_swdft_2d(x, WindowSpec((3, 2)), host_out=np.empty((63, 47, 8, 4), np.complex64))
    with pytest.raises(ValueError):
        tree_swdft_2d(x, WindowSpec((3, 2)), host_out=np.empty((63, 47, 4, 8), np.complex128))


@pytest.mark.parametrize("m0", list(range(0, 7)))
def test_every_k1_window_fp64_bitwise_fp32_tol(cuda, oracle_lib, m0):
    """Every window n0 x n1 with n0, n1 in 1..64 (all 49 K1 instantiations per
    precision): fp64 bitwise vs the oracle, fp32 within tolerance, ragged extents."""
    rng = np.random.default_rng(500 + m0)
    for m1 in range(0, 7):
        n0, n1 = 1 << m0, 1 << m1
        N0, N1 = n0 + 3 + (m1 * 5) % 7, n1 + 2 + (m0 * 3) % 5
        x = rng.standard_normal((N0, N1)) + 1j * rng.standard_normal((N0, N1))
        ref = oracle_lib.tree2d(x, m0, m1)
        kern = "stream" if m0 > 0 else "rows"
        assert bits_equal(run(x, m0, m1, "fp64", kernel=kern), ref), (m0, m1)
        assert rel_err(run(x.astype(np.complex64), m0, m1, "fp32", kernel=kern), ref) <= FP32_TOL


@pytest.mark.parametrize("m,extra", [((9, 2), 40), ((7, 3), 50), ((10, 1), 20)])
def test_separable_deep_tiles_many_rows(cuda, oracle_lib, m, extra):
    """KC's deep tile rule (short output runs: n1 x element <= 512 B) with more window rows
    than one tile holds (TP0 = 16, a partial last tile), including the 227 KB tiles of
    n0 >= 512 windows: bitwise vs the oracle in fp64, fp32 in tolerance."""
    m0, m1 = m
    n0, n1 = 1 << m0, 1 << m1
    rng = np.random.default_rng(100 + m0)
    N0, N1 = n0 + extra, n1 + 37
    x = rng.standard_normal((N0, N1))
    ref = oracle_lib.tree2d(x, m0, m1)
    assert bits_equal(run(x, m0, m1, "fp64"), ref)
    assert rel_err(run(x.astype(np.float32), m0, m1, "fp32"), ref) <= FP32_TOL


@pytest.mark.parametrize("m0,m1", [(7, 0), (7, 1), (7, 2), (7, 3), (7, 4), (7, 5), (8, 0), (8, 1),
                                   (8, 2), (9, 0), (9, 1)])
def test_k1_128_row_windows(cuda, oracle_lib, m0, m1):
    """K1's 128-row windows (m0 = 7, n1 <= 16, fp32 only; 128-entry twiddle table read at
    stride for every smaller window): within BASELINE's tolerance of the oracle, through
    the stream kernel explicitly and through auto; fp64 of the same window takes the
    separable path and stays bitwise."""
    n0, n1 = 1 << m0, 1 << m1
    rng = np.random.default_rng(100 * m0 + m1)
    N0, N1 = n0 + 37, n1 + 45
    x = rng.standard_normal((N0, N1))
    ref = oracle_lib.tree2d(x, m0, m1)
    assert _lib.stream_kernel_info(m0, m1, 0)["Q"] == m0 - 4
    assert rel_err(run(x.astype(np.float32), m0, m1, "fp32", kernel="stream"), ref) <= FP32_TOL
    assert rel_err(run(x.astype(np.float32), m0, m1, "fp32"), ref) <= FP32_TOL
    assert bits_equal(run(x, m0, m1, "fp64"), ref)


def test_first_call_inside_graph_capture(cuda):
    """A fresh process whose FIRST library call is captured into a CUDA graph: the one-time
    setup (device state, twiddle tables, kernel attributes, module loading) must not
    invalidate the capture, and the replay equals a plain call."""
    import subprocess
    import sys

    from conftest import ROOT

    r = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "first_capture_check.py")],
                       capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert "first-call capture ok True" in r.stdout, r.stdout + r.stderr


@pytest.mark.gpu
@pytest.mark.parametrize("split,rank,pieces", [((2, 2), 3, 2), ((4, 1), 2, 3), ((1, 3), 1, 2)])
def test_pipelined_block_receive_on_device(cuda, monkeypatch, split, rank, pieces):
    """The receiver side of partition.pipelined_block_forward on the GPU, with the NCCL
    point-to-point layer replaced by copies on a 'link' stream that deliver each piece
    late (a device sleep first): the pieces' K1 launches alternate between the current
    stream and the side stream, each waits for its own piece only, and the rank's block
    equals its block of the single-device output bitwise (fp64)."""
    from paper_1707_08213_b200 import partition

    rng = np.random.default_rng(rank)
    x = torch.from_numpy(rng.standard_normal((90, 77))).to(cuda)
    m0, m1 = 3, 2
    n0, n1 = 8, 4
    P0, P1 = 90 - 7, 77 - 3
    full = torch.empty((P0, P1, n0, n1), dtype=torch.complex128, device=cuda)
    forward_into(x, m0, m1, full, prec=_lib.PREC_FP64)
    a, b, c0, c1, rb, re, cb, ce = partition.block_plan(P0, P1, m0, m1, *split)[rank]
    link = torch.cuda.Stream(cuda)
    sent = x[rb:re, cb:ce].contiguous()

    class Op:
        def __init__(self, fn, tensor, peer, group=None):
            self.fn, self.tensor, self.peer = fn, tensor, peer

    class Work:
        def __init__(self, ev):
            self.ev = ev

        def wait(self):
            torch.cuda.current_stream(cuda).wait_event(self.ev)

    def fake_batch(ops):
        works = []
        for op in ops:
            assert op.fn is partition.dist.irecv and op.peer == 0
            row0 = (op.tensor.data_ptr() - local_base[0]) // (op.tensor.stride(0) * 8)
            link.wait_stream(torch.cuda.current_stream(cuda))
            with torch.cuda.stream(link):
                torch.cuda._sleep(200000)  # the piece arrives late
                op.tensor.copy_(sent[row0:row0 + op.tensor.shape[0]])
                ev = torch.cuda.Event()
                ev.record(link)
            works.append(Work(ev))
        return works

    recv = torch.full((re - rb, ce - cb), float("nan"), dtype=torch.float64, device=cuda)
    local_base = [recv.data_ptr()]
    monkeypatch.setattr(partition.dist, "get_rank", lambda group=None: rank)
    monkeypatch.setattr(partition.dist, "get_world_size", lambda group=None: split[0] * split[1])
    monkeypatch.setattr(partition.dist, "P2POp", Op)
    monkeypatch.setattr(partition.dist, "batch_isend_irecv", fake_batch)
    out = torch.full((b - a, c1 - c0, n0, n1), float("nan"), dtype=torch.complex128, device=cuda)
    streams = set()

    def compute(local, w0, w1):
        streams.add(torch.cuda.current_stream(cuda).cuda_stream)
        forward_into(local, m0, m1, out[w0:w1], prec=_lib.PREC_FP64, p0_begin=w0, p0_end=w1)

    partition.pipelined_block_forward(None, (90, 77), m0, m1, split, torch.float64, cuda,
                                      compute, recv=recv, pieces=pieces)
    torch.cuda.synchronize()
    assert len(streams) == (2 if min(pieces, b - a) > 1 else 1)
    assert torch.equal(out.view(torch.float64), full[a:b, c0:c1].contiguous().view(torch.float64))
