"""Host-side logic: the reference-interface mirror, the C ABI's non-device entry
points, budget/op-count accounting and the strip partition.  CPU only (the
library is loaded but no device function is called)."""
import ctypes
import os
import re

import numpy as np
import pytest

from conftest import ROOT, sha
from paper_1707_08213_b200 import (BudgetError, CoefficientArray, InvalidWindowError, OpCounter,
                                   ShapeError, WindowSpec, WindowTooLargeError, core,
                                   tree_swdft_2d)
from paper_1707_08213_b200 import _lib
from paper_1707_08213_b200.partition import strip_plan, strip_plan_py
from paper_1707_08213_b200.tree2d import replay_counter


def header_functions():
    with open(os.path.join(ROOT, "include", "swdft2d.h")) as f:
        src = f.read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+\s*\*?\s*(swdft2d_\w+)\s*\(", src, re.M)))


def test_library_loads_and_exports_every_header_symbol():
    lib = _lib.load()
    names = header_functions()
    assert len(names) >= 9
    for n in names:
        assert hasattr(lib, n), n
        assert n in _lib.SIGNATURES, n
    assert lib.swdft2d_abi_version() == _lib.ABI_VERSION
    # nothing but the C ABI is exported (static cudart stays private)
    import subprocess

    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True,
                         text=True).stdout
    exported = {l.split()[-1] for l in out.splitlines() if l.strip()}
    assert exported == set(names)


def test_abi_twiddles_bitwise(golden):
    meta, _ = golden
    for n, h in meta["twiddles"].items():
        assert sha(_lib.twiddles(int(n))) == h
    with pytest.raises(InvalidWindowError):
        _lib.twiddles(6)


def test_abi_output_shape_and_bytes(golden):
    meta, _ = golden
    lib = _lib.load()
    P0, P1 = ctypes.c_int64(), ctypes.c_int64()
    assert lib.swdft2d_output_shape(4096, 4096, 4, 4, ctypes.byref(P0), ctypes.byref(P1)) == 0
    assert (P0.value, P1.value) == (4081, 4081)
    rc = lib.swdft2d_output_shape(10, 4096, 4, 4, ctypes.byref(P0), ctypes.byref(P1))
    assert rc == _lib.E_WINDOW_TOO_LARGE
    with pytest.raises(WindowTooLargeError):
        _lib.check(rc)
    lat, out = ctypes.c_int64(), ctypes.c_int64()
    assert lib.swdft2d_reference_bytes(431, 431, 5, 5, ctypes.byref(lat), ctypes.byref(out)) == 0
    assert out.value == meta["budget"]["paper_output_bytes"] == 2621440000  # SPEC acceptance 5
    assert lat.value == meta["budget"]["paper_lattice_bytes"]
    spec = WindowSpec.from_sizes((32, 32))
    assert core.output_bytes((431, 431), spec) == 2621440000
    assert core.lattice_bytes((431, 431), spec) == lat.value


def test_forward_argument_errors_without_device():
    lib = _lib.load()
    # invalid codes are rejected before any CUDA call
    assert lib.swdft2d_forward(None, 9, 8, 8, 8, 1, 1, 0, 1.0, 0, 7, None, 0, None) == _lib.E_INVALID_ARG
    assert lib.swdft2d_forward(None, 0, 8, 8, 8, 1, 1, 5, 1.0, 0, 7, None, 0, None) == _lib.E_INVALID_ARG
    assert lib.swdft2d_forward(None, 0, 8, 8, 4, 1, 1, 0, 1.0, 0, 7, None, 0, None) == _lib.E_INVALID_ARG
    assert lib.swdft2d_forward(None, 0, 8, 8, 8, 4, 1, 0, 1.0, 0, 7, None, 0, None) == _lib.E_WINDOW_TOO_LARGE
    assert lib.swdft2d_forward(None, 0, 8, 8, 8, 1, 1, 0, 1.0, 0, 9, None, 0, None) == _lib.E_INVALID_ARG
    assert "outside" in _lib.last_error()
    assert lib.swdft2d_forward(None, 0, 0, 8, 8, 1, 1, 0, 1.0, 0, 0, None, 0, None) == _lib.E_SHAPE


def test_window_spec_mirror():
    s = WindowSpec.from_sizes((16, 8))
    assert s.exponents == (4, 3) and s.sizes == (16, 8) and s.window_elements == 128
    with pytest.raises(InvalidWindowError):
        WindowSpec.from_sizes((12, 8))
    with pytest.raises(InvalidWindowError):
        WindowSpec((1, 1), "paper-1d")
    with pytest.raises(InvalidWindowError):
        WindowSpec((-1, 1))
    with pytest.raises(WindowTooLargeError):
        s.check_fits((8, 8))
    with pytest.raises(ShapeError):
        s.check_fits((8,))
    assert core.normalization_factor(WindowSpec((2, 2), "unitary")) == 0.25
    assert core.normalization_factor(WindowSpec((2, 2), "paper-2d")) == 0.25
    assert core.normalization_factor(WindowSpec((2, 2))) == 1.0


def test_coefficient_array_checks():
    spec = WindowSpec((1, 2))
    v = np.zeros((5, 4, 2, 4), dtype=np.complex64)
    c = CoefficientArray(v, (6, 7), spec)
    assert c.positions == (5, 4)
    with pytest.raises(ShapeError):
        CoefficientArray(v[:, :3], (6, 7), spec)
    with pytest.raises(ShapeError):
        CoefficientArray(v[0], (6, 7), spec)


def test_wrapper_validation_order(golden):
    """tree2d.py:189-196 order: 2D check, check_fits, loop_order, budget — all before
    anything touches the device (so this runs on CPU)."""
    meta, _ = golden
    x = np.zeros((8, 8))
    with pytest.raises(ShapeError, match="2D array and 2D window"):
        tree_swdft_2d(np.zeros(8), WindowSpec((1, 1)))
    with pytest.raises(ShapeError):
        tree_swdft_2d(x, WindowSpec((1,)))
    with pytest.raises(WindowTooLargeError):
        tree_swdft_2d(x, WindowSpec((4, 1)))
    with pytest.raises(ValueError, match="loop_order"):
        tree_swdft_2d(x, WindowSpec((1, 1)), loop_order="rows-first")
    with pytest.raises(BudgetError) as ei:
        tree_swdft_2d(np.ones((8, 8)), WindowSpec((1, 1)), budget=10)
    ref = meta["budget"]["error"]
    assert ei.value.required_bytes == ref["required"] and ei.value.budget_bytes == ref["budget"]
    assert str(ei.value) == ref["msg"]
    # default budget (4 GiB) rejects config 4 exactly as the reference does
    with pytest.raises(BudgetError):
        tree_swdft_2d(np.zeros((4096, 4096), np.float32), WindowSpec((4, 4)))
    with pytest.raises(WindowTooLargeError):  # empty / ragged extents: check_fits (core.py:116)
        tree_swdft_2d(np.zeros((0, 5)), WindowSpec((0, 0)))
    with pytest.raises(ValueError):  # ragged nested lists are not arrays
        tree_swdft_2d([[1.0, 2.0], [3.0]], WindowSpec((0, 0)))
    with pytest.raises(ValueError):  # np.asarray(x, complex128) fails first (tree2d.py:189)
        tree_swdft_2d(np.array([["a", "b"], ["c", "d"]]), WindowSpec((1, 1)))


def test_opcounter_replay(golden):
    meta, _ = golden
    for rec in meta["opcount"]:
        shape = (rec["N0"], rec["N1"])
        c = OpCounter(shape)
        replay_counter(c, shape, WindowSpec((rec["m0"], rec["m1"])))
        for order in ("levels-outer", "trees-outer"):
            assert c.total == rec[order]["total"] == rec["predict_ops"]
            assert sha(c.position_ops) == rec[order]["pos_sha"]
    for n, ops in meta["ops_per_interior_window"].items():  # Eq. 8: 2(n0 n1 - 1)
        n = int(n)
        c = OpCounter((2 * n, 2 * n))
        replay_counter(c, (2 * n, 2 * n), WindowSpec.from_sizes((n, n)))
        assert c.position_ops[-1, -1] == ops == 2 * (n * n - 1)


@pytest.mark.parametrize("P0,m0,world", [(4081, 4, 1), (4081, 4, 2), (4081, 4, 8), (1985, 6, 8),
                                         (3, 2, 8), (0, 0, 4), (2017, 5, 7)])
def test_strip_plan(P0, m0, world):
    plan = strip_plan(P0, m0, world)
    assert plan == strip_plan_py(P0, m0, world)
    n0 = 1 << m0
    assert plan[0][0] == 0 and plan[-1][1] == P0
    for g in range(world):
        a, b, rb, re = plan[g]
        if g:
            assert a == plan[g - 1][1]
        assert rb == a and (re == b + n0 - 1 if b > a else re == rb)
        assert abs((b - a) - P0 / world) < 1.0 + 1e-9  # imbalance <= 1 row


def _build_c_example(tmpdir):
    """gcc the pure-C ABI example against include/swdft2d.h and libswdft2d.so."""
    import subprocess

    exe = os.path.join(tmpdir, "forward_c")
    cmd = ["gcc", "-O2", "-I", os.path.join(ROOT, "include"), "-I", "/usr/local/cuda/include",
           os.path.join(ROOT, "examples", "forward_c.c"), "-L", os.path.dirname(_lib.LIB_PATH),
           "-lswdft2d", "-L", "/usr/local/cuda/lib64", "-lcudart", "-lm",
           "-Wl,-rpath," + os.path.dirname(_lib.LIB_PATH), "-o", exe]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return exe


def test_c_abi_example_compiles_and_links(tmp_path):
    """A C program (no Python, no torch) builds against the header and the library."""
    assert os.path.exists(_build_c_example(str(tmp_path)))


@pytest.mark.gpu
def test_c_abi_example_runs(tmp_path):
    """The C program computes config-1-like output through the ABI alone, checks it
    against a direct DFT, and sees an invalid call fail with its status code."""
    import subprocess

    r = subprocess.run([_build_c_example(str(tmp_path))], capture_output=True, text=True,
                       timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "max window-relative error" in r.stdout


def test_kernels_keep_their_state_in_registers():
    """ptxas -v of the last build: no hot-path kernel uses a local-memory stack frame
    (a forced call or a dynamically indexed array there once made K1 4.6x slower).
    Known exceptions: the fp64 64x64 K1 (128-register cap at 512 threads), KR/KC's largest
    fp64/fp32 trees (<= 24 B), and K0, the bring-up kernel with per-thread row arrays —
    bounded: its windows above 64 keep a stack of m1 + 1 nodes, not n-entry arrays (a
    32 KB frame per thread made the driver reserve ~9.7 GB of local memory)."""
    from paper_1707_08213_b200 import build

    res = build.kernel_resources()
    if not res:
        pytest.skip("no ptxas logs (library built elsewhere)")
    k1 = {k: v for k, v in res.items() if "k1_stream_kernel" in k}
    assert len(k1) >= 196
    allowed_k1 = ("k1_stream_kernelIdLi6ELi6E",)
    for name, (regs, stack, spill) in res.items():
        if "k0_window_kernel" in name:
            assert stack <= 4096, (name, regs, stack, spill)  # 64-entry arrays at most
            continue
        if "k0_window_large_kernel" in name:
            assert stack <= 512, (name, regs, stack, spill)
            continue
        if "k1_stream_kernel" in name and any(a in name for a in allowed_k1):
            continue
        limit = 0 if ("k1_stream_kernel" in name or "k2_push" in name) else 24
        assert stack <= limit, (name, regs, stack, spill)
