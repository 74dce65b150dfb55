"""The reference's own entry point served by the B200 library (integration/swdft_b200.py).

The UNMODIFIED reference package is staged into the git-ignored baseline/_ref/ by
scripts/stage_reference.sh (run by __graft_entry__.build() where /root/reference
exists; the copy travels to the GPU box with the snapshot).  These tests import
``swdft`` from there, enable the backend, and check the drop-in contract against the
reference's own types, exceptions, counter and golden outputs.
"""
import os
import sys

import numpy as np
import pytest

from conftest import ROOT, sha
from golden_inputs import kat6_input

REF_DIR = os.path.join(ROOT, "baseline", "_ref")
INTEG_DIR = os.path.join(ROOT, "integration")


@pytest.fixture(scope="module")
def swdft():
    if not os.path.isfile(os.path.join(REF_DIR, "swdft", "tree2d.py")):
        pytest.skip("reference package not staged (scripts/stage_reference.sh)")
    for d in (REF_DIR, INTEG_DIR):
        if d not in sys.path:
            sys.path.insert(0, d)
    import swdft.bench
    import swdft.core
    import swdft.tree2d
    import swdft_b200

    orig = swdft.tree2d.tree_swdft_2d
    swdft_b200.enable()
    assert swdft.tree2d.tree_swdft_2d is not orig and swdft_b200.enabled()
    yield swdft
    swdft_b200.disable()
    assert swdft.tree2d.tree_swdft_2d is orig


def test_reference_exceptions_through_backend(swdft):
    """Validation runs before any device work, with the reference's classes and messages."""
    core, tree2d = swdft.core, swdft.tree2d
    spec = core.WindowSpec.from_sizes((4, 4))
    with pytest.raises(core.ShapeError):
        tree2d.tree_swdft_2d(np.zeros((4, 4, 4)), spec)
    with pytest.raises(core.WindowTooLargeError):
        tree2d.tree_swdft_2d(np.zeros((3, 8)), spec)
    with pytest.raises(ValueError, match="loop_order"):
        tree2d.tree_swdft_2d(np.zeros((8, 8)), spec, loop_order="rows-first")
    with pytest.raises(core.BudgetError) as e:
        tree2d.tree_swdft_2d(np.zeros((64, 64)), spec, budget=1000)
    # the same numbers and text the reference's own implementation raises
    import swdft_b200

    with pytest.raises(core.BudgetError) as e_ref:
        swdft_b200._STATE["orig"](np.zeros((64, 64)), spec, budget=1000)
    assert str(e.value) == str(e_ref.value)
    assert e.value.required_bytes == e_ref.value.required_bytes
    with pytest.raises(core.InvalidWindowError):
        core.WindowSpec.from_sizes((3, 4))


@pytest.mark.gpu
def test_reference_entry_point_bitwise(swdft, golden, cuda):
    core, tree2d = swdft.core, swdft.tree2d
    meta, arr = golden
    x = np.array(meta["kat"]["kat1"]["x"])
    r = tree2d.tree_swdft_2d(x, core.WindowSpec.from_sizes((2, 2)))
    assert isinstance(r, core.CoefficientArray)
    assert isinstance(r.values, np.ndarray) and r.values.dtype == np.complex128
    assert np.array_equal(r.values.view(np.uint64), arr["kat1_out"].view(np.uint64))
    r = tree2d.tree_swdft_2d(np.ones((8, 8)), core.WindowSpec.from_sizes((4, 4)))
    assert np.array_equal(r.values.view(np.uint64), arr["kat2_out"].view(np.uint64))
    k6, nx = kat6_input()
    r = tree2d.tree_swdft_2d(k6, core.WindowSpec.from_sizes((2, 4)))
    assert np.array_equal(r.values.view(np.uint64), arr["kat6_out"].view(np.uint64))
    for mode in ("unitary", "paper-2d"):
        spec = core.WindowSpec((2, 1), mode)
        r = tree2d.tree_swdft_2d(nx, spec)
        assert r.normalization == mode
        assert np.array_equal(r.values.view(np.uint64), arr[f"norm_{mode}_out"].view(np.uint64))
        with pytest.raises(core.StateError):  # the record behaves like normalize()'s output
            core.normalize(r, mode)
    from paper_1707_08213_b200.workloads import CONFIGS

    cfg = CONFIGS["c1"]
    r = tree2d.tree_swdft_2d(cfg.generate(), core.WindowSpec((cfg.m0, cfg.m1)))
    assert sha(r.values) == meta["configs"]["c1"]["full_sha"]


@pytest.mark.gpu
def test_reference_entry_point_matches_reference_run(swdft, cuda):
    """Same output bits and the same OpCounter state as the reference's own numpy code
    on the same inputs (both loop orders, a normalization mode, odd shapes)."""
    import swdft_b200

    core, tree2d, bench = swdft.core, swdft.tree2d, swdft.bench
    orig = swdft_b200._STATE["orig"]
    rng = np.random.default_rng(8)
    for shape, sizes, mode in [((37, 29), (4, 8), "none"), ((20, 33), (8, 2), "unitary"),
                               ((16, 16), (16, 1), "paper-2d"), ((9, 40), (1, 32), "none")]:
        x = rng.standard_normal(shape) + 1j * rng.standard_normal(shape)
        spec = core.WindowSpec(tuple(int(s).bit_length() - 1 for s in sizes), mode)
        for order in tree2d.LOOP_ORDERS:
            c_ref, c_b200 = bench.OpCounter(shape), bench.OpCounter(shape)
            ref = orig(x, spec, loop_order=order, counter=c_ref)
            got = tree2d.tree_swdft_2d(x, spec, loop_order=order, counter=c_b200, threads=4)
            assert got.normalization == ref.normalization == mode
            assert got.source_shape == ref.source_shape
            assert np.array_equal(got.values.view(np.uint64), ref.values.view(np.uint64))
            assert c_b200.total == c_ref.total
            assert np.array_equal(c_b200.position_ops, c_ref.position_ops)


@pytest.mark.gpu
def test_reference_entry_point_device_values(swdft, cuda):
    import torch

    import swdft_b200

    core, tree2d = swdft.core, swdft.tree2d
    x = np.random.default_rng(2).standard_normal((70, 90))
    spec = core.WindowSpec.from_sizes((16, 16))
    host = tree2d.tree_swdft_2d(x, spec)
    swdft_b200.enable(values="device")
    try:
        dev = tree2d.tree_swdft_2d(x, spec)
    finally:
        swdft_b200.enable(values="numpy")
    assert isinstance(dev, core.CoefficientArray) and isinstance(dev.values, torch.Tensor)
    assert dev.values.is_cuda and dev.values.dtype == torch.complex128
    assert np.array_equal(dev.values.cpu().numpy().view(np.uint64), host.values.view(np.uint64))


@pytest.mark.gpu
def test_reference_cli_through_backend(swdft, cuda, tmp_path, capsys):
    """The reference's own CLI (cli.py:131-185, unmodified) with the backend enabled: its
    ``transform`` writes a file byte-identical to the one its numpy path writes (window
    2-D, plain and paper-2d), ``verify`` passes (tree bitwise equal to its swfft_2d, within
    1e-10 of naive) and fails with --corrupt, and ``bench`` reports the reference's op
    counts for the tree rows."""
    import swdft.cli

    import swdft_b200

    x = np.random.default_rng(11).standard_normal((24, 30))
    src = tmp_path / "x.csv"
    np.savetxt(src, x, delimiter=",", fmt="%.17g")
    for window, mode in (("8x4", "none"), ("4x16", "paper-2d")):
        outs = {}
        for backend in ("b200", "numpy"):
            if backend == "numpy":
                swdft_b200.disable()
            try:
                o = tmp_path / f"{backend}_{window}_{mode}.swdf"
                assert swdft.cli.main(["transform", "--input", str(src), "--output", str(o),
                                       "--window", window, "--normalization", mode]) == 0
                outs[backend] = o.read_bytes()
            finally:
                swdft_b200.enable()
        assert outs["b200"] == outs["numpy"]
    assert swdft.cli.main(["verify", "--input", str(src), "--window", "8x8"]) == 0
    assert "exact_fft_match=true" in capsys.readouterr().out
    assert swdft.cli.main(["verify", "--input", str(src), "--window", "8x8", "--corrupt"]) == 1
    csv = tmp_path / "bench.csv"
    served = swdft.tree2d.tree_swdft_2d
    calls = []

    def counting(*a, **k):
        calls.append(a[0].shape)
        return served(*a, **k)

    swdft.tree2d.tree_swdft_2d = counting
    try:
        assert swdft.cli.main(["bench", "--size", "40x40", "--windows", "4x4,8x2",
                               "--algorithms", "tree", "--repetitions", "1",
                               "--output", str(csv)]) == 0
    finally:
        swdft.tree2d.tree_swdft_2d = served
    assert calls and all(c == (40, 40) for c in calls)  # the bench timed the backend
    lines = csv.read_text().strip().splitlines()
    head = lines[0].split(",")
    rows = [dict(zip(head, ln.split(","))) for ln in lines[1:]]
    assert len(rows) == 2
    for r in rows:
        assert r["algorithm"] == "tree"
        sizes = (int(r["n0"]), int(r["n1"]))
        assert int(r["ops"]) == swdft.bench.predict_ops("tree", (40, 40), sizes)


@pytest.mark.gpu
def test_reference_1d_kd_entry_points(swdft, cuda, tmp_path):
    """swdft.tree1d.tree_swdft_1d and swdft.treekd.tree_swdft_kd routed to the B200: the
    reference's types, exceptions and counter state, output bits equal to its own numpy
    code; the reference CLI transforms a 3-D SWDF container byte-identically."""
    import swdft.cli
    import swdft.container
    import swdft.tree1d
    import swdft.treekd

    import swdft_b200

    core, bench = swdft.core, swdft.bench
    rng = np.random.default_rng(21)
    o1 = swdft_b200.original("tree1d", "tree_swdft_1d")
    okd = swdft_b200.original("treekd", "tree_swdft_kd")
    for N, n, mode in ((50, 8, "none"), (33, 32, "unitary"), (7, 1, "none")):
        x = rng.standard_normal(N) + 1j * rng.standard_normal(N)
        spec = core.WindowSpec((n.bit_length() - 1,), mode)
        c_ref, c_got = bench.OpCounter((N,)), bench.OpCounter((N,))
        ref = o1(x, spec, counter=c_ref)
        got = swdft.tree1d.tree_swdft_1d(x, spec, counter=c_got)
        assert isinstance(got, core.CoefficientArray) and got.normalization == mode
        assert np.array_equal(got.values.view(np.uint64), ref.values.view(np.uint64))
        assert c_got.total == c_ref.total
        assert np.array_equal(c_got.position_ops, c_ref.position_ops)
    with pytest.raises(core.ShapeError):
        swdft.tree1d.tree_swdft_1d(np.zeros((4, 4)), core.WindowSpec((1,)))
    with pytest.raises(core.WindowTooLargeError):
        swdft.tree1d.tree_swdft_1d(np.zeros(3), core.WindowSpec((2,)))
    for shape, exps in (((9, 8, 10), (2, 1, 2)), ((6, 6, 6), (1, 1, 1)), ((12, 10), (2, 3))):
        x = rng.standard_normal(shape)
        spec = core.WindowSpec(exps)
        c_ref, c_got = bench.OpCounter(shape), bench.OpCounter(shape)
        ref = okd(x, spec, counter=c_ref)
        got = swdft.treekd.tree_swdft_kd(x, spec, counter=c_got)
        assert isinstance(got, core.CoefficientArray) and got.values.shape == ref.values.shape
        assert np.array_equal(got.values.view(np.uint64), ref.values.view(np.uint64))
        assert c_got.total == c_ref.total
    with pytest.raises(core.ShapeError):
        swdft.treekd.tree_swdft_kd(np.zeros((4, 4)), core.WindowSpec((1, 1, 1)))
    with pytest.raises(core.BudgetError) as e:
        swdft.treekd.tree_swdft_kd(np.zeros((8, 8, 8)), core.WindowSpec((1, 1, 1)), budget=100)
    with pytest.raises(core.BudgetError) as e_ref:
        okd(np.zeros((8, 8, 8)), core.WindowSpec((1, 1, 1)), budget=100)
    assert str(e.value) == str(e_ref.value)
    # the reference CLI on a 3-D container: same bytes with and without the backend
    src = tmp_path / "x3.swdf"
    swdft.container.write_swdf(src, rng.standard_normal((7, 9, 8)).astype(np.complex128))
    outs = {}
    for backend in ("b200", "numpy"):
        if backend == "numpy":
            swdft_b200.disable()
        try:
            o = tmp_path / f"{backend}.swdf"
            assert swdft.cli.main(["transform", "--input", str(src), "--output", str(o),
                                   "--window", "4x2x4", "--normalization", "unitary"]) == 0
            outs[backend] = o.read_bytes()
        finally:
            swdft_b200.enable()
    assert outs["b200"] == outs["numpy"]


@pytest.mark.gpu
def test_reference_stream_classes(swdft, cuda):
    """swdft.tree2d.SlidingRowStream2D and swdft.tree1d.SlidingStream1D routed to the B200:
    the reference's exceptions and attributes; 2-D slabs bitwise equal to the rows of the
    reference's own batch transform (its own stream raises for windows above 1x1, App. A
    #11, and is compared where it runs: 1x1); 1-D vectors, per-push ops and counters bitwise
    / exactly equal to the reference's own 1-D stream."""
    import swdft.tree1d

    import swdft_b200

    core, bench, tree2d = swdft.core, swdft.bench, swdft.tree2d
    rng = np.random.default_rng(33)
    batch = swdft_b200.original("tree2d", "tree_swdft_2d")
    for (N0, N1), exps, mode in (((20, 17), (2, 3), "none"), ((12, 9), (3, 0), "unitary"),
                                 ((70, 40), (5, 2), "none")):
        x = rng.standard_normal((N0, N1)) + 1j * rng.standard_normal((N0, N1))
        spec = core.WindowSpec(exps, mode)
        n0, n1 = spec.sizes
        ref = batch(x, spec, budget=1 << 40).values
        cnt = bench.OpCounter((N0, N1))
        st = tree2d.SlidingRowStream2D(spec, N1, counter=cnt)
        assert type(st).__name__ == "SlidingRowStream2D_b200" and st.n0 == n0 and st.N1 == N1
        for r in range(N0):
            slab = st.push_row(x[r])
            assert st.rows_pushed == r + 1
            if r < n0 - 1:
                assert slab is None
            else:
                assert isinstance(slab, np.ndarray) and slab.shape == (N1 - n1 + 1, n0, n1)
                assert np.array_equal(slab.view(np.uint64),
                                      np.ascontiguousarray(ref[r - n0 + 1]).view(np.uint64))
                assert st.last_push_position_ops[-1] == 2 * (n0 * n1 - 1)   # SPEC acceptance 7
        cb = bench.OpCounter((N0, N1))
        batch(x, spec, counter=cb, budget=1 << 40)
        assert cnt.total == cb.total and np.array_equal(cnt.position_ops, cb.position_ops)
        with pytest.raises(core.ShapeError):
            st.push_row(np.zeros(N1 + 1))
        st.close()
        assert st.closed
        with pytest.raises(core.StateError):
            st.push_row(x[0])
    with pytest.raises(core.ShapeError):
        tree2d.SlidingRowStream2D(core.WindowSpec((2,)), 8)
    with pytest.raises(core.WindowTooLargeError):
        tree2d.SlidingRowStream2D(core.WindowSpec((1, 4)), 8)
    # 1x1 windows: the one case the reference's own 2-D stream runs
    RefStream = swdft_b200.original("tree2d", "SlidingRowStream2D")
    spec = core.WindowSpec((0, 0))
    a, b = RefStream(spec, 6), tree2d.SlidingRowStream2D(spec, 6)
    for r in range(4):
        row = rng.standard_normal(6)
        ra, rb = a.push_row(row), b.push_row(row)
        assert np.array_equal(ra.view(np.uint64), rb.view(np.uint64))
        assert a.ops_last_push == b.ops_last_push
    # 1-D stream vs the reference's own
    Ref1 = swdft_b200.original("tree1d", "SlidingStream1D")
    for m, mode in ((3, "none"), (6, "unitary"), (0, "none"), (7, "none")):
        spec = core.WindowSpec((m,), mode)
        ca, cb = bench.OpCounter((200,)), bench.OpCounter((200,))
        a, b = Ref1(spec, counter=ca), swdft.tree1d.SlidingStream1D(spec, counter=cb)
        for p in range(200):
            v = complex(rng.standard_normal(), rng.standard_normal())
            ra, rb = a.push(v), b.push(v)
            assert (ra is None) == (rb is None) and a.ops_last_push == b.ops_last_push
            if ra is not None:
                assert np.array_equal(ra.view(np.uint64), rb.view(np.uint64)), (m, p)
        assert ca.total == cb.total and b.pushed == 200
        b.close()
        with pytest.raises(core.StateError):
            b.push(0.0)


STUB = r"""
import ctypes, os, sys
import numpy as np
sys.path.insert(0, {root!r})
import oracle                                     # the checker (numpy + C, no torch)

lib = ctypes.CDLL({lib!r})
i64, cint, vp = ctypes.c_int64, ctypes.c_int, ctypes.c_void_p
lib.swdft2d_forward_host.argtypes = [vp, cint, i64, i64, i64, cint, cint, cint, ctypes.c_double,
                                     i64, i64, vp, i64, cint, vp]
lib.swdft2d_forward_host.restype = cint
lib.swdft2d_last_error.restype = ctypes.c_char_p
rng = np.random.default_rng(21)
x = np.ascontiguousarray(rng.standard_normal((300, 200)) + 1j * rng.standard_normal((300, 200)))
m0, m1 = 4, 3
out = np.empty((300 - 15, 200 - 7, 16, 8), dtype=np.complex128)
rc = lib.swdft2d_forward_host(x.ctypes.data, 3, 300, 200, 200, m0, m1, 1, 1.0, 0, 285,
                              out.ctypes.data, 1 << 22, 0, None)
assert rc == 0, lib.swdft2d_last_error()
ref = oracle.tree2d(x, m0, m1)
assert np.array_equal(out.view(np.uint64), ref.view(np.uint64))
rc = lib.swdft2d_forward_host(x.ctypes.data, 3, 300, 200, 200, 9, m1, 1, 1.0, 0, 1,
                              out.ctypes.data, 0, 0, None)
assert rc == -3 and b"window" in lib.swdft2d_last_error().lower()   # WindowTooLargeError
assert "torch" not in sys.modules
print("stub ok")
"""


@pytest.mark.gpu
def test_ctypes_stub_needs_no_torch(oracle_lib):
    """INTEGRATION.md's stub as a maintainer would write it: numpy + ctypes only, one
    swdft2d_forward_host call on numpy buffers, in a process that never imports torch
    (the library brings its own CUDA runtime); bitwise equal to the oracle."""
    import subprocess

    from paper_1707_08213_b200 import _lib

    code = STUB.format(root=ROOT, lib=_lib.LIB_PATH)
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and "stub ok" in r.stdout, r.stdout + r.stderr
