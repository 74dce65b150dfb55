"""SURVEY.md 8(f) rows built on the path: row-push stream, SWDF container, on-device
verify + bench CSV, 1D tree.  CPU tests cover the host-only parts; GPU tests go
through libswdft2d.so."""
import hashlib

import numpy as np
import pytest
import torch

from conftest import sha
from paper_1707_08213_b200 import ContainerError, OpCounter, WindowSpec
from paper_1707_08213_b200 import container
from paper_1707_08213_b200.verify import predict_ops


def file_sha(p):
    return hashlib.sha256(open(p, "rb").read()).hexdigest()


# ---------------------------------------------------------------- CPU

def test_container_host_bytes_match_reference(golden, tmp_path, oracle_lib):
    meta, _ = golden
    x = np.random.default_rng(21).standard_normal((12, 9))
    p = tmp_path / "real.swdf"
    container.write_swdf(p, x)
    assert file_sha(p) == meta["next"]["swdf_real_12x9"]
    vals = oracle_lib.tree2d(x, 2, 1, scale=1.0 / np.sqrt(8.0))
    p2 = tmp_path / "c.swdf"
    container.write_swdf(p2, vals, normalization="unitary")
    assert file_sha(p2) == meta["next"]["swdf_unitary_12x9_w4x2"]
    back, mode = container.read_swdf(p2)
    assert mode == "unitary" and np.array_equal(back.view(np.uint64), vals.view(np.uint64))
    assert len(container.header_bytes((2, 3, 4, 5), True, "none")) == 46  # 14 + 8*ndim bytes


def test_container_errors(tmp_path):
    p = tmp_path / "bad.swdf"
    p.write_bytes(b"NOPE" + bytes(20))
    with pytest.raises(ContainerError):
        container.read_swdf(p)
    with pytest.raises(ContainerError):
        container.write_swdf(tmp_path / "x.swdf", np.zeros(3), normalization="bogus")
    good = tmp_path / "g.swdf"
    container.write_swdf(good, np.array([1.0, np.inf]))
    with pytest.raises(ContainerError, match="non-finite"):
        container.read_swdf(good)
    raw = good.read_bytes()
    (tmp_path / "t.swdf").write_bytes(raw[:-3])
    with pytest.raises(ContainerError, match="payload"):
        container.read_swdf(tmp_path / "t.swdf")
    csv = tmp_path / "x.csv"
    csv.write_text("1,2\n3,nan\n")
    with pytest.raises(ContainerError):
        container.read_csv_2d(csv)


def test_bench_predict_ops(golden):
    meta, _ = golden
    for w, d in meta["next"]["fig4_predict_ops"].items():
        for alg, ops in d.items():
            assert predict_ops(alg, (100, 100), (int(w), int(w))) == ops


def test_treekd_counter_replay(golden):
    from paper_1707_08213_b200.treekd import level_regions_kd

    meta, _ = golden
    for rec in meta["next"]["treekd"]:
        c = OpCounter(tuple(rec["shape"]))
        for region, nodes, positions in level_regions_kd(tuple(rec["shape"]), rec["m"]):
            c.add_region(region, nodes, positions)
        assert c.total == rec["total"] and sha(c.position_ops) == rec["pos_sha"]


# ---------------------------------------------------------------- GPU

@pytest.mark.gpu
def test_container_from_device_tensor(golden, cuda, tmp_path):
    from paper_1707_08213_b200 import tree_swdft_2d

    meta, _ = golden
    x = np.random.default_rng(21).standard_normal((12, 9))
    res = tree_swdft_2d(x, WindowSpec((2, 1), "unitary"))
    p = tmp_path / "d.swdf"
    container.write_swdf(p, res.values, normalization=res.normalization, chunk_bytes=256)
    assert file_sha(p) == meta["next"]["swdf_unitary_12x9_w4x2"]
    # complex64 device output is widened to the format's complex128
    res32 = tree_swdft_2d(x.astype(np.float32), WindowSpec((2, 1)))
    container.write_swdf(tmp_path / "f.swdf", res32.values, chunk_bytes=1000)
    back, _ = container.read_swdf(tmp_path / "f.swdf")
    assert np.array_equal(back, res32.values.cpu().numpy().astype(np.complex128))


@pytest.mark.gpu
@pytest.mark.parametrize("kernel", ["auto", "stream"])
@pytest.mark.parametrize("shape,m", [((30, 20), (2, 2)), ((19, 33), (3, 1)), ((12, 12), (0, 3)),
                                     ((70, 130), (6, 6)), ((7, 6), (0, 0)), ((40, 9), (5, 0)),
                                     ((22, 70), (1, 6))])
def test_row_stream_equals_batch(cuda, oracle_lib, shape, m, kernel):
    """kernel "auto": incremental K2 pushes over the level state; "stream": K1 re-run
    over the raw ring per push.  Both bitwise equal to the batch rows (fp64)."""
    from paper_1707_08213_b200.stream import SlidingRowStream2D

    rng = np.random.default_rng(shape[0] * 7 + m[0])
    x = rng.standard_normal(shape) + 1j * rng.standard_normal(shape)
    n0, n1 = 1 << m[0], 1 << m[1]
    ref = oracle_lib.tree2d(x, *m)
    c = OpCounter(shape)
    st = SlidingRowStream2D(WindowSpec(m), shape[1], counter=c, kernel=kernel)
    assert (st._state is not None) == (kernel == "auto")
    for p0 in range(shape[0]):
        slab = st.push_row(x[p0])
        if p0 < n0 - 1:
            assert slab is None
            continue
        got = slab.cpu().numpy()
        assert np.array_equal(got.view(np.uint64), ref[p0 - n0 + 1].view(np.uint64))
        # SPEC.md:342 / acceptance 7: a warmed stream costs 2(n0 n1 - 1) per position
        assert np.all(st.last_push_position_ops[n1 - 1:] == 2 * (n0 * n1 - 1))
    # the pushes' add_region calls sum to the batch transform's
    from paper_1707_08213_b200.tree2d import replay_counter

    cb = OpCounter(shape)
    replay_counter(cb, shape, WindowSpec(m))
    assert c.total == cb.total and np.array_equal(c.position_ops, cb.position_ops)
    st.close()
    from paper_1707_08213_b200 import StateError

    with pytest.raises(StateError):
        st.push_row(x[0])


@pytest.mark.gpu
@pytest.mark.parametrize("pinned", [True, False])
def test_row_stream_reused_host_buffer(cuda, oracle_lib, pinned):
    """The usual streaming pattern: ONE host row buffer refilled before every push, no
    synchronisation by the caller.  push_row reads the caller's buffer before returning
    (an asynchronous H2D straight from it read the next row's data)."""
    import torch

    from paper_1707_08213_b200.stream import SlidingRowStream2D

    shape, m = (300, 2000), (4, 4)
    rng = np.random.default_rng(3)
    x = rng.standard_normal(shape)
    ref = oracle_lib.tree2d(x, *m)
    st = SlidingRowStream2D(WindowSpec(m), shape[1])
    buf = torch.empty(shape[1], dtype=torch.float64, pin_memory=pinned)
    slabs = []
    for p0 in range(shape[0]):
        buf.copy_(torch.from_numpy(x[p0]))
        s = st.push_row(buf)
        if s is not None:
            slabs.append(s)
    got = torch.stack(slabs).cpu().numpy()
    assert np.array_equal(got.view(np.uint64), ref.view(np.uint64))


@pytest.mark.gpu
@pytest.mark.parametrize("shape,m", [((40, 21), (2, 2)), ((70, 130), (6, 6)), ((9, 12), (3, 1))])
def test_row_stream_blocks_equal_batch(cuda, oracle_lib, shape, m):
    """push_rows(block) == the same rows pushed one by one == the batch rows."""
    from paper_1707_08213_b200.stream import SlidingRowStream2D

    rng = np.random.default_rng(shape[1] + m[1])
    x = rng.standard_normal(shape) + 1j * rng.standard_normal(shape)
    ref = oracle_lib.tree2d(x, *m)
    c = OpCounter(shape)
    st = SlidingRowStream2D(WindowSpec(m), shape[1], counter=c)
    got, r = [], 0
    for k in [1, 2, 5, 1, (1 << m[0]) + 3, 7, 100]:
        blk = x[r:r + k]
        r += len(blk)
        if len(blk) == 0:
            break
        out = st.push_rows(blk)
        if out is not None:
            got.append(out.cpu().numpy())
    got = np.concatenate(got)
    assert np.array_equal(got.view(np.uint64), ref.view(np.uint64))
    from paper_1707_08213_b200.tree2d import replay_counter

    cb = OpCounter(shape)
    replay_counter(cb, shape, WindowSpec(m))
    assert c.total == cb.total and np.array_equal(c.position_ops, cb.position_ops)
    st2 = SlidingRowStream2D(WindowSpec(m), shape[1])  # mixed single pushes after a block
    st2.push_rows(x[:3])
    tail = [st2.push_row(x[i]) for i in range(3, shape[0])]
    n0 = 1 << m[0]
    assert np.array_equal(tail[-1].cpu().numpy().view(np.uint64), ref[-1].view(np.uint64))


@pytest.mark.gpu
@pytest.mark.parametrize("precision", ["fp64", "fp32"])
@pytest.mark.parametrize("shape,m", [((90, 75), (4, 3)), ((150, 70), (6, 6)), ((33, 17), (2, 4))])
def test_row_stream_mixed_pushes(cuda, oracle_lib, shape, m, precision):
    """Blocks and single pushes interleaved (the level state is re-derived from the raw
    ring after each block), unitary normalization, real float32 rows: every slab equals
    the batch row — bitwise in fp64, within 1e-4 of the window norm in fp32."""
    from paper_1707_08213_b200.core import normalization_factor
    from paper_1707_08213_b200.stream import SlidingRowStream2D

    rng = np.random.default_rng(sum(shape) + m[0])
    x = rng.standard_normal(shape).astype(np.float32)
    spec = WindowSpec(m, "unitary")
    n0 = 1 << m[0]
    ref = oracle_lib.tree2d(x, *m, scale=normalization_factor(spec))
    st = SlidingRowStream2D(spec, shape[1], precision=precision)
    xd = torch.from_numpy(x).to(cuda)
    got, r = {}, 0
    plan = [1, 3, n0 + 2, 1, 1, 2, 5, n0 - 1 if n0 > 1 else 1, 1, 7, 1]
    while r < shape[0]:
        for k in plan:
            k = min(k, shape[0] - r)
            if k <= 0:
                break
            if k == 1 and r % 2 == 0:
                slab = st.push_row(xd[r])
                if slab is not None:
                    got[r - n0 + 1] = slab.cpu().numpy()
            else:
                out = st.push_rows(xd[r:r + k])
                if out is not None:
                    first = max(0, r - n0 + 1)
                    for i in range(out.shape[0]):
                        got[first + i] = out[i].cpu().numpy()
            r += k
    assert sorted(got) == list(range(ref.shape[0]))
    g = np.stack([got[i] for i in range(ref.shape[0])])
    if precision == "fp64":
        assert np.array_equal(g.view(np.uint64), ref.view(np.uint64))
    else:
        import oracle

        assert oracle.window_rel_err(g, ref) <= 1e-4


@pytest.mark.gpu
def test_row_stream_1x1_matches_reference_stream(golden, cuda):
    from paper_1707_08213_b200.stream import SlidingRowStream2D

    meta, _ = golden
    xs = np.random.default_rng(55).standard_normal((7, 6))
    st = SlidingRowStream2D(WindowSpec((0, 0)), 6)
    slabs = np.stack([st.push_row(r).cpu().numpy() for r in xs])
    assert sha(slabs) == meta["next"]["stream_1x1_sha"]


@pytest.mark.gpu
def test_tree1d_bitwise(golden, cuda):
    from paper_1707_08213_b200.tree1d import tree_swdft_1d

    meta, _ = golden
    for rec in meta["next"]["tree1d"]:
        s = (np.random.default_rng(rec["seed_re"]).standard_normal(rec["N"])
             + 1j * np.random.default_rng(rec["seed_im"]).standard_normal(rec["N"]))
        c = OpCounter((rec["N"],))
        v = tree_swdft_1d(s, WindowSpec((rec["m"],)), counter=c).values.cpu().numpy()
        assert sha(v) == rec["sha"]
        assert c.total == rec["total"] and sha(c.position_ops) == rec["pos_sha"]


@pytest.mark.gpu
def test_verify_tri_oracle(golden, cuda):
    from paper_1707_08213_b200.verify import verify

    meta, _ = golden
    x = np.random.default_rng(21).standard_normal((12, 9))
    err, exact, ok = verify(x, (4, 2))
    assert exact and ok and err <= 1e-10
    assert meta["next"]["verify"]["plain"]["rc"] == 0
    err2, exact2, ok2 = verify(x, (4, 2), corrupt=True)
    assert not exact2 and not ok2  # the detector fires, as the reference's does (rc 1)
    assert meta["next"]["verify"]["corrupt"]["rc"] == 1


@pytest.mark.gpu
def test_bench_csv_fig4(cuda, golden):
    from paper_1707_08213_b200.verify import bench_records, to_csv

    meta, _ = golden
    recs = bench_records(windows=((4, 4), (16, 16), (64, 64)), repetitions=2)
    text = to_csv(recs)
    lines = text.strip().splitlines()
    assert lines[0] == "algorithm,N0,N1,n0,n1,seconds,ops,peak_bytes"
    for r in recs:
        assert r.ops == meta["next"]["fig4_predict_ops"][str(r.window[0])][r.algorithm]
        assert r.seconds > 0


@pytest.mark.gpu
def test_transform_file_bytes(golden, cuda, tmp_path):
    """cmd_transform equivalent: CSV -> GPU tree (fp64) -> SWDF, byte-identical to the reference's."""
    from paper_1707_08213_b200.container import transform_file

    meta, _ = golden
    x = np.random.default_rng(21).standard_normal((12, 9))
    csvp = tmp_path / "x.csv"
    np.savetxt(csvp, x, delimiter=",")
    shape = transform_file(csvp, tmp_path / "t.swdf", (4, 2), normalization="paper-2d")
    assert shape == (9, 8, 4, 2)
    assert file_sha(tmp_path / "t.swdf") == meta["next"]["transform"]["sha"]


@pytest.mark.gpu
def test_treekd_bitwise(golden, cuda):
    """k-D tree by composition (slices through K1, then a dim-0 K1 pass): bitwise equal to the
    reference's generic engine, counter calls equal (SPEC acceptance 6 shapes)."""
    from paper_1707_08213_b200.treekd import tree_swdft_kd

    meta, _ = golden
    for rec in meta["next"]["treekd"]:
        rng = np.random.default_rng(rec["seed"])
        shape = tuple(rec["shape"])
        x = rng.standard_normal(shape) + 1j * rng.standard_normal(shape)
        c = OpCounter(shape)
        v = tree_swdft_kd(x, WindowSpec(tuple(rec["m"]), rec["mode"]), counter=c).values
        assert sha(v.cpu().numpy()) == rec["sha"], rec
        assert c.total == rec["total"] and sha(c.position_ops) == rec["pos_sha"]
    # 2D through the kD entry equals the 2D drop-in
    from paper_1707_08213_b200 import tree_swdft_2d

    x2 = np.random.default_rng(3).standard_normal((20, 17))
    a = tree_swdft_kd(x2, WindowSpec((2, 3))).values
    b = tree_swdft_2d(x2, WindowSpec((2, 3))).values
    assert torch_equal(a, b)


def torch_equal(a, b):
    import torch

    return torch.equal(a, b)


@pytest.mark.gpu
def test_stream1d_matches_reference(golden, cuda):
    """SlidingStream1D on the GPU: the emitted vectors are bitwise the reference's own
    sample-push stream (paper-1d normalization), per-push op counts and counter equal."""
    from paper_1707_08213_b200.stream import SlidingStream1D

    meta, _ = golden
    rec = meta["next"]["stream1d"]
    sig = (np.random.default_rng(57).standard_normal(40)
           + 1j * np.random.default_rng(58).standard_normal(40))
    c = OpCounter((40,))
    st = SlidingStream1D(WindowSpec((3,), "paper-1d"), counter=c)
    outs, ops = [], []
    for v in sig:
        r = st.push(v)
        ops.append(st.ops_last_push)
        if r is not None:
            outs.append(r.cpu().numpy())
    assert sha(np.stack(outs)) == rec["sha"]
    assert ops == rec["ops"] and c.total == rec["total"] and sha(c.position_ops) == rec["pos_sha"]


@pytest.mark.gpu
@pytest.mark.parametrize("m", [0, 1, 4, 6, 8])
def test_stream1d_equals_batch(cuda, m):
    """Sample pushes (K2 for n <= 64, the ring + KR above) emit the batch 1D tree's
    rows bitwise (fp64), with the unitary scale."""
    from paper_1707_08213_b200.stream import SlidingStream1D
    from paper_1707_08213_b200.tree1d import tree_swdft_1d

    rng = np.random.default_rng(70 + m)
    n = 1 << m
    sig = rng.standard_normal(n + 37) + 1j * rng.standard_normal(n + 37)
    spec = WindowSpec((m,), "unitary")
    ref = tree_swdft_1d(sig, spec).values.cpu().numpy()
    st = SlidingStream1D(spec)
    assert (st._state is not None) == (m <= 6)
    got = [st.push(v) for v in sig]
    assert all(g is None for g in got[:n - 1])
    g = np.stack([x.cpu().numpy() for x in got[n - 1:]])
    assert np.array_equal(g.view(np.uint64), ref.view(np.uint64))


@pytest.mark.gpu
def test_treekd_columns_and_m0_zero(cuda):
    """3-D and 4-D through the column-tree pass: equal (fp64 bits) to composing the
    2-D drop-in per slice and a dim-0 tree computed with the 1-D drop-in along i0;
    a window with n0 = 1 equals the per-slice 2-D result."""
    from paper_1707_08213_b200 import tree_swdft_2d
    from paper_1707_08213_b200.tree1d import tree_swdft_1d
    from paper_1707_08213_b200.treekd import tree_swdft_kd

    rng = np.random.default_rng(91)
    x = rng.standard_normal((19, 12, 14)) + 1j * rng.standard_normal((19, 12, 14))
    v = tree_swdft_kd(x, WindowSpec((3, 2, 3))).values.cpu().numpy()   # (P0,P1,P2,n0,n1,n2)
    sl = np.stack([tree_swdft_2d(x[i], WindowSpec((2, 3))).values.cpu().numpy()
                   for i in range(19)])                               # (N0,P1,P2,n1,n2)
    col = sl.reshape(19, -1)
    ref = np.stack([tree_swdft_1d(col[:, j], WindowSpec((3,))).values.cpu().numpy()
                    for j in range(col.shape[1])], axis=1)            # (P0, M, n0)
    ref = np.ascontiguousarray(ref.reshape((12, 9, 7, 4, 8, 8)).transpose(0, 1, 2, 5, 3, 4))
    assert np.array_equal(v.view(np.uint64), ref.view(np.uint64))
    v0 = tree_swdft_kd(x, WindowSpec((0, 2, 3))).values.cpu().numpy()
    assert np.array_equal(v0.view(np.uint64), sl.reshape(19, 9, 7, 1, 4, 8).view(np.uint64))


@pytest.mark.gpu
def test_row_stream_large_window(cuda, oracle_lib):
    """Windows beyond K2's 64 (here 128 x 4): pushes re-run the large-window path over
    the raw ring; slabs bitwise equal to the batch rows, blocks and singles mixed."""
    from paper_1707_08213_b200.stream import SlidingRowStream2D

    rng = np.random.default_rng(123)
    x = rng.standard_normal((140, 20)) + 1j * rng.standard_normal((140, 20))
    ref = oracle_lib.tree2d(x, 7, 2)
    st = SlidingRowStream2D(WindowSpec((7, 2)), 20)
    assert st._state is None
    out = st.push_rows(x[:130])
    got = [out.cpu().numpy()]
    for r in range(130, 140):
        got.append(st.push_row(x[r]).cpu().numpy()[None])
    g = np.concatenate(got)
    assert np.array_equal(g.view(np.uint64), ref.view(np.uint64))
