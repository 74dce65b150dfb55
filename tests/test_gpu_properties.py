"""SPEC.md acceptance 8 property suite on the device path, plus a seeded fuzz of
shapes / windows / dtypes against the pinned oracle (fp64 bitwise)."""
import numpy as np
import pytest
from hypothesis import HealthCheck, given, settings
from hypothesis import strategies as st

from paper_1707_08213_b200 import WindowSpec, tree_swdft_2d

pytestmark = pytest.mark.gpu


def run(x, m, precision="fp64", kernel="auto", normalization="none"):
    return tree_swdft_2d(x, WindowSpec(m, normalization), precision=precision, kernel=kernel,
                         budget=1 << 62).values.cpu().numpy()


@settings(max_examples=60, deadline=None, suppress_health_check=list(HealthCheck))
@given(N0=st.integers(1, 40), N1=st.integers(1, 70), m0=st.integers(0, 5), m1=st.integers(0, 6),
       cplx=st.booleans(), kernel=st.sampled_from(["auto", "window", "stream_tma"]),
       seed=st.integers(0, 2**31 - 1))
def test_fuzz_fp64_bitwise(cuda, oracle_lib, N0, N1, m0, m1, cplx, kernel, seed):
    if (1 << m0) > N0 or (1 << m1) > N1:
        return
    rng = np.random.default_rng(seed)
    x = rng.standard_normal((N0, N1)) + (1j * rng.standard_normal((N0, N1)) if cplx else 0)
    ref = oracle_lib.tree2d(x, m0, m1)
    got = run(x, (m0, m1), kernel=kernel)
    assert np.array_equal(got.view(np.uint64), ref.view(np.uint64))


@pytest.mark.parametrize("m", [(2, 2), (3, 1), (4, 4), (1, 5)])
def test_parseval_per_window(cuda, m):
    """sum_k |a_k|^2 = n0 n1 sum_j |x_j|^2 per window, 1e-9 relative."""
    rng = np.random.default_rng(sum(m))
    x = rng.standard_normal((48, 40)) + 1j * rng.standard_normal((48, 40))
    a = run(x, m)
    n0, n1 = 1 << m[0], 1 << m[1]
    w = np.lib.stride_tricks.sliding_window_view(x, (n0, n1))
    lhs = (np.abs(a) ** 2).sum((-1, -2))
    rhs = n0 * n1 * (np.abs(w) ** 2).sum((-1, -2))
    assert np.max(np.abs(lhs - rhs) / rhs) <= 1e-9


def test_unitary_and_paper2d_scaling(cuda):
    """Normalization is the per-window factor 1/sqrt(n0 n1) of the raw transform."""
    rng = np.random.default_rng(4)
    x = rng.standard_normal((30, 20))
    raw = run(x, (2, 3))
    for mode in ("unitary", "paper-2d"):
        got = run(x, (2, 3), normalization=mode)
        assert np.array_equal(got, raw * (1.0 / np.sqrt(32.0)))


def test_axis_permutation_kd(cuda):
    """Permuting the axes of a 3D array permutes position and frequency axes alike
    (SPEC.md acceptance 8), within 1e-10."""
    from paper_1707_08213_b200.treekd import tree_swdft_kd

    rng = np.random.default_rng(5)
    x = rng.standard_normal((9, 8, 7)) + 1j * rng.standard_normal((9, 8, 7))
    m = (2, 1, 2)
    a = tree_swdft_kd(x, WindowSpec(m)).values.cpu().numpy()
    perm = (2, 0, 1)
    b = tree_swdft_kd(np.ascontiguousarray(x.transpose(perm)),
                      WindowSpec(tuple(m[p] for p in perm))).values.cpu().numpy()
    full_perm = perm + tuple(3 + p for p in perm)
    assert np.abs(b - a.transpose(full_perm)).max() <= 1e-10


def test_fp32_accuracy_bound_large_values(cuda, oracle_lib):
    """fp32 tolerance holds for inputs with a large DC offset (worst case for
    cancellation in the window-relative metric)."""
    import oracle

    rng = np.random.default_rng(6)
    x = (1e3 + rng.standard_normal((80, 70))).astype(np.float32)
    for m in [(4, 4), (5, 3), (6, 6)]:
        ref = oracle_lib.tree2d(x.astype(np.float64), *m)
        got = run(x, m, precision="fp32")
        assert oracle.window_rel_err(got, ref) <= 1e-4


def test_special_values_fp64(cuda, oracle_lib):
    """Infinities, NaNs, signed zeros and subnormals flow through the device tree exactly
    as through the reference's arithmetic: identical bits wherever the result is not
    NaN, and NaN in exactly the same places."""
    rng = np.random.default_rng(9)
    x = rng.standard_normal((24, 20))
    x[3, 4] = np.inf
    x[10, 11] = -np.inf
    x[15, 2] = np.nan
    x[5, 15] = -0.0
    x[20, 7] = 5e-324
    x[0, 0] = 2.2250738585072014e-308 / 3
    for m in [(2, 2), (3, 1), (1, 3)]:
        ref = oracle_lib.tree2d(x, *m)
        for kernel in ("auto", "window"):
            got = run(x, m, kernel=kernel)
            rn, gn = np.isnan(ref.view(np.float64)), np.isnan(got.view(np.float64))
            assert np.array_equal(rn, gn)
            assert np.array_equal(ref.view(np.uint64)[~rn], got.view(np.uint64)[~gn])


@settings(max_examples=40, deadline=None, suppress_health_check=list(HealthCheck))
@given(N0=st.integers(1, 3), m1=st.integers(0, 10), extra=st.integers(0, 700),
       cplx=st.booleans(), seed=st.integers(0, 2**31 - 1))
def test_fuzz_row_kernel_fp64_bitwise(cuda, oracle_lib, N0, m1, extra, cplx, seed):
    """KR (n0 = 1, n1 up to 1024) on random widths, ragged tiles included."""
    N1 = (1 << m1) + extra
    rng = np.random.default_rng(seed)
    x = rng.standard_normal((N0, N1)) + (1j * rng.standard_normal((N0, N1)) if cplx else 0)
    ref = oracle_lib.tree2d(x, 0, m1)
    got = run(x, (0, m1), kernel="rows")
    assert np.array_equal(got.view(np.uint64), ref.view(np.uint64))


@settings(max_examples=25, deadline=None, suppress_health_check=list(HealthCheck))
@given(N0=st.integers(1, 30), N1=st.integers(1, 50), m0=st.integers(0, 5), m1=st.integers(0, 5),
       blocks=st.lists(st.integers(1, 9), min_size=1, max_size=12), seed=st.integers(0, 2**31 - 1))
def test_fuzz_row_stream_fp64_bitwise(cuda, oracle_lib, N0, N1, m0, m1, blocks, seed):
    """Row-push stream (K2 single pushes, K1 blocks, state catch-up) == batch rows."""
    from paper_1707_08213_b200.stream import SlidingRowStream2D

    if (1 << m0) > N0 or (1 << m1) > N1:
        return
    rng = np.random.default_rng(seed)
    x = rng.standard_normal((N0, N1)) + 1j * rng.standard_normal((N0, N1))
    ref = oracle_lib.tree2d(x, m0, m1)
    st_ = SlidingRowStream2D(WindowSpec((m0, m1)), N1)
    n0, got, r, i = 1 << m0, [], 0, 0
    while r < N0:
        k = min(blocks[i % len(blocks)], N0 - r)
        i += 1
        if k == 1:
            s = st_.push_row(x[r])
            if s is not None:
                got.append(s.cpu().numpy()[None])
        else:
            o = st_.push_rows(x[r:r + k])
            if o is not None:
                got.append(o.cpu().numpy())
        r += k
    g = np.concatenate(got)
    assert np.array_equal(g.view(np.uint64), ref.view(np.uint64))
