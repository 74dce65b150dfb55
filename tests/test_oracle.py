"""Pin the oracle (C + numpy restatements) to the reference's golden vectors.  CPU only."""
import numpy as np
import pytest

from conftest import sha
from golden_inputs import acc_input, kat6_input
from paper_1707_08213_b200.workloads import CONFIGS


def test_twiddles_bitwise(golden, oracle_lib):
    meta, _ = golden
    from oracle import tree2d_np

    for n, h in meta["twiddles"].items():
        assert sha(oracle_lib.twiddles(int(n))) == h
        assert sha(tree2d_np.twiddles(int(n))) == h


def test_kats(golden, oracle_lib):
    meta, arr = golden
    x = np.array(meta["kat"]["kat1"]["x"])
    out = oracle_lib.tree2d(x, 1, 1)
    assert np.array_equal(out.view(np.uint64), arr["kat1_out"].view(np.uint64))
    # [[10,-2],[-4,0]] within rounding (imag parts ~1e-16: sin(pi) != 0)
    assert np.allclose(out[0, 0], [[10, -2], [-4, 0]], atol=1e-15)
    out = oracle_lib.tree2d(np.ones((8, 8)), 2, 2)
    assert np.array_equal(out.view(np.uint64), arr["kat2_out"].view(np.uint64))
    assert np.all(out[..., 0, 0] == 16)
    k6, nx = kat6_input()
    assert np.array_equal(oracle_lib.tree2d(k6, 1, 2).view(np.uint64), arr["kat6_out"].view(np.uint64))
    f = 1.0 / np.sqrt(8.0)
    for mode in ("unitary", "paper-2d"):
        got = oracle_lib.tree2d(nx, 2, 1, scale=f)
        assert np.array_equal(got.view(np.uint64), arr[f"norm_{mode}_out"].view(np.uint64))


def test_acceptance_sweep_bitwise(golden, oracle_lib):
    """SPEC.md acceptance 1+2: 50 arrays x windows {1,2,4,8}^2, SHA-256 of the reference output."""
    meta, _ = golden
    from oracle import tree2d_np

    for i, rec in enumerate(meta["acc"]):
        x = acc_input(rec["case"])
        assert sha(x) == rec["in_sha"]
        out = oracle_lib.tree2d(x, rec["m0"], rec["m1"], threads=2)
        assert sha(out) == rec["sha"], rec
        if i % 7 == 0:
            assert sha(tree2d_np.tree2d_levels_outer(x, rec["m0"], rec["m1"])) == rec["sha"]


def test_acceptance_naive_tolerance(oracle_lib):
    """SPEC.md acceptance 1: tree vs the literal double sum (Eq. 2) <= 1e-10."""
    for case in range(0, 50, 5):
        x = acc_input(case)
        for m0 in range(4):
            for m1 in range(4):
                n0, n1 = 1 << m0, 1 << m1
                if n0 > x.shape[0] or n1 > x.shape[1]:
                    continue
                out = oracle_lib.tree2d(x, m0, m1)
                win = np.lib.stride_tricks.sliding_window_view(x, (n0, n1))
                k0 = np.exp(-2j * np.pi / n0 * np.outer(np.arange(n0), np.arange(n0)))
                k1 = np.exp(-2j * np.pi / n1 * np.outer(np.arange(n1), np.arange(n1)))
                naive = np.einsum("pqjl,kj,ml->pqkm", win, k0, k1)
                assert np.abs(out - naive).max() <= 1e-10


def test_window_fft_schedule_bitwise(oracle_lib):
    """oracle.swfft_2d's per-window schedule reproduces the tree bit for bit."""
    x = acc_input(3)
    for m0, m1 in [(3, 2), (2, 3), (0, 3), (3, 0)]:
        full = oracle_lib.tree2d(x, m0, m1)
        for (p0, p1) in [(0, 0), (full.shape[0] - 1, full.shape[1] - 1),
                         (full.shape[0] // 2, full.shape[1] // 3)]:
            w = oracle_lib.window_fft(x, m0, m1, p0, p1)
            assert np.array_equal(w.view(np.uint64), full[p0, p1].view(np.uint64))


def test_config1_full_bitwise(golden, oracle_lib):
    meta, arr = golden
    cfg = CONFIGS["c1"]
    x = cfg.generate()
    assert sha(x) == meta["configs"]["c1"]["in_sha"]
    out = oracle_lib.tree2d(x, cfg.m0, cfg.m1, threads=4)
    assert sha(out) == meta["configs"]["c1"]["full_sha"]


@pytest.mark.parametrize("name", ["c1", "c2", "c3", "c4", "c5"])
def test_config_windows_and_strips(golden, oracle_lib, name):
    """Sampled windows (values) and small strips (SHA-256) of every config."""
    meta, arr = golden
    cfg = CONFIGS[name]
    x = cfg.generate()
    assert sha(x) == meta["configs"][name]["in_sha"]
    for (p0, p1), ref in zip(arr[f"{name}_win_pos"], arr[f"{name}_win_out"]):
        sub = x[p0:p0 + cfg.n0, p1:p1 + cfg.n1]
        got = oracle_lib.tree2d(sub, cfg.m0, cfg.m1)[0, 0]
        assert np.array_equal(got.view(np.uint64), ref.view(np.uint64))
        # independent check: numpy's FFT of the same window (not bitwise)
        f = np.fft.fft2(sub.astype(np.complex128))
        assert np.abs(f - ref).max() <= 1e-10 * max(1.0, np.linalg.norm(ref))
    for st in meta["configs"][name]["strips"]:
        sub = x[st["p0"]:st["p0"] + st["rows"] + cfg.n0 - 1, st["p1"]:st["p1"] + st["cols"] + cfg.n1 - 1]
        assert sha(oracle_lib.tree2d(sub, cfg.m0, cfg.m1, threads=4)) == st["sha"]


def test_strip_invariance(oracle_lib):
    """Output rows computed as strips equal the full run bitwise."""
    x = acc_input(11)
    full = oracle_lib.tree2d(x, 2, 3)
    for a, b in [(0, 1), (1, 4), (2, full.shape[0])]:
        part = oracle_lib.tree2d(x, 2, 3, p0_begin=a, p0_end=b, max_lattice_bytes=1)
        assert np.array_equal(part.view(np.uint64), full[a:b].view(np.uint64))
