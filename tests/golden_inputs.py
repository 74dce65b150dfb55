"""Regenerate the seeded inputs the golden vectors were made from
(mirrors tests/golden/make_golden.py; no reference import)."""
import numpy as np


def acc_input(case: int):
    rng = np.random.default_rng(1000 + case)
    N0 = int(rng.integers(8, 17))
    N1 = int(rng.integers(8, 17))
    return rng.standard_normal((N0, N1)) + 1j * rng.standard_normal((N0, N1))


def kat6_input():
    rng = np.random.default_rng(77)
    x = rng.standard_normal((6, 8)) + 1j * rng.standard_normal((6, 8))
    norm_x = rng.standard_normal((12, 10))
    return x, norm_x
