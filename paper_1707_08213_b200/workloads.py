"""Seeded synthetic workloads of BASELINE.json's five configurations.

There is no public dataset for this path; these generators
produce inputs with the configs' shapes, dtypes and value distributions.  They
are deterministic for a given numpy version (PCG64 streams are stable), so the
build container, the GPU box and the golden fixtures agree on the inputs.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class Workload:
    name: str
    N0: int
    N1: int
    m0: int
    m1: int
    dtype: str      # numpy dtype of the input
    precision: str  # "fp64" (complex128 out) or "fp32" (complex64 out)
    desc: str

    @property
    def n0(self) -> int:
        return 1 << self.m0

    @property
    def n1(self) -> int:
        return 1 << self.m1

    @property
    def P0(self) -> int:
        return self.N0 - self.n0 + 1

    @property
    def P1(self) -> int:
        return self.N1 - self.n1 + 1

    @property
    def coefficients(self) -> int:
        return self.P0 * self.P1 * self.n0 * self.n1

    @property
    def out_bytes_per_coef(self) -> int:
        return 16 if self.precision == "fp64" else 8

    @property
    def in_bytes(self) -> int:
        return self.N0 * self.N1 * np.dtype(self.dtype).itemsize

    def algorithmic_bytes(self, rows: int | None = None, precision: str | None = None) -> int:
        """Output bytes written + input bytes read, for the
        full output or for ``rows`` window rows, at the config's precision or
        ``precision`` ("fp32": 8 B per coefficient, "fp64": 16 B)."""
        ob = self.out_bytes_per_coef if precision is None else (16 if precision == "fp64" else 8)
        if rows is None:
            return self.coefficients * ob + self.in_bytes
        in_rows = rows + self.n0 - 1
        return (rows * self.P1 * self.n0 * self.n1 * ob
                + in_rows * self.N1 * np.dtype(self.dtype).itemsize)

    def generate(self, rows: int | None = None) -> np.ndarray:
        """The input array; ``rows`` limits it to its first input rows."""
        x = GENERATORS[self.name]()
        return x if rows is None else np.ascontiguousarray(x[:rows])


def _c1():
    return np.random.default_rng(0).standard_normal((64, 64))


def _c2():
    return np.random.default_rng(1).uniform(-1.0, 1.0, (512, 512)).astype(np.float32)


def _c3():
    return np.random.default_rng(2).standard_normal((2048, 2048)).astype(np.float32)


def _c4():
    rng = np.random.default_rng(3)
    f0 = rng.uniform(0.0, 0.5, 20)
    f1 = rng.uniform(0.0, 0.5, 20)
    ph = rng.uniform(0.0, 2.0 * np.pi, 20)
    i = np.arange(4096, dtype=np.float64)[:, None]
    j = np.arange(4096, dtype=np.float64)[None, :]
    x = np.zeros((4096, 4096), dtype=np.float64)
    for k in range(20):
        x += np.cos(2.0 * np.pi * (f0[k] * i + f1[k] * j) + ph[k])
    x += rng.normal(0.0, 0.1, (4096, 4096))
    return x.astype(np.float32)


def _c5():
    rng = np.random.default_rng(4)
    re = rng.standard_normal((2048, 2048))
    im = rng.standard_normal((2048, 2048))
    return (re + 1j * im).astype(np.complex64)


GENERATORS = {"c1": _c1, "c2": _c2, "c3": _c3, "c4": _c4, "c5": _c5}

CONFIGS = {
    "c1": Workload("c1", 64, 64, 3, 3, "float64", "fp64",
                   "64x64 f64 N(0,1) seed 0, 8x8 windows -> 57x57x8x8 complex128"),
    "c2": Workload("c2", 512, 512, 4, 4, "float32", "fp32",
                   "512x512 f32 U[-1,1] seed 1, 16x16 -> 497x497x16x16 complex64"),
    "c3": Workload("c3", 2048, 2048, 5, 3, "float32", "fp32",
                   "2048x2048 f32 N(0,1) seed 2, 32x8 -> 2017x2041x32x8 complex64"),
    "c4": Workload("c4", 4096, 4096, 4, 4, "float32", "fp32",
                   "4096x4096 f32 20 sinusoids + N(0,0.1^2) seed 3, 16x16 -> 4081x4081x16x16 complex64"),
    "c5": Workload("c5", 2048, 2048, 6, 6, "complex64", "fp32",
                   "2048x2048 c64 N(0,1) re/im seed 4, 64x64 -> 1985x1985x64x64 complex64"),
}
