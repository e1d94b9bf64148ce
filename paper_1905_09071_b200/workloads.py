"""Synthetic inputs for the BASELINE.json configurations.

There is no public dataset for this path: these seeded recipes *are* the
workloads.  Shared by ``bench.py``, the tests and ``oracle/make_golden.py``.

* Permutation-power CP kernel of order d with exponents a[:d]:
  C_{i1..id} = sum over permutations s of prod_m i_m^{a[s(m)]}; rank R = d!,
  one column per permutation in ``itertools.permutations(range(d))`` order,
  column s of mode m is i^{a[s(m)]} = exp(a log i) (kernels.py:58-60, 443-450).
* Seeds: ``np.random.default_rng(0)`` (the reference's default seed,
  config.py:54, cli.py:123).
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from itertools import permutations

import numpy as np

__all__ = [
    "power_vector",
    "permutation_power_cp",
    "ConfigSpec",
    "CONFIGS",
    "initial_state",
]


def power_vector(n_classes: int, exponent: float) -> np.ndarray:
    """i^mu for i = 1..N computed as exp(mu log i) — kernels.py:58-60."""
    sizes = np.arange(1, n_classes + 1, dtype=np.float64)
    return np.exp(exponent * np.log(sizes))


def permutation_power_cp(exponents, n_classes: int) -> tuple[np.ndarray, ...]:
    """Exact CP factors (d arrays N x d!) of the permutation-power kernel."""
    d = len(exponents)
    pows = [power_vector(n_classes, float(a)) for a in exponents]
    perms = list(permutations(range(d)))
    factors = []
    for mode in range(d):
        f = np.empty((n_classes, len(perms)))
        for col, sigma in enumerate(perms):
            f[:, col] = pows[sigma[mode]]
        factors.append(f)
    return tuple(factors)


@dataclass(frozen=True)
class ConfigSpec:
    name: str
    n_classes: int
    orders: tuple
    exponents: tuple
    initial: str
    dt: float
    steps: int
    kind: str = "cp"

    def cp_factors(self, n_classes=None):
        n = n_classes or self.n_classes
        return {d: permutation_power_cp(self.exponents[:d], n) for d in self.orders}


# BASELINE.json "configs" (SURVEY.md §8(d) recipes)
CONFIGS = {
    "C1": ConfigSpec("C1", 4096, (2, 3), (0.1, -0.1, 0.0), "mono", 0.01, 100),
    "C2": ConfigSpec("C2", 65536, (2, 3), (0.15, -0.15, 0.05), "c2", 0.0, 1000),
    "C3": ConfigSpec("C3", 262144, (2, 3, 4), (0.1, -0.1, 0.05, -0.05), "exp256", 0.005, 200),
    "C4": ConfigSpec("C4", 1 << 20, (2, 3), (), "mono", 0.01, 100, kind="tt"),
    "C5": ConfigSpec("C5", 1 << 20, (2, 3, 4, 5), (0.1, -0.1, 0.05, -0.05, 0.0), "c5", 0.002, 50),
}


def initial_state(kind: str, n_classes: int, *, normalised: bool = False) -> np.ndarray:
    """Seeded initial concentrations of the configs."""
    k = np.arange(1, n_classes + 1, dtype=np.float64)
    if kind == "mono":
        n = np.zeros(n_classes)
        n[0] = 1.0
    elif kind == "c2":
        u = np.random.default_rng(0).random(n_classes)
        n = np.exp(-k / 64.0) * (1.0 + 0.1 * u)
    elif kind == "exp256":
        n = np.exp(-k / 256.0)
    elif kind == "c5":
        u = np.random.default_rng(0).random(n_classes)
        n = np.exp(-k / 1024.0) * (1.0 + 0.05 * (2.0 * u - 1.0))
    else:
        raise ValueError(kind)
    if normalised:
        n = n / n.sum()
    return n


def factorial(d: int) -> int:
    return math.factorial(d)
