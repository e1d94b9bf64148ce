"""Kernel containers — name- and behaviour-compatible with the reference's
``TTKernel`` / ``CPKernel`` / ``KernelError`` (``ttagg/kernels.py:48-215``).

They are plain immutable fp64 holders; construction (Brownian TT builder,
specs, dense expansions) is outside this build's scope.
The GPU operators accept these *or* the reference's own objects (anything
with ``.factors`` / ``.cores``).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

__all__ = ["KernelError", "TTKernel", "CPKernel", "DenseKernel", "constant_cp", "constant_tt"]


class KernelError(ValueError):
    """Malformed kernel data, out-of-range index, or budget violation (kernels.py:48-49)."""


def _readonly(arr) -> np.ndarray:
    out = np.ascontiguousarray(arr, dtype=np.float64)
    if out is arr:
        out = arr.copy()
    out.setflags(write=False)
    return out


@dataclass(frozen=True, eq=False)
class TTKernel:
    """Chain of 3-way cores (R_prev, N, R_next), boundary ranks 1 (kernels.py:137-180)."""

    cores: tuple

    def __post_init__(self):
        cores = tuple(_readonly(c) for c in self.cores)
        if len(cores) < 2:
            raise KernelError("a TT kernel needs at least two cores")
        for lam, core in enumerate(cores, start=1):
            if core.ndim != 3:
                raise KernelError(f"core {lam} is not a 3-way array")
        if cores[0].shape[0] != 1 or cores[-1].shape[2] != 1:
            raise KernelError("boundary TT ranks must equal 1")
        n_classes = cores[0].shape[1]
        for lam in range(len(cores)):
            if cores[lam].shape[1] != n_classes:
                raise KernelError("all cores must share the same mode size")
            if lam and cores[lam - 1].shape[2] != cores[lam].shape[0]:
                raise KernelError(f"rank mismatch between cores {lam} and {lam + 1}")
        object.__setattr__(self, "cores", cores)

    @property
    def dimension(self) -> int:
        return len(self.cores)

    @property
    def n_classes(self) -> int:
        return self.cores[0].shape[1]

    @property
    def ranks(self) -> tuple:
        return (1,) + tuple(c.shape[2] for c in self.cores)

    @property
    def max_rank(self) -> int:
        return max(self.ranks)


@dataclass(frozen=True, eq=False)
class CPKernel:
    """One N x R factor matrix per mode (kernels.py:183-215)."""

    factors: tuple

    def __post_init__(self):
        factors = tuple(_readonly(f) for f in self.factors)
        if len(factors) < 2:
            raise KernelError("a CP kernel needs at least two factors")
        shape = factors[0].shape
        if len(shape) != 2:
            raise KernelError("CP factors must be N x R matrices")
        for f in factors:
            if f.shape != shape:
                raise KernelError("all CP factors must share the same N x R shape")
        object.__setattr__(self, "factors", factors)

    @property
    def dimension(self) -> int:
        return len(self.factors)

    @property
    def n_classes(self) -> int:
        return self.factors[0].shape[0]

    @property
    def rank(self) -> int:
        return self.factors[0].shape[1]


def constant_tt(value: float, dimension: int, n_classes: int) -> TTKernel:
    """Rank-1 TT kernel with every coefficient equal to value (kernels.py:373-379)."""
    if dimension < 2:
        raise KernelError("kernel dimension must be >= 2")
    cores = [np.ones((1, n_classes, 1)) for _ in range(dimension)]
    cores[0] = cores[0] * float(value)
    return TTKernel(tuple(cores))


def constant_cp(value: float, dimension: int, n_classes: int) -> CPKernel:
    """Rank-1 CP kernel with every coefficient equal to value (kernels.py:382-388)."""
    if dimension < 2:
        raise KernelError("kernel dimension must be >= 2")
    factors = [np.ones((n_classes, 1)) for _ in range(dimension)]
    factors[0] = factors[0] * float(value)
    return CPKernel(tuple(factors))


@dataclass(frozen=True, eq=False)
class DenseKernel:
    """Fully materialized kernel (kernels.py:218-238): N^d coefficients,
    row-major, equal mode sizes; evaluated by direct summation."""

    values: np.ndarray

    def __post_init__(self):
        values = _readonly(self.values)
        if values.ndim < 2:
            raise KernelError("dense kernels must have dimension >= 2")
        n_classes = values.shape[0]
        if any(s != n_classes for s in values.shape):
            raise KernelError("dense kernels must have equal mode sizes")
        object.__setattr__(self, "values", values)

    @property
    def dimension(self) -> int:
        return self.values.ndim

    @property
    def n_classes(self) -> int:
        return self.values.shape[0]
