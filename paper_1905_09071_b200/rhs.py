"""GPU right-hand-side operators with the reference's API (``ttagg/rhs.py``).

Same names, signatures, argument meaning, return types and error behaviour
as the reference:

* ``rhs_cp_P(kernel, state, plan=None)``  — rhs.py:345-391
* ``rhs_cp_Q(kernel, state, plan=None)``  — rhs.py:394-414
* ``rhs_tt_P(kernel, state, plan=None)``  — rhs.py:234-302
* ``rhs_tt_Q(kernel, state, plan=None)``  — rhs.py:321-338
* ``rhs_dense_P(kernel, state)`` / ``rhs_dense_Q(kernel, state)`` — rhs.py:202-227
* ``rhs_total(kernels, state, plan=None, *, breakdown=False)`` — rhs.py:421-459

All arithmetic runs in the sm_100a CUDA extension (``libttagg_b200.so``);
there is no CPU fallback.  Inputs may be this package's containers or the
reference's own ``CPKernel`` / ``TTKernel`` / ``DenseKernel`` / ``ConcentrationState`` /
``KernelSet`` objects.  Outputs are fresh fp64 numpy arrays owned by the
caller (rhs.py:296, 385, 459).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from ._lib import active_group, get_context
from .kernels import CPKernel, DenseKernel, KernelError, TTKernel
from .parallel import SERIAL_PLAN, ExecutionPlan

__all__ = [
    "ConcentrationState",
    "KernelSet",
    "RhsResult",
    "kernel_element",
    "sample_symmetry_violation",
    "rhs_tt_P",
    "rhs_tt_Q",
    "rhs_cp_P",
    "rhs_cp_Q",
    "rhs_dense_P",
    "rhs_dense_Q",
    "rhs_total",
    "DENSE_RHS_BUDGET",
]

DENSE_RHS_BUDGET = 1 << 26  # rhs.py:47

_SYMMETRY_CHECK_MAX_N = 64
_SYMMETRY_TOL = 1e-8


_PIN_MIN = 1 << 16


def _host_copy(n: np.ndarray) -> np.ndarray:
    """The state's own copy (rhs.py:66-68); large states land in page-locked
    memory so every RHS on them transfers by DMA without a staging copy."""
    if n.size >= _PIN_MIN:
        try:
            import torch

            if torch.cuda.is_available():
                out = torch.empty(n.size, dtype=torch.float64, pin_memory=True).numpy()
                np.copyto(out, n)
                return out
        except Exception:  # no CUDA runtime: plain copy
            pass
    return n.copy()


@dataclass(frozen=True)
class ConcentrationState:
    """Per-size concentrations n_1..n_N at time t (rhs.py:54-79)."""

    n: np.ndarray
    t: float = 0.0

    def __post_init__(self):
        n = np.ascontiguousarray(self.n, dtype=np.float64)
        if n is self.n or n.size >= _PIN_MIN:
            n = _host_copy(n)
        if n.ndim != 1 or n.size < 2:
            raise ValueError("concentration state must be a vector of length >= 2")
        if not np.all(np.isfinite(n)):
            raise ValueError("concentration state contains non-finite entries")
        n.setflags(write=False)
        object.__setattr__(self, "n", n)
        object.__setattr__(self, "t", float(self.t))

    @property
    def n_classes(self) -> int:
        return self.n.size


def _is_cp(k) -> bool:
    return hasattr(k, "factors")


def _is_tt(k) -> bool:
    return hasattr(k, "cores")


def _is_dense(k) -> bool:
    return hasattr(k, "values") and not (_is_cp(k) or _is_tt(k))


def _dimension(k) -> int:
    if _is_dense(k):
        return np.ndim(k.values)
    return len(k.factors) if _is_cp(k) else len(k.cores)


def _n_classes(k) -> int:
    if _is_dense(k):
        return k.values.shape[0]
    return k.factors[0].shape[0] if _is_cp(k) else k.cores[0].shape[1]


def kernel_element(kernel, idx) -> float:
    """One coefficient of a CP, TT or dense kernel (rhs.py:80-91; kernels.py:310-325)."""
    entries = tuple(int(i) for i in idx)
    d = _dimension(kernel)
    if len(entries) != d:
        raise KernelError(f"index has {len(entries)} entries, kernel dimension is {d}")
    if _is_cp(kernel):
        acc = np.ones(kernel.factors[0].shape[1])
        for size, f in zip(entries, kernel.factors):
            acc = acc * f[size - 1]
        return float(acc.sum())
    if _is_tt(kernel):
        v = kernel.cores[0][:, entries[0] - 1, :]
        for size, core in zip(entries[1:], kernel.cores[1:]):
            v = v @ core[:, size - 1, :]
        return float(v[0, 0])
    if _is_dense(kernel):
        return float(kernel.values[tuple(i - 1 for i in entries)])
    raise KernelError(f"unsupported kernel representation {type(kernel).__name__}")


def sample_symmetry_violation(kernel, samples: int = 32, seed: int = 0) -> float:
    """Largest relative coefficient change under index permutations (rhs.py:94-111)."""
    rng = np.random.default_rng(seed)
    d, n = _dimension(kernel), _n_classes(kernel)
    worst = 0.0
    for _ in range(samples):
        idx = rng.integers(1, n + 1, size=d)
        ref = kernel_element(kernel, idx)
        for alt_idx in (idx[::-1], rng.permutation(idx)):
            alt = kernel_element(kernel, alt_idx)
            scale = max(abs(ref), abs(alt), 1e-300)
            worst = max(worst, abs(ref - alt) / scale)
    return worst


@dataclass(frozen=True)
class KernelSet:
    """Kernels by collision order d >= 2 sharing one N (rhs.py:114-161)."""

    kernels: dict

    def __post_init__(self):
        checked = {}
        n_classes = None
        for order, kernel in self.kernels.items():
            d = int(order)
            if d < 2:
                raise KernelError(f"collision order must be >= 2, got {d}")
            if not (_is_cp(kernel) or _is_tt(kernel) or _is_dense(kernel)):
                raise KernelError(f"unsupported kernel representation {type(kernel).__name__}")
            if _dimension(kernel) != d:
                raise KernelError(f"kernel for order {d} has dimension {_dimension(kernel)}")
            if n_classes is None:
                n_classes = _n_classes(kernel)
            elif _n_classes(kernel) != n_classes:
                raise KernelError("all kernels in a set must share the same N")
            checked[d] = kernel
        if n_classes is not None and n_classes <= _SYMMETRY_CHECK_MAX_N:
            for d, kernel in checked.items():
                violation = sample_symmetry_violation(kernel)
                if violation > _SYMMETRY_TOL:
                    raise KernelError(
                        f"kernel for order {d} is not symmetric "
                        f"(sampled relative violation {violation:.2e})"
                    )
        object.__setattr__(self, "kernels", checked)

    @property
    def orders(self) -> tuple:
        return tuple(sorted(self.kernels))

    @property
    def n_classes(self) -> int:
        if not self.kernels:
            raise KernelError("empty kernel set has no mode size")
        return _n_classes(next(iter(self.kernels.values())))

    def __getitem__(self, order: int):
        return self.kernels[order]


@dataclass(frozen=True)
class RhsResult:
    """Gain p, loss q, s = p + q, optionally per order (rhs.py:164-171)."""

    p: np.ndarray
    q: np.ndarray
    s: np.ndarray
    by_order: dict | None = None


def _state_n(state) -> np.ndarray:
    n = state.n if hasattr(state, "n") else state
    return np.ascontiguousarray(n, dtype=np.float64)


def _check_pair(kernel, state) -> tuple:
    n = _state_n(state)
    if _n_classes(kernel) != n.size:
        raise KernelError(f"kernel has N = {_n_classes(kernel)}, state has N = {n.size}")
    return _dimension(kernel), n


def _one(kernel, state, want_p: bool, want_q: bool, kind_ok, label: str):
    if not kind_ok(kernel):
        kind = {_is_cp: "CP", _is_tt: "TT", _is_dense: "dense"}[kind_ok]
        raise KernelError(f"{label} needs a {kind} kernel, got {type(kernel).__name__}")
    d, n = _check_pair(kernel, state)
    if kind_ok is _is_dense:
        _dense_budget_check(d, n.size)
    grp = active_group()
    if grp is not None:
        out = grp.rhs_host([kernel], n, outputs=("p",) if want_p else ("q",))
        return out["p"] if want_p else out["q"]
    ctx = get_context()
    dk = ctx.device_kernel(kernel)
    out = ctx.rhs_host([dk], n, want_p=want_p, want_q=want_q,
                       outputs=("p",) if want_p else ("q",))
    return out["p"] if want_p else out["q"]


def rhs_tt_P(kernel: TTKernel, state: ConcentrationState, plan: ExecutionPlan | None = None) -> np.ndarray:
    """Gain vector through a TT kernel (rhs.py:234-302), on the GPU."""
    return _one(kernel, state, True, False, _is_tt, "rhs_tt_P")


def rhs_tt_Q(kernel: TTKernel, state: ConcentrationState, plan: ExecutionPlan | None = None) -> np.ndarray:
    """Loss vector through a TT kernel (rhs.py:321-338), on the GPU."""
    return _one(kernel, state, False, True, _is_tt, "rhs_tt_Q")


def rhs_cp_P(kernel: CPKernel, state: ConcentrationState, plan: ExecutionPlan | None = None) -> np.ndarray:
    """Gain vector through a CP kernel (rhs.py:345-391), on the GPU."""
    return _one(kernel, state, True, False, _is_cp, "rhs_cp_P")


def rhs_cp_Q(kernel: CPKernel, state: ConcentrationState, plan: ExecutionPlan | None = None) -> np.ndarray:
    """Loss vector through a CP kernel (rhs.py:394-414), on the GPU."""
    return _one(kernel, state, False, True, _is_cp, "rhs_cp_Q")


def _dense_budget_check(order: int, n_classes: int) -> None:
    """rhs.py:188-199."""
    if n_classes**order > DENSE_RHS_BUDGET:
        raise KernelError(
            f"dense evaluation needs {n_classes**order} elements, over the "
            f"budget of {DENSE_RHS_BUDGET}; reduce N"
        )


def rhs_dense_P(kernel: DenseKernel, state: ConcentrationState) -> np.ndarray:
    """Gain vector by direct summation over all d-tuples (rhs.py:202-216), on the GPU."""
    return _one(kernel, state, True, False, _is_dense, "rhs_dense_P")


def rhs_dense_Q(kernel: DenseKernel, state: ConcentrationState) -> np.ndarray:
    """Loss vector by contracting the first d-1 modes with the state (rhs.py:219-227), on the GPU."""
    return _one(kernel, state, False, True, _is_dense, "rhs_dense_Q")


def _kernel_items(kernels):
    """(order, kernel) pairs in ascending order from a KernelSet-like object."""
    if hasattr(kernels, "orders") and hasattr(kernels, "__getitem__"):
        return [(d, kernels[d]) for d in kernels.orders]
    if isinstance(kernels, dict):
        return [(d, kernels[d]) for d in sorted(kernels)]
    raise KernelError(f"unsupported kernel set {type(kernels).__name__}")


def rhs_total(kernels: KernelSet, state: ConcentrationState, plan: ExecutionPlan | None = None,
              *, breakdown: bool = False) -> RhsResult:
    """Sum of gain and loss over every configured order (rhs.py:421-459).

    One fused GPU evaluation over all orders (gains, losses, order sum and
    s = p + q in a single combine pass).  With ``breakdown`` each order is
    evaluated separately and accumulated in ascending order like the
    reference, so ``sum(p_d) == p`` exactly.
    """
    items = _kernel_items(kernels)
    if not items:
        raise KernelError("no collision orders configured")
    n = _state_n(state)
    n_classes = _n_classes(items[0][1])
    if n_classes != n.size:
        raise KernelError(f"kernel set has N = {n_classes}, state has N = {n.size}")
    for d, k in items:
        if not (_is_cp(k) or _is_tt(k) or _is_dense(k)):
            raise KernelError(f"unsupported kernel representation {type(k).__name__}")
        if _is_dense(k):
            _dense_budget_check(d, n.size)
    grp = active_group()
    if grp is not None:  # several GPUs: rank-sharded partials, one all-reduce
        run = lambda objs, outputs=("p", "q", "s"): grp.rhs_host(objs, n, outputs=outputs)  # noqa: E731
        units = [k for _, k in items]
    else:
        ctx = get_context()
        run = lambda dks, outputs=("p", "q", "s"): ctx.rhs_host(dks, n, outputs=outputs)  # noqa: E731
        units = [ctx.device_kernel(k) for _, k in items]
    if not breakdown:
        out = run(units)
        return RhsResult(p=out["p"], q=out["q"], s=out["s"], by_order=None)
    p = np.zeros(n.size)
    q = np.zeros(n.size)
    per = {}
    for (d, _), u in zip(items, units):
        out = run([u], outputs=("p", "q"))
        p += out["p"]
        q += out["q"]
        per[d] = (out["p"], out["q"])
    return RhsResult(p=p, q=q, s=p + q, by_order=per)


def inverse_factorial(d: int) -> float:
    return 1.0 / math.factorial(d)
