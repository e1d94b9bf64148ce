"""CPU oracle for the Smoluchowski right-hand side — TEST INFRASTRUCTURE ONLY.

This module is a plain numpy/scipy restatement of the reference package's hot
path (``ttagg`` v0.1.0, ``/root/reference/pkg/src/ttagg``).  It exists so the
CUDA path in ``paper_1905_09071_b200`` can be checked; it is never part of the
product.  Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU
baseline / ``--impl reference`` arm may import it.

Parity is PINNED: ``tests/test_oracle.py`` checks every function here against
golden vectors produced by the reference itself (``oracle/make_golden.py``,
committed fixtures under ``tests/golden/``) and against the reference's own
known answers (``test_rhs.py:87-110, 226-232``; the M0 trajectory in
``pkg/demos/out_ternary/m0_vs_time.csv``).

The FFT arithmetic of the reference lives in scipy.fft (pocketfft, vendored in
scipy; version not pinned by the reference, ``pyproject.toml:10``).  This
oracle calls the same scipy.fft routines.

Conventions follow the reference exactly:
* CP factors: ``d`` arrays of shape (N, R), C-contiguous fp64 (kernels.py:191-203)
* TT cores:   ``d`` arrays of shape (R_prev, N, R_next) (kernels.py:145-164)
* size i lives at transform position i (position 0 empty), rhs.py:267, 367
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
import scipy.fft as _fft

__all__ = [
    "fft_length",
    "cp_gain",
    "cp_loss",
    "tt_gain",
    "tt_loss",
    "dense_gain",
    "dense_loss",
    "dense_from_cp",
    "dense_from_tt",
    "rhs_total",
    "OracleSeries",
    "OracleStepFailure",
    "integrate",
    "moments",
]


def fft_length(order: int, n_classes: int, policy: str = "pow2") -> int:
    """Transform length policy — parallel.py:340-344."""
    needed = order * n_classes + 1
    if policy == "min":
        return needed
    return 1 << (needed - 1).bit_length()


def _workers(workers):
    import os

    return max(1, min(int(workers or 1), os.cpu_count() or 1))


# ---------------------------------------------------------------------------
# CP gain / loss — rhs.py:345-414
# ---------------------------------------------------------------------------

def cp_gain(factors, n, *, policy="pow2", workers=1, rank_chunk=None, ranks=None):
    """Gain vector of a CP kernel — restates rhs.py:345-391.

    (1) weight factor columns by n with size i at position i (rhs.py:364-369),
    (2) rfft of every column at the plan length (rhs.py:371), (3) per bin the
    product over modes and the sum over ranks (rhs.py:375-381), (4) one irfft
    (rhs.py:383), (5) p[k-1] = coeffs[k] / d! for k = d..N (rhs.py:387-390).

    ``rank_chunk`` processes the ranks in chunks (bounded memory for the CPU
    baseline at N = 2^20); ``ranks`` restricts the sum to a subset of rank
    indices (the rank-sharded partial gain of one GPU).
    """
    d = len(factors)
    n = np.asarray(n, dtype=np.float64)
    n_classes = n.size
    length = fft_length(d, n_classes, policy)
    all_ranks = np.arange(factors[0].shape[1]) if ranks is None else np.asarray(ranks)
    chunk = all_ranks.size if not rank_chunk else int(rank_chunk)
    w = _workers(workers)
    out_spec = None
    for lo in range(0, all_ranks.size, max(chunk, 1)):
        sel = all_ranks[lo : lo + chunk]
        rank = sel.size
        buf = np.zeros((d * rank, length))
        for mode, factor in enumerate(factors):
            buf[mode * rank : (mode + 1) * rank, 1 : 1 + n_classes] = (
                factor[:, sel] * n[:, None]
            ).T
        spectra = _fft.rfft(buf, axis=1, workers=w)
        del buf
        acc = spectra[0:rank].copy()
        for mode in range(1, d):
            acc *= spectra[mode * rank : (mode + 1) * rank]
        part = acc.sum(axis=0)
        out_spec = part if out_spec is None else out_spec + part
        del spectra, acc
    if out_spec is None:
        out_spec = np.zeros(length // 2 + 1, dtype=np.complex128)
    coeffs = _fft.irfft(out_spec, n=length, workers=w)
    p = np.zeros(n_classes)
    p[d - 1 :] = coeffs[d : n_classes + 1] / math.factorial(d)
    return p


def cp_loss(factors, n, *, ranks=None):
    """Loss vector of a CP kernel — restates rhs.py:394-414.

    s_r = prod_{m<d-1} <F^(m)[:, r], n>;  q = -n * (F^(d-1) @ s) / (d-1)!
    """
    d = len(factors)
    n = np.asarray(n, dtype=np.float64)
    sel = slice(None) if ranks is None else np.asarray(ranks)
    scalars = np.ones(factors[0][:, sel].shape[1])
    for mode in range(d - 1):
        scalars = scalars * (n @ factors[mode][:, sel])
    tail = factors[d - 1][:, sel] @ scalars
    return -(n * tail) / math.factorial(d - 1)


# ---------------------------------------------------------------------------
# TT gain / loss — rhs.py:234-338
# ---------------------------------------------------------------------------

def tt_gain(cores, n, *, policy="pow2", workers=1):
    """Gain vector of a TT kernel — restates rhs.py:234-302.

    Buffer row offsets[lam] + rp * R_next + rn holds H^(lam)[rp, :, rn] * n
    (rhs.py:257-269); per bin the 1 x R spectral row vector is chained left to
    right through the R_prev x R_next spectral matrices (rhs.py:277-290).
    """
    d = len(cores)
    n = np.asarray(n, dtype=np.float64)
    n_classes = n.size
    length = fft_length(d, n_classes, policy)
    ranks = (1,) + tuple(c.shape[2] for c in cores)
    rows = [ranks[lam] * ranks[lam + 1] for lam in range(d)]
    offsets = np.concatenate([[0], np.cumsum(rows)]).astype(int)
    buf = np.zeros((int(offsets[-1]), length))
    for lam, core in enumerate(cores):
        block = core * n[None, :, None]
        buf[offsets[lam] : offsets[lam + 1], 1 : 1 + n_classes] = block.transpose(
            0, 2, 1
        ).reshape(rows[lam], n_classes)
    spectra = _fft.rfft(buf, axis=1, workers=_workers(workers))
    del buf
    v = [spectra[offsets[0] + r] for r in range(ranks[1])]
    for lam in range(1, d):
        r_prev, r_next = ranks[lam], ranks[lam + 1]
        base = offsets[lam]
        new = []
        for rn in range(r_next):
            acc = v[0] * spectra[base + rn]
            for rp in range(1, r_prev):
                acc = acc + v[rp] * spectra[base + rp * r_next + rn]
            new.append(acc)
        v = new
    coeffs = _fft.irfft(v[0], n=length, workers=_workers(workers))
    p = np.zeros(n_classes)
    p[d - 1 :] = coeffs[d : n_classes + 1] / math.factorial(d)
    return p


def tt_loss(cores, n):
    """Loss vector of a TT kernel — restates rhs.py:305-338 (_contract_core, rhs_tt_Q)."""
    d = len(cores)
    n = np.asarray(n, dtype=np.float64)
    w = np.einsum("rns,n->rs", cores[0], n)
    for lam in range(1, d - 1):
        w = w @ np.einsum("rns,n->rs", cores[lam], n)
    tail = w[0] @ cores[d - 1][:, :, 0]
    return -(n * tail) / math.factorial(d - 1)


# ---------------------------------------------------------------------------
# dense operators (O(N^d), FFT-free) — rhs.py:202-227
# ---------------------------------------------------------------------------

def dense_from_cp(factors):
    """kernels.py:467-478"""
    values = np.zeros((factors[0].shape[0],) * len(factors))
    for r in range(factors[0].shape[1]):
        term = factors[0][:, r]
        for f in factors[1:]:
            term = np.multiply.outer(term, f[:, r])
        values += term
    return values


def dense_from_tt(cores):
    """kernels.py:456-464"""
    out = cores[0][0]
    for core in cores[1:]:
        out = np.tensordot(out, core, axes=([out.ndim - 1], [0]))
    return out[..., 0]


def dense_gain(values, n):
    """rhs.py:202-217 — bincount over index sums."""
    d = values.ndim
    n = np.asarray(n, dtype=np.float64)
    n_classes = n.size
    weighted = values.copy()
    for axis in range(d):
        shape = [1] * d
        shape[axis] = n_classes
        weighted *= n.reshape(shape)
    sizes = np.arange(1, n_classes + 1)
    grid = sizes
    for _ in range(d - 1):
        grid = np.add.outer(grid, sizes)
    totals = np.bincount(grid.ravel(), weights=weighted.ravel(), minlength=d * n_classes + 1)
    p = np.zeros(n_classes)
    p[d - 1 :] = totals[d : n_classes + 1] / math.factorial(d)
    return p


def dense_loss(values, n):
    """rhs.py:220-227"""
    d = values.ndim
    n = np.asarray(n, dtype=np.float64)
    w = values
    for _ in range(d - 1):
        w = np.tensordot(n, w, axes=(0, 0))
    return -(n * w) / math.factorial(d - 1)


# ---------------------------------------------------------------------------
# combined RHS and RK2 — rhs.py:421-459, integrator.py:141-228
# ---------------------------------------------------------------------------

def _kind(kernel):
    if isinstance(kernel, dict):
        return kernel["kind"], kernel["arrays"]
    if hasattr(kernel, "factors"):
        return "cp", kernel.factors
    if hasattr(kernel, "cores"):
        return "tt", kernel.cores
    if hasattr(kernel, "values"):
        return "dense", kernel.values
    raise TypeError(type(kernel))


def rhs_total(kernels: dict, n, *, policy="pow2", workers=1, breakdown=False):
    """rhs.py:421-459: accumulate p and q over ascending orders; s = p + q."""
    n = np.asarray(n, dtype=np.float64)
    p = np.zeros(n.size)
    q = np.zeros(n.size)
    per = {}
    for d in sorted(kernels):
        kind, arrays = _kind(kernels[d])
        if kind == "cp":
            pd, qd = cp_gain(arrays, n, policy=policy, workers=workers), cp_loss(arrays, n)
        elif kind == "tt":
            pd, qd = tt_gain(arrays, n, policy=policy, workers=workers), tt_loss(arrays, n)
        else:
            pd, qd = dense_gain(arrays, n), dense_loss(arrays, n)
        p += pd
        q += qd
        if breakdown:
            per[d] = (pd, qd)
    return (p, q, p + q, per) if breakdown else (p, q, p + q)


def moments(n, orders=(0, 1, 2)):
    """integrator.py:141-150"""
    sizes = np.arange(1, n.size + 1, dtype=np.float64)
    return [float((sizes**m) @ n) for m in orders]


class OracleStepFailure(RuntimeError):
    """integrator.py:34-44 — non-finite step; carries step index and series."""

    def __init__(self, msg, step_index=None, series=None):
        super().__init__(msg)
        self.step_index = step_index
        self.series = series


@dataclass
class OracleSeries:
    """integrator.py:108-138"""

    times: list = field(default_factory=list)
    m0: list = field(default_factory=list)
    m1: list = field(default_factory=list)
    m2: list = field(default_factory=list)
    min_n: list = field(default_factory=list)
    m1_drift: list = field(default_factory=list)
    negativity_flagged: bool = False

    def record(self, t, n):
        m = moments(n)
        self.times.append(float(t))
        self.m0.append(m[0])
        self.m1.append(m[1])
        self.m2.append(m[2])
        self.min_n.append(float(n.min()))
        ref = self.m1[0]
        self.m1_drift.append((m[1] - ref) / ref if ref else 0.0)

    def rows(self):
        return list(zip(self.times, self.m0, self.m1, self.m2, self.min_n))

    def __len__(self):
        return len(self.times)


def integrate(kernels: dict, n0, *, t0=0.0, dt, steps, record_every=1,
              policy="pow2", workers=1):
    """integrator.py:153-228: explicit midpoint RK2 with moment records.

    k1 = S(n); k2 = S(n + dt/2 k1); n' = n + dt k2 (integrator.py:153-157);
    a non-finite state aborts with the partial series (integrator.py:177, 207-215);
    min(n) < -1e-9 max|n| sets the negativity flag (integrator.py:216-223).
    """
    n = np.array(n0, dtype=np.float64)
    t = float(t0)
    series = OracleSeries()
    series.record(t, n)
    for step in range(1, steps + 1):
        def S(x):
            if not np.all(np.isfinite(x)):
                raise ValueError("concentration state contains non-finite entries")
            return rhs_total(kernels, x, policy=policy, workers=workers)[2]
        try:
            k1 = S(n)
            k2 = S(n + (0.5 * dt) * k1)
            n_new = n + dt * k2
            if not np.all(np.isfinite(n_new)):
                raise ValueError("time step produced non-finite concentrations")
        except ValueError as exc:
            raise OracleStepFailure(
                f"integration aborted at step {step}: {exc}", step_index=step, series=series
            ) from exc
        n = n_new
        t = t + dt
        if float(n.min()) < -1e-9 * float(np.abs(n).max()):
            series.negativity_flagged = True
        if step % record_every == 0:
            series.record(t, n)
    return n, t, series
