"""Rank-sharded RHS and RK2 across GPUs.

One process per GPU (torch.distributed, NCCL over NVLink).  Every GPU owns a
subset of the CP rank terms (LPT balanced on cost ~ d^2), evaluates its
partial dn/dt — gains through its own inverse transforms, losses through its
own rank scalars, both linear in the rank sum — and one all-reduce(sum) of
the length-N partial per RHS completes dn/dt on every rank.  Every rank then
applies the identical RK2 stage update to its replica of n.

The arithmetic is done by an *engine*; the default is the CUDA extension
(perm-layout device tensors).  Tests inject a CPU engine built on the oracle
to exercise exactly this orchestration under a gloo world of size 2.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from .parallel import lpt_rank_shards

__all__ = ["shard_for_rank", "tt_shard_for_rank", "CudaEngine", "DistRK2Result", "DistRHS"]


def shard_for_rank(rank_counts: dict, world: int, rank: int) -> dict:
    """{d: [rank indices]} owned by `rank` (deterministic LPT)."""
    return lpt_rank_shards(rank_counts, world)[rank]


def tt_shard_for_rank(tt_by_order: dict, world: int, rank: int) -> dict:
    """{d: cores sliced to this rank's share of the first internal TT rank}.

    Gain and loss are linear in that index (rhs.py:277-290, 305-338), so the
    partial RHS of all ranks sums to the full one; orders whose first rank is
    smaller than the world leave some ranks without a slice."""
    from .construct import tt_rank_shard

    out = {}
    for d, cores in tt_by_order.items():
        sl = tt_rank_shard(cores, world, rank)
        if sl is not None:
            out[d] = sl
    return out


class CudaEngine:
    """Partial RHS + stage updates on this process's GPU (perm layout).

    ``factors_by_order`` / ``shard``: CP factors and this rank's CP rank terms;
    ``tt_cores``: TT kernels already sliced by :func:`tt_shard_for_rank`."""

    def __init__(self, factors_by_order: dict, shard: dict, n_classes: int, device: int,
                 tt_cores: dict | None = None):
        import torch

        from ._lib import geometry, get_context

        self.torch = torch
        self.ctx = get_context(device)
        self.device = torch.device("cuda", device)
        self.n_classes = n_classes
        self.Np, _, _ = geometry(n_classes)
        self.dks = []
        for d in sorted(factors_by_order):
            sub = shard.get(d, [])
            if sub:
                self.dks.append(self.ctx.upload_cp(factors_by_order[d], rank_subset=sub))
        for d in sorted(tt_cores or {}):
            self.dks.append(self.ctx.upload_tt(tt_cores[d]))
        self.diag = torch.zeros((2, 8), dtype=torch.float64, device=self.device)

    def vector(self):
        return self.torch.zeros(self.Np, dtype=self.torch.float64, device=self.device)

    def to_layout(self, n: np.ndarray):
        t = self.torch.from_numpy(np.ascontiguousarray(n, dtype=np.float64)).to(self.device)
        out = self.vector()
        self.ctx.permute(self.n_classes, t.data_ptr(), out.data_ptr(), 0, self._stream())
        return out

    def from_layout(self, v) -> np.ndarray:
        out = self.torch.empty(self.n_classes, dtype=self.torch.float64, device=self.device)
        self.ctx.permute(self.n_classes, v.data_ptr(), out.data_ptr(), 1, self._stream())
        return out.cpu().numpy()

    def _stream(self):
        return self.torch.cuda.current_stream(self.device).cuda_stream

    def partial(self, n, k, alpha, out):
        """out = partial RHS at n + alpha k over this rank's terms."""
        if self.dks:
            self.ctx.rhs_perm(self.dks, n.data_ptr(), None if k is None else k.data_ptr(), alpha,
                              out.data_ptr(), self._stream())
        else:
            out.zero_()

    def stage(self, base, s, a, out, slot=0, row=None):
        """out = base + a s; diagnostics (nonfinite, min, max|.|, M0, M1, M2)
        stay on the device — in `slot` of :meth:`diags`, or in row `row` of
        the history (:meth:`diag_history`) — until read."""
        d = self.diag[slot] if row is None else self.hist[row, slot]
        self.ctx.stage(self.n_classes, base.data_ptr(), s.data_ptr(), a,
                       None if out is None else out.data_ptr(), d.data_ptr(), self._stream())

    def diags(self) -> np.ndarray:
        """Both diagnostic slots in one device-to-host read: (2, 6)."""
        return self.diag.cpu().numpy()[:, :6]

    def diag_history(self, rows: int):
        """Device rows for the diagnostics of `rows` steps (2 stages each)."""
        self.hist = self.torch.zeros((rows, 2, 8), dtype=self.torch.float64, device=self.device)

    def read_history(self, rows: int) -> np.ndarray:
        """The first `rows` history rows in one device-to-host read: (rows, 2, 6)."""
        return self.hist[:rows].cpu().numpy()[:, :, :6]

    def copy(self, v):
        return v.clone()


@dataclass
class DistRK2Result:
    n: np.ndarray
    rows: list = field(default_factory=list)  # (t, M0, M1, M2, min_n)
    fail_step: int = 0
    neg_step: int = 0


class DistRHS:
    """All-reduced RHS and midpoint RK2 over a torch.distributed group."""

    def __init__(self, engine, group=None):
        import torch.distributed as dist

        self.engine = engine
        self.dist = dist
        self.group = group

    def allreduce(self, v):
        if self.dist.is_initialized() and self.dist.get_world_size(self.group) > 1:
            self.dist.all_reduce(v, group=self.group)
        return v

    def rhs(self, n, k=None, alpha=0.0, out=None):
        out = self.engine.vector() if out is None else out
        self.engine.partial(n, k, alpha, out)
        return self.allreduce(out)

    def rk2(self, n0: np.ndarray, t0: float, dt: float, steps: int, record_every: int = 1,
            poll_every: int = 64) -> DistRK2Result:
        """Explicit midpoint (integrator.py:153-228) with the state resident on the device:
        k1 = S(n); mid = n + dt/2 k1; k2 = S(mid); n <- n + dt k2 (all-reduce per S).

        The stage diagnostics of each step stay on the device and are read
        once every `poll_every` steps (one host sync per chunk, not per
        step); a failing step found in a chunk is re-located by replaying the
        chunk from its saved first state, so the returned state is the last
        finite one, as in the per-step loop."""
        if not dt > 0:
            raise ValueError("dt must be positive")
        e = self.engine
        n = e.to_layout(n0)
        s = e.vector()
        mid = e.vector()
        nxt = e.vector()
        zero = e.vector()
        e.stage(n, zero, 0.0, None, 0)
        d0 = e.diags()[0]  # diagnostics of the initial state
        res = DistRK2Result(n=np.asarray(n0))
        res.rows.append((float(t0), float(d0[3]), float(d0[4]), float(d0[5]), float(d0[1])))
        K = max(1, min(poll_every, steps))
        e.diag_history(K)

        def one_step(row):
            nonlocal n, nxt
            self.rhs(n, out=s)
            e.stage(n, s, 0.5 * dt, mid, 0, row)
            self.rhs(mid, out=s)
            e.stage(n, s, dt, nxt, 1, row)
            n, nxt = nxt, n

        t = float(t0)
        step = 0
        while step < steps:
            first = e.copy(n)
            count = min(K, steps - step)
            for j in range(count):
                one_step(j)
            hist = e.read_history(count)  # one host sync per chunk
            for j in range(count):
                dm, dn = hist[j]
                stp = step + j + 1
                if dm[0] != 0.0 or dn[0] != 0.0:
                    res.fail_step = stp
                    n = first  # replay up to the last finite state
                    for jj in range(j):
                        one_step(jj)
                    break
                t = t + dt
                if res.neg_step == 0 and dn[1] < -1e-9 * dn[2]:
                    res.neg_step = stp
                if stp % record_every == 0:
                    res.rows.append((t, float(dn[3]), float(dn[4]), float(dn[5]), float(dn[1])))
            if res.fail_step:
                break
            step += count
        res.n = e.from_layout(n)
        return res


def rank_counts_of(factors_by_order: dict) -> dict:
    return {d: f[0].shape[1] for d, f in factors_by_order.items()}


def ideal_speedup(rank_counts: dict, world: int) -> float:
    """LPT makespan ratio (2.00/3.99/7.98 at 2/4/8 for C5)."""
    shards = lpt_rank_shards(rank_counts, world)
    total = sum(int(d) ** 2 * R for d, R in rank_counts.items())
    worst = max(sum(int(d) ** 2 * len(v) for d, v in s.items()) for s in shards)
    return total / worst if worst else math.inf
