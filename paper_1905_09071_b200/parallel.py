"""Execution plan — signature-compatible with ``ttagg.parallel.ExecutionPlan``
(parallel.py:310-359) and the rank sharding used across GPUs.

On the GPU the CPU thread-pool knobs (workers, parallel_fft, parallel_blocks)
have no meaning and are accepted for compatibility only.  The transform
length is always L = d * Np with Np = the padded size count; both reference
policies ("pow2": next power of two >= dN+1, "min": dN+1) agree with it to
roundoff because every length >= dN - d + 1 is alias-free for sizes <= N
(pinned by test_rhs.py:360-366).
"""

from __future__ import annotations

import heapq
from dataclasses import dataclass

from .kernels import KernelError

__all__ = ["ExecutionPlan", "SERIAL_PLAN", "lpt_rank_shards"]


@dataclass(frozen=True)
class ExecutionPlan:
    workers: int = 1
    fft_length_policy: str = "pow2"
    parallel_fft: bool = True
    parallel_blocks: bool = True
    deterministic_reduction: bool = True

    def __post_init__(self):
        if self.workers < 1:
            raise KernelError("worker count must be >= 1")
        if self.fft_length_policy not in ("pow2", "min"):
            raise KernelError(f"unknown fft_length_policy {self.fft_length_policy!r}")

    def fft_length(self, order: int, n_classes: int) -> int:
        """The reference's CPU transform length (parallel.py:340-344), kept for callers."""
        needed = order * n_classes + 1
        if self.fft_length_policy == "min":
            return needed
        return 1 << (needed - 1).bit_length()


SERIAL_PLAN = ExecutionPlan()


def lpt_rank_shards(rank_counts: dict, world: int) -> list[dict]:
    """Longest-processing-time assignment of CP rank terms (d, r) to `world` GPUs.

    Cost of one rank term of order d ~ d columns x transform length d*N,
    i.e. proportional to d^2.  Returns, per GPU, a dict
    {d: [rank indices]} (sorted).  Deterministic: ties break on (d, r, gpu).
    """
    items = []
    for d, R in rank_counts.items():
        for r in range(int(R)):
            items.append((-(int(d) ** 2), int(d), r))
    items.sort()
    heap = [(0, g) for g in range(world)]
    heapq.heapify(heap)
    out = [dict() for _ in range(world)]
    for negcost, d, r in items:
        load, g = heapq.heappop(heap)
        out[g].setdefault(d, []).append(r)
        heapq.heappush(heap, (load - negcost, g))
    for g in range(world):
        for d in out[g]:
            out[g][d].sort()
    return out
