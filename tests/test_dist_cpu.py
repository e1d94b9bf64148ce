"""Multi-GPU host logic on CPU: rank sharding + all-reduce + replicated RK2
stage updates (paper_1905_09071_b200.dist), world size 2 over gloo, with the
oracle standing in for the CUDA engine (test double, never the product)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import rel_inf
from oracle import rhs_oracle as orc
from paper_1905_09071_b200.dist import (DistRHS, ideal_speedup, rank_counts_of, shard_for_rank,
                                         tt_shard_for_rank)
from paper_1905_09071_b200.parallel import lpt_rank_shards
from paper_1905_09071_b200.workloads import permutation_power_cp


class OracleEngine:
    """CPU test double of dist.CudaEngine (natural layout torch tensors)."""

    def __init__(self, factors_by_order, shard, n_classes, tt_cores=None):
        self.f = factors_by_order
        self.shard = shard
        self.n_classes = n_classes
        self.tt = tt_cores or {}
        self._diag = np.zeros((2, 6))

    def vector(self):
        return torch.zeros(self.n_classes, dtype=torch.float64)

    def to_layout(self, n):
        return torch.from_numpy(np.array(n, dtype=np.float64))

    def from_layout(self, v):
        return v.numpy().copy()

    def partial(self, n, k, alpha, out):
        x = n.numpy() if k is None else (n + alpha * k).numpy()
        acc = np.zeros(self.n_classes)
        for d in sorted(self.f):
            sub = self.shard.get(d, [])
            if sub:
                acc += orc.cp_gain(self.f[d], x, ranks=sub)
                acc += orc.cp_loss(self.f[d], x, ranks=sub)
        for d in sorted(self.tt):
            acc += orc.tt_gain(self.tt[d], x)
            acc += orc.tt_loss(self.tt[d], x)
        out.copy_(torch.from_numpy(acc))

    def stage(self, base, s, a, out, slot=0, row=None):
        v = (base + a * s).numpy()
        k = np.arange(1, v.size + 1, dtype=np.float64)
        if out is not None:
            out.copy_(torch.from_numpy(v))
        d = np.array([0.0 if np.all(np.isfinite(v)) else 1.0, v.min(), np.abs(v).max(),
                      v.sum(), k @ v, (k * k) @ v])
        if row is None:
            self._diag[slot] = d
        else:
            self._hist[row, slot] = d

    def diags(self):
        return self._diag.copy()

    def diag_history(self, rows):
        self._hist = np.zeros((rows, 2, 6))

    def read_history(self, rows):
        return self._hist[:rows].copy()

    def copy(self, v):
        return v.clone()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        N = 300
        exps = (0.1, -0.1, 0.05, -0.05, 0.0)
        f = {d: permutation_power_cp(exps[:d], N) for d in (2, 3, 4, 5)}
        shard = shard_for_rank(rank_counts_of(f), world, rank)
        rng = np.random.default_rng(3)
        n0 = np.exp(-np.arange(1, N + 1) / 40.0) * (1 + 0.05 * rng.random(N))
        n0 = n0 / n0.sum()
        drhs = DistRHS(OracleEngine(f, shard, N))
        s = drhs.rhs(torch.from_numpy(n0.copy()))
        res = drhs.rk2(n0, 0.0, 0.002, 4, record_every=2)
        q.put((rank, s.numpy(), res.n, res.rows, res.fail_step, {d: list(v) for d, v in shard.items()}))
    finally:
        dist.destroy_process_group()


def test_world2_sharded_rhs_and_rk2_match_unsharded_oracle():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    out.sort(key=lambda x: x[0])
    N = 300
    exps = (0.1, -0.1, 0.05, -0.05, 0.0)
    f = {d: permutation_power_cp(exps[:d], N) for d in (2, 3, 4, 5)}
    rng = np.random.default_rng(3)
    n0 = np.exp(-np.arange(1, N + 1) / 40.0) * (1 + 0.05 * rng.random(N))
    n0 = n0 / n0.sum()
    ks = {d: {"kind": "cp", "arrays": v} for d, v in f.items()}
    s_ref = orc.rhs_total(ks, n0)[2]
    n_ref, _, series = orc.integrate(ks, n0, dt=0.002, steps=4, record_every=2)
    for rank, s, n, rows, fail, shard in out:
        assert rel_inf(s, s_ref) <= 1e-12
        assert rel_inf(n, n_ref) <= 1e-12
        assert fail == 0
        np.testing.assert_allclose(np.array(rows), np.array(series.rows()), rtol=1e-11, atol=1e-16)
    # replicas stay bitwise identical across ranks (same all-reduced sums, same updates)
    np.testing.assert_array_equal(out[0][2], out[1][2])
    # the two shards partition every order's rank terms
    for d in (2, 3, 4, 5):
        got = sorted(out[0][5].get(d, []) + out[1][5].get(d, []))
        assert got == list(range(len(f[d][0][0])))


def test_lpt_balance_c5():
    """ideal speedups 2.00 / 3.99 / 7.98 at 2 / 4 / 8 GPUs."""
    counts = {2: 2, 3: 6, 4: 24, 5: 120}
    assert ideal_speedup(counts, 1) == pytest.approx(1.0)
    assert ideal_speedup(counts, 2) >= 1.99
    assert ideal_speedup(counts, 4) >= 3.98
    assert ideal_speedup(counts, 8) >= 7.95
    for world in (1, 2, 3, 4, 8):
        shards = lpt_rank_shards(counts, world)
        for d, R in counts.items():
            owned = sorted(r for s in shards for r in s.get(d, []))
            assert owned == list(range(R))
        assert shards == lpt_rank_shards(counts, world)  # deterministic


def _tt_kernels(N):
    rng = np.random.default_rng(11)
    i = np.arange(1, N + 1, dtype=np.float64)
    c1 = np.zeros((1, N, 3))
    c1[0, :, 0], c1[0, :, 1], c1[0, :, 2] = i ** (2 / 3), 2 * i ** (1 / 3), 1.0
    c2 = np.zeros((3, N, 1))
    c2[0, :, 0], c2[1, :, 0], c2[2, :, 0] = 1.0, i ** (1 / 3), i ** (2 / 3)
    t3 = (rng.random((1, N, 4)) + 0.5, rng.random((4, N, 3)) + 0.5, rng.random((3, N, 1)) + 0.5)
    return {2: (c1, c2), 3: t3}


def _tt_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        N = 200
        tt = _tt_kernels(N)
        f = {4: permutation_power_cp((0.1, -0.1, 0.05, 0.0), N)}
        shard = shard_for_rank(rank_counts_of(f), world, rank)
        mine = tt_shard_for_rank(tt, world, rank)
        n0 = np.exp(-np.arange(1, N + 1) / 30.0)
        n0 = n0 / n0.sum()
        drhs = DistRHS(OracleEngine(f, shard, N, tt_cores=mine))
        s = drhs.rhs(torch.from_numpy(n0.copy()))
        res = drhs.rk2(n0, 0.0, 0.002, 3)
        q.put((rank, s.numpy(), res.n))
    finally:
        dist.destroy_process_group()


def test_world2_tt_rank_sharding_matches_unsharded_oracle():
    """TT kernels sliced over their first internal rank (construct.tt_rank_shard)
    plus CP rank shards: the all-reduced partials equal the full RHS."""
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_tt_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    N = 200
    tt = _tt_kernels(N)
    ks = {d: {"kind": "tt", "arrays": v} for d, v in tt.items()}
    ks[4] = {"kind": "cp", "arrays": permutation_power_cp((0.1, -0.1, 0.05, 0.0), N)}
    n0 = np.exp(-np.arange(1, N + 1) / 30.0)
    n0 = n0 / n0.sum()
    s_ref = orc.rhs_total(ks, n0)[2]
    n_ref, _, _ = orc.integrate(ks, n0, dt=0.002, steps=3)
    for _, s, n in out:
        assert rel_inf(s, s_ref) <= 1e-12
        assert rel_inf(n, n_ref) <= 1e-12


def test_chunked_diagnostics_polling_matches_per_step_semantics():
    """DistRHS.rk2 reads the stage diagnostics once per chunk: chunk
    boundaries change nothing, and a failing step inside a chunk is reported
    at the reference's step with the last finite state (oracle integrate,
    integrator.py:207-215)."""
    N = 120
    exps = (0.1, -0.1, 0.05)
    f = {d: permutation_power_cp(exps[:d], N) for d in (2, 3)}
    shard = lpt_rank_shards(rank_counts_of(f), 1)[0]
    n0 = np.exp(-np.arange(1, N + 1) / 15.0)
    n0 = n0 / n0.sum()
    drhs = DistRHS(OracleEngine(f, shard, N))
    a = drhs.rk2(n0, 0.0, 0.01, 10, record_every=2, poll_every=3)
    b = drhs.rk2(n0, 0.0, 0.01, 10, record_every=2, poll_every=64)
    np.testing.assert_array_equal(a.n, b.n)
    assert a.rows == b.rows and a.fail_step == b.fail_step == 0
    kern = {d: {"kind": "cp", "arrays": f[d]} for d in f}
    ref_n, _, _ = orc.integrate(kern, n0, dt=0.01, steps=10)
    assert rel_inf(a.n, ref_n) <= 1e-12
    # a step size that blows up: the oracle raises at some step k
    big = 400.0
    with pytest.raises(orc.OracleStepFailure) as exc:
        orc.integrate(kern, n0, dt=big, steps=40)
    k = exc.value.step_index
    for poll in (1, 3, 64):
        r = drhs.rk2(n0, 0.0, big, 40, poll_every=poll)
        assert r.fail_step == k
        if k > 1:
            ref_last, _, _ = orc.integrate(kern, n0, dt=big, steps=k - 1)
            assert rel_inf(r.n, ref_last) <= 1e-12
