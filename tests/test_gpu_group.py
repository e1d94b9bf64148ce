"""Device groups (ttagg_group_*, use_devices): the single-process multi-GPU
path.  This pool's boxes have one GPU, so the group here has one device —
with its NCCL communicator forced on (TTAGG_GROUP_NCCL=1), so the dlopen'ed
NCCL, the per-RHS all-reduce, the sharded upload table and the group RK2 all
run; the rank-shard arithmetic itself (partials summing to the full RHS) is
covered by test_gpu_parity.py::test_rank_shards_sum_to_full_rhs and, at world
size 2, by tests/test_dist_cpu.py."""

import os

import numpy as np
import pytest

import paper_1905_09071_b200 as g
from conftest import rel_inf
from oracle import rhs_oracle as orc
from paper_1905_09071_b200 import _lib
from paper_1905_09071_b200.workloads import CONFIGS, initial_state, permutation_power_cp

pytestmark = pytest.mark.gpu


@pytest.fixture
def group():
    old = os.environ.get("TTAGG_GROUP_NCCL")
    os.environ["TTAGG_GROUP_NCCL"] = "1"
    try:
        grp = g.use_devices([0])
        yield grp
    finally:
        g.use_devices(None)
        if old is None:
            os.environ.pop("TTAGG_GROUP_NCCL", None)
        else:
            os.environ["TTAGG_GROUP_NCCL"] = old


def _c5_set(N):
    exps = CONFIGS["C5"].exponents
    return g.KernelSet({d: g.CPKernel(permutation_power_cp(exps[:d], N)) for d in (2, 3, 4, 5)})


def test_group_rhs_total_matches_single_device(group):
    N = 1 << 20
    ks = _c5_set(N)
    st = g.ConcentrationState(initial_state("c5", N))
    got = g.rhs_total(ks, st)
    g.use_devices(None)
    ref = g.rhs_total(ks, st)
    for a, b in ((got.p, ref.p), (got.q, ref.q), (got.s, ref.s)):
        np.testing.assert_array_equal(a, b)


def test_group_operators_and_mixed_set_vs_oracle(group):
    N = 3001
    rng = np.random.default_rng(1)
    i = np.arange(1, N + 1, dtype=np.float64)
    tt2 = g.TTKernel((np.stack([i ** (2 / 3), 2 * i ** (1 / 3), np.ones(N)], axis=1)[None],
                      np.stack([np.ones(N), i ** (1 / 3), i ** (2 / 3)], axis=0)[:, :, None]))
    cp3 = g.CPKernel(permutation_power_cp((0.1, -0.1, 0.05), N))
    ks = g.KernelSet({2: tt2, 3: cp3})
    n = rng.random(N) * np.exp(-i / 300.0)
    st = g.ConcentrationState(n)
    res = g.rhs_total(ks, st)
    p_ref, q_ref, s_ref = orc.rhs_total({2: tt2, 3: cp3}, n)
    assert rel_inf(res.p, p_ref) <= 1e-10
    assert rel_inf(res.q, q_ref) <= 1e-10
    assert rel_inf(res.s, s_ref) <= 1e-10
    assert rel_inf(g.rhs_cp_P(cp3, st), orc.cp_gain(cp3.factors, n)) <= 1e-10
    assert rel_inf(g.rhs_tt_Q(tt2, st), orc.tt_loss(tt2.cores, n)) <= 1e-10
    br = g.rhs_total(ks, st, breakdown=True)
    assert rel_inf(br.s, s_ref) <= 1e-10


def test_group_rk2_matches_single_device_fused_rk2(group):
    N = 1 << 16
    ks = _c5_set(N)
    n0 = initial_state("c5", N, normalised=True)
    objs = [ks[d] for d in ks.orders]
    gn, grec, gfail, gneg = group.rk2_host(objs, n0, 0.0, 2e-3, 20, 5)
    ctx = _lib.get_context()
    sn, srec, sfail, sneg = ctx.rk2_host([ctx.device_kernel(k) for k in objs], n0, 0.0, 2e-3, 20, 5)
    assert (gfail, gneg) == (sfail, sneg) == (0, 0)
    assert rel_inf(gn, sn) <= 1e-13
    np.testing.assert_allclose(grec, srec, rtol=1e-12, atol=0)
    ref_n, _, _ = orc.integrate({d: ks[d] for d in ks.orders}, n0, dt=2e-3, steps=20)
    assert rel_inf(gn, ref_n) <= 1e-10


def test_group_integrate_matches_single_device(group):
    """integrate() through the group (records every 2 steps) against the
    single-device fused run."""
    cfg = CONFIGS["C3"]
    N = 1 << 12
    ks = g.KernelSet({d: g.CPKernel(f) for d, f in cfg.cp_factors(N).items()})

    class Cfg:
        n_classes = N
        record_every = 2

        class initial:
            @staticmethod
            def state(n_classes, t0):
                return g.ConcentrationState(initial_state("exp256", n_classes, normalised=True), t0)

        time = g.TimeGrid(t0=0.0, dt=cfg.dt, steps=10)

    st, series = g.integrate(Cfg, kernels=ks)
    g.use_devices(None)
    st1, series1 = g.integrate(Cfg, kernels=ks)
    assert rel_inf(st.n, st1.n) <= 1e-13
    assert len(series.times) == len(series1.times) == 6
    np.testing.assert_allclose(series.m1, series1.m1, rtol=1e-12)


def test_group_rejects_duplicate_devices():
    from paper_1905_09071_b200.kernels import KernelError

    with pytest.raises(KernelError, match="twice"):
        _lib.Group([0, 0])
