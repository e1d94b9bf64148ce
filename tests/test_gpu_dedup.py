"""Opt-in identical-column deduplication (ttagg_cp_upload_dedup,
SURVEY.md §8(f)2): the same RHS as the plain upload — bitwise, since every
stored pair is transformed exactly as before and pass B walks the same
rank/mode structure — and the same as the oracle within the per-RHS
tolerance, at full size and on ragged / partially duplicated kernels."""

import numpy as np
import pytest

import paper_1905_09071_b200 as g
from conftest import rel_inf
from oracle import rhs_oracle as orc
from paper_1905_09071_b200 import _lib
from paper_1905_09071_b200.workloads import CONFIGS, initial_state, permutation_power_cp

pytestmark = pytest.mark.gpu
TOL = 1e-10


def _rhs(ctx, dks, n):
    r = ctx.rhs_host(dks, n)
    return [r["p"].copy(), r["q"].copy(), r["s"].copy()]


def test_c5_full_size_dedup_matches_plain_upload():
    ctx = _lib.get_context()
    N = 1 << 20
    exps = CONFIGS["C5"].exponents
    n = initial_state("c5", N)
    plain, dedup = [], []
    for d in (2, 3, 4, 5):
        f = permutation_power_cp(exps[:d], N)
        plain.append(ctx.upload_cp(f))
        dedup.append(ctx.upload_cp(f, dedup=True))
    a = _rhs(ctx, plain, n)
    b = _rhs(ctx, dedup, n)
    for x, y in zip(a, b):
        np.testing.assert_array_equal(x, y)


@pytest.mark.parametrize("N", [37, 1000, 4099])
def test_partially_duplicated_random_cp_vs_oracle(N):
    rng = np.random.default_rng(N)
    ctx = _lib.get_context()
    R = 7
    base = [rng.random((N, R)) for _ in range(3)]
    # duplicate some columns across factors and ranks
    base[1][:, 2] = base[0][:, 5]
    base[2][:, 0] = base[0][:, 5]
    base[2][:, 4] = base[1][:, 4]
    base[0][:, 6] = base[0][:, 1]
    n = rng.random(N) * np.exp(-np.arange(N) / (N / 4))
    dk_plain = ctx.upload_cp(base)
    dk_dedup = ctx.upload_cp(base, dedup=True)
    a = _rhs(ctx, [dk_plain], n)
    b = _rhs(ctx, [dk_dedup], n)
    for x, y in zip(a, b):
        np.testing.assert_array_equal(x, y)
    p_ref, q_ref, s_ref = orc.rhs_total({3: {"kind": "cp", "arrays": base}}, n)
    assert rel_inf(b[0], p_ref) <= TOL
    assert rel_inf(b[1], q_ref) <= TOL
    assert rel_inf(b[2], s_ref) <= TOL


def test_dedup_rank_shards_sum_to_full():
    ctx = _lib.get_context()
    N = 1 << 14
    f = permutation_power_cp(CONFIGS["C5"].exponents, N)
    n = initial_state("c5", N)
    full = _rhs(ctx, [ctx.upload_cp(f, dedup=True)], n)[2]
    parts = [ctx.upload_cp(f, rank_subset=list(range(k, 120, 3)), dedup=True) for k in range(3)]
    total = sum(_rhs(ctx, [p], n)[2] for p in parts)
    assert rel_inf(total, full) <= 1e-12


def test_public_switch_and_fused_rk2():
    N = 1 << 16
    exps = CONFIGS["C5"].exponents
    n0 = initial_state("c5", N, normalised=True)
    ks = g.KernelSet({d: g.CPKernel(permutation_power_cp(exps[:d], N)) for d in (2, 3, 4, 5)})
    ctx = _lib.get_context()
    plain = ctx.rk2_host([ctx.device_kernel(ks[d]) for d in ks.orders], n0, 0.0, 2e-3, 5, 1)
    prev = g.dedup_identical_columns(True)
    try:
        res = g.rhs_total(ks, g.ConcentrationState(n0))
        dd = ctx.rk2_host([ctx.device_kernel(ks[d]) for d in ks.orders], n0, 0.0, 2e-3, 5, 1)
    finally:
        g.dedup_identical_columns(prev)
    base = g.rhs_total(ks, g.ConcentrationState(n0))
    np.testing.assert_array_equal(res.s, base.s)
    np.testing.assert_array_equal(plain[0], dd[0])
    np.testing.assert_array_equal(plain[1], dd[1])
