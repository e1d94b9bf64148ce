"""GPU parity for TT kernels with zero structure: the upload drops all-zero
fibers and fibers on chain paths that are zero (dead input state or unused
output state); gain and loss must still match the oracle, which evaluates
every fiber (rhs.py:234-338).  The reference's own exact Brownian TT
(kernels.py:332-363) is mostly such zeros."""

import itertools
import math

import numpy as np
import pytest

import paper_1905_09071_b200 as g
from conftest import rel_inf
from oracle import rhs_oracle as orc
from paper_1905_09071_b200 import _lib
from paper_1905_09071_b200.workloads import permutation_power_cp

pytestmark = pytest.mark.gpu
TOL = 1e-10


def st(n):
    return g.ConcentrationState(n)


def subset_tt(exponents, n_classes):
    """Subset-structured TT of the permutation-power kernel (the construction
    of build_brownian_tt, kernels.py:332-363): rank index at level lam = a
    lam-subset of exponent labels, fiber S -> T the power vector of T \\ S."""
    d = len(exponents)
    i = np.arange(1, n_classes + 1, dtype=np.float64)
    pows = [i ** a for a in exponents]
    levels = [list(itertools.combinations(range(d), k)) for k in range(d + 1)]
    index = [{s: r for r, s in enumerate(lv)} for lv in levels]
    cores = []
    for lam in range(1, d + 1):
        core = np.zeros((len(levels[lam - 1]), n_classes, len(levels[lam])))
        for rc, T in enumerate(levels[lam]):
            for label in T:
                S = tuple(x for x in T if x != label)
                core[index[lam - 1][S], :, rc] = pows[label]
        cores.append(core)
    return tuple(cores)


def uploaded_columns(kernel):
    return _lib.get_context().device_kernel(kernel).info()[3]


@pytest.mark.parametrize("n_classes", [4096, 1 << 17])
@pytest.mark.parametrize("order", [2, 3, 4, 5])
def test_subset_tt_vs_cp_route(n_classes, order):
    a = (0.1, -0.1, 0.05, -0.05, 0.0)[:order]
    rng = np.random.default_rng(order)
    n = np.exp(-np.arange(n_classes) / 512.0) * (1 + 0.05 * rng.random(n_classes))
    tt = g.TTKernel(subset_tt(a, n_classes))
    cp = g.CPKernel(permutation_power_cp(a, n_classes))
    # only the d 2^(d-1) nonzero fibers travel (of sum C(d,l-1) C(d,l))
    assert uploaded_columns(tt) == order * 2 ** (order - 1)
    assert rel_inf(g.rhs_tt_P(tt, st(n)), g.rhs_cp_P(cp, st(n))) <= TOL
    assert rel_inf(g.rhs_tt_Q(tt, st(n)), g.rhs_cp_Q(cp, st(n))) <= TOL
    if n_classes <= 4096:
        assert rel_inf(g.rhs_tt_P(tt, st(n)), orc.tt_gain(tt.cores, n)) <= TOL
        assert rel_inf(g.rhs_tt_Q(tt, st(n)), orc.tt_loss(tt.cores, n)) <= TOL


def _random_cores(rng, ranks, n_classes):
    return [rng.random((ranks[l], n_classes, ranks[l + 1])) for l in range(len(ranks) - 1)]


@pytest.mark.parametrize("n_classes", [1000, 1 << 17])
def test_dead_chain_paths_vs_oracle(n_classes):
    rng = np.random.default_rng(11)
    ranks = (1, 4, 5, 3, 1)
    cores = _random_cores(rng, ranks, n_classes)
    cores[0][0, :, 1] = 0.0          # state (1, 1) has no input: its outgoing fibers drop too
    cores[1][:, :, 2] = 0.0          # state (2, 2) has no input
    cores[2][3, :, :] = 0.0          # state (2, 3) feeds nothing: its incoming fibers drop
    cores[1][0, :, 4] = 0.0          # a single zero fiber
    cores[2][1, : n_classes // 2, 0] = 0.0  # partly zero: stays
    cores = tuple(cores)
    n = rng.random(n_classes)
    k = g.TTKernel(cores)
    full = sum(ranks[l] * ranks[l + 1] for l in range(4))
    assert uploaded_columns(k) < full
    assert rel_inf(g.rhs_tt_P(k, st(n)), orc.tt_gain(cores, n)) <= TOL
    assert rel_inf(g.rhs_tt_Q(k, st(n)), orc.tt_loss(cores, n)) <= TOL


def test_all_zero_tt_kernel_is_exactly_zero():
    n_classes = 5000
    cores = (np.zeros((1, n_classes, 3)), np.zeros((3, n_classes, 2)), np.zeros((2, n_classes, 1)))
    n = np.random.default_rng(2).random(n_classes)
    k = g.TTKernel(cores)
    assert np.all(g.rhs_tt_P(k, st(n)) == 0.0)
    assert np.all(g.rhs_tt_Q(k, st(n)) == 0.0)


def test_subset_tt_set_matches_cp_set_in_total():
    """The C5 tensor at reduced N through both routes in one KernelSet call."""
    n_classes = 1 << 16
    ex = (0.1, -0.1, 0.05, -0.05, 0.0)
    n = np.exp(-np.arange(n_classes) / 1024.0)
    ks_tt = g.KernelSet({d: g.TTKernel(subset_tt(ex[:d], n_classes)) for d in range(2, 6)})
    ks_cp = g.KernelSet({d: g.CPKernel(permutation_power_cp(ex[:d], n_classes)) for d in range(2, 6)})
    a = g.rhs_total(ks_tt, st(n))
    b = g.rhs_total(ks_cp, st(n))
    assert rel_inf(a.s, b.s) <= TOL
    assert math.isfinite(float(np.abs(a.s).max()))


@pytest.mark.parametrize("ranks", [(1, 64, 1), (1, 3, 64, 2, 1), (1, 64, 64, 1)])
def test_tt_max_ranks_vs_oracle(ranks):
    """The largest TT ranks the build takes (64): chain state and loss chain."""
    n_classes = 3000
    rng = np.random.default_rng(sum(ranks))
    cores = tuple(rng.random((ranks[l], n_classes, ranks[l + 1])) / ranks[l] for l in range(len(ranks) - 1))
    n = rng.random(n_classes)
    k = g.TTKernel(cores)
    assert rel_inf(g.rhs_tt_P(k, st(n)), orc.tt_gain(cores, n)) <= TOL
    assert rel_inf(g.rhs_tt_Q(k, st(n)), orc.tt_loss(cores, n)) <= TOL


def test_tt_rank_above_64_is_rejected():
    cores = (np.ones((1, 16, 65)), np.ones((65, 16, 1)))
    with pytest.raises(Exception, match="64"):
        g.rhs_tt_P(g.TTKernel(cores), st(np.ones(16)))
