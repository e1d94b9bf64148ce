"""GPU parity of the direct-summation (dense) operators rhs_dense_P /
rhs_dense_Q (rhs.py:202-227) against the reference's own outputs (golden
dense.npz: TableSpec and Brownian dense kernels, a mixed KernelSet) and the
oracle; dense orders inside rhs_total and the fused RK2 integrator."""

import numpy as np
import pytest

import paper_1905_09071_b200 as g
from conftest import rel_inf
from oracle import rhs_oracle as orc
from paper_1905_09071_b200.workloads import permutation_power_cp

pytestmark = pytest.mark.gpu
TOL = 1e-10


def st(n):
    return g.ConcentrationState(n)


@pytest.mark.parametrize("tag", ["d2", "d3", "d4", "d5", "brown3"])
def test_dense_vs_reference(golden, tag):
    c = golden("dense.npz")
    k = g.DenseKernel(c[f"{tag}_values"])
    n = c[f"{tag}_n"]
    assert rel_inf(g.rhs_dense_P(k, st(n)), c[f"{tag}_P"]) <= TOL
    assert rel_inf(g.rhs_dense_Q(k, st(n)), c[f"{tag}_Q"]) <= TOL


def test_dense_mixed_set_vs_reference(golden):
    c = golden("dense.npz")
    n = c["brown3_n"]
    N = n.size
    ks = g.KernelSet({2: g.DenseKernel(c["d2_values"][:N, :N].copy()), 3: g.DenseKernel(c["brown3_values"])})
    r = g.rhs_total(ks, st(n))
    assert rel_inf(r.p, c["mix_p"]) <= TOL and rel_inf(r.q, c["mix_q"]) <= TOL and rel_inf(r.s, c["mix_s"]) <= TOL


@pytest.mark.parametrize("order,n_classes", [(2, 8192), (2, 1000), (3, 400), (4, 64), (6, 16), (8, 9)])
def test_dense_sizes_vs_oracle(order, n_classes):
    rng = np.random.default_rng(order * 1000 + n_classes)
    v = rng.random((n_classes,) * order)
    n = rng.random(n_classes)
    k = g.DenseKernel(v)
    assert rel_inf(g.rhs_dense_P(k, st(n)), orc.dense_gain(v, n)) <= TOL
    assert rel_inf(g.rhs_dense_Q(k, st(n)), orc.dense_loss(v, n)) <= TOL


def test_dense_matches_cp_route():
    """The same tensor as a dense and as a CP kernel (the reference's own
    cross-check of the FFT paths, test_rhs.py)."""
    N = 300
    fs = permutation_power_cp((0.1, -0.1, 0.05), N)
    dense = orc.dense_from_cp(fs)
    n = np.exp(-np.arange(N) / 50.0)
    cp, dk = g.CPKernel(fs), g.DenseKernel(dense)
    assert rel_inf(g.rhs_dense_P(dk, st(n)), g.rhs_cp_P(cp, st(n))) <= TOL
    assert rel_inf(g.rhs_dense_Q(dk, st(n)), g.rhs_cp_Q(cp, st(n))) <= TOL


def test_dense_with_fft_orders_and_rk2():
    N = 256
    rng = np.random.default_rng(3)
    a = rng.random((N, N))
    v2 = a + a.T
    cp3 = permutation_power_cp((0.1, -0.1, 0.0), N)
    kernels = {2: g.DenseKernel(v2), 3: g.CPKernel(cp3)}
    n0 = np.zeros(N)
    n0[0] = 1.0
    ref_p, ref_q, ref_s = orc.rhs_total({2: g.DenseKernel(v2), 3: g.CPKernel(cp3)}, n0 + 0.01)
    r = g.rhs_total(g.KernelSet(kernels), st(n0 + 0.01))
    assert rel_inf(r.s, ref_s) <= TOL
    ref_n, _, _ = orc.integrate(kernels, n0, dt=1e-3, steps=20)
    final, _ = g.integrate(_Cfg(n0, 1e-3, 20), kernels=g.KernelSet(kernels))
    assert rel_inf(final.n, ref_n) <= 1e-8


class _Cfg:
    def __init__(self, n0, dt, steps):
        self.n_classes = n0.size
        self.initial = g.InitialCondition.from_vector(n0)
        self.time = g.TimeGrid(0.0, dt, steps)
        self.record_every = 1


def test_dense_budget_and_errors():
    with pytest.raises(g.KernelError, match="budget"):
        g.rhs_dense_P(g.DenseKernel(np.zeros((8193, 8193))), st(np.ones(8193)))
    with pytest.raises(g.KernelError):
        g.rhs_dense_P(g.CPKernel((np.ones((4, 1)), np.ones((4, 1)))), st(np.ones(4)))
    with pytest.raises(g.KernelError):
        g.rhs_dense_Q(g.DenseKernel(np.ones((5, 5))), st(np.ones(6)))
