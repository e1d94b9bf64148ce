"""Host kernel construction for config C4 (construct.py): TT-cross accuracy,
the exact rank-3 d = 2 kernel, and TT rank slices summing to the full RHS."""

import numpy as np

from conftest import rel_inf
from oracle import rhs_oracle as orc
from paper_1905_09071_b200.construct import _c4_d3, c4_kernels, maxvol, tt_cross, tt_rank_shard


def _tt_eval(cores, pts):
    v = cores[0][0, pts[:, 0] - 1, :]
    for k in range(1, len(cores)):
        v = np.einsum("pa,apb->pb", v, cores[k][:, pts[:, k] - 1, :])
    return v[:, 0]


def test_maxvol_finds_dominant_rows():
    rng = np.random.default_rng(0)
    a = rng.standard_normal((200, 5))
    a[[7, 50, 99, 120, 180]] *= 100.0
    assert sorted(maxvol(a).tolist()) == [7, 50, 99, 120, 180]


def test_tt_cross_c4_kernel_small_grid():
    N = 300
    cores = tt_cross(_c4_d3, N, 3, 16)
    assert [c.shape for c in cores] == [(1, N, 16), (16, N, 16), (16, N, 1)]
    rng = np.random.default_rng(1)
    pts = rng.integers(1, N + 1, size=(5000, 3))
    vals = _c4_d3(pts)
    err = np.abs(_tt_eval(cores, pts) - vals).max() / np.abs(vals).max()
    assert err <= 1e-6  # BASELINE C4 tolerance


def test_c4_d2_exact_and_dense_match():
    N = 40
    (c1, c2), cores3 = c4_kernels(N, rank=8)
    i = np.arange(1, N + 1, dtype=np.float64)
    want = (i[:, None] ** (1 / 3) + i[None, :] ** (1 / 3)) ** 2
    np.testing.assert_allclose(orc.dense_from_tt((c1, c2)), want, rtol=1e-13)
    dense3 = orc.dense_from_tt(cores3)
    g = i[:, None, None] + i[None, :, None] + i[None, None, :]
    want3 = np.sqrt(g) * (i[:, None, None] * i[None, :, None] * i[None, None, :]) ** (-1 / 6)
    assert np.abs(dense3 - want3).max() / want3.max() <= 1e-6


def test_tt_rank_shards_sum_to_full_rhs():
    N = 120
    rng = np.random.default_rng(2)
    cores = (rng.random((1, N, 5)), rng.random((5, N, 3)), rng.random((3, N, 1)))
    n = rng.random(N)
    full_g, full_l = orc.tt_gain(cores, n), orc.tt_loss(cores, n)
    for world in (2, 3, 8):
        parts = [tt_rank_shard(cores, world, r) for r in range(world)]
        parts = [p for p in parts if p is not None]
        assert len(parts) == min(world, 5)
        g = sum(orc.tt_gain(p, n) for p in parts)
        l = sum(orc.tt_loss(p, n) for p in parts)
        assert rel_inf(g, full_g) <= 1e-13
        assert rel_inf(l, full_l) <= 1e-13


def test_cross_skeleton_reproduces_cores():
    """The stored skeleton (I, J) rebuilds the cross cores bit for bit."""
    from paper_1905_09071_b200 import construct

    (c1, c2), cores3, (I, J) = construct.c4_kernels(300, rank=6, return_skeleton=True)
    again = construct.c4_d3_from_skeleton(300, I, J)
    for a, b in zip(cores3, again):
        assert np.array_equal(a, b)
