"""GPU parity: the sm_100a path through the public API vs the reference's
own golden vectors, the pinned oracle and FFT-independent properties.
Tolerance: relative max-norm error <= 1e-10 per RHS (BASELINE north star)."""

import numpy as np
import pytest

import paper_1905_09071_b200 as g
from conftest import rel_inf
from oracle import rhs_oracle as orc
from paper_1905_09071_b200 import _lib
from paper_1905_09071_b200.workloads import CONFIGS, initial_state, permutation_power_cp

pytestmark = pytest.mark.gpu
TOL = 1e-10


def st(n):
    return g.ConcentrationState(n)


def test_extension_is_loaded_and_device_present():
    ctx = _lib.get_context()
    assert ctx.handle
    maps = open("/proc/self/maps").read()
    assert "libttagg_b200.so" in maps


@pytest.mark.parametrize("order", [2, 3, 4, 5])
def test_cp_random_factors_vs_reference(golden, order):
    u = golden("unit.npz")
    k = g.CPKernel(tuple(u[f"cp{order}_f{i}"] for i in range(order)))
    for s in range(3):
        n = u[f"cp{order}_n{s}"]
        assert rel_inf(g.rhs_cp_P(k, st(n)), u[f"cp{order}_P{s}"]) <= TOL
        assert rel_inf(g.rhs_cp_Q(k, st(n)), u[f"cp{order}_Q{s}"]) <= TOL


@pytest.mark.parametrize("tag,order", [("cpodd", 3), ("cptiny", 2)])
def test_cp_ragged_vs_reference(golden, tag, order):
    u = golden("unit.npz")
    k = g.CPKernel(tuple(u[f"{tag}_f{i}"] for i in range(order)))
    assert rel_inf(g.rhs_cp_P(k, st(u[f"{tag}_n"])), u[f"{tag}_P"]) <= TOL
    assert rel_inf(g.rhs_cp_Q(k, st(u[f"{tag}_n"])), u[f"{tag}_Q"]) <= TOL


@pytest.mark.parametrize("order", [2, 3, 4])
def test_tt_brownian_vs_reference(golden, order):
    u = golden("unit.npz")
    k = g.TTKernel(tuple(u[f"tt{order}_c{i}"] for i in range(order)))
    for s in range(3):
        n = u[f"tt{order}_n{s}"]
        assert rel_inf(g.rhs_tt_P(k, st(n)), u[f"tt{order}_P{s}"]) <= TOL
        assert rel_inf(g.rhs_tt_Q(k, st(n)), u[f"tt{order}_Q{s}"]) <= TOL


def test_mixed_sets_vs_reference(golden):
    u = golden("unit.npz")
    n = u["mix2_n"]
    ks = g.KernelSet({2: g.CPKernel(permutation_power_cp((0.2, -0.3), n.size)),
                      3: g.CPKernel(permutation_power_cp((0.3, -0.2, 0.1), n.size))})
    r = g.rhs_total(ks, st(n))
    assert rel_inf(r.p, u["mix2_p"]) <= TOL and rel_inf(r.q, u["mix2_q"]) <= TOL
    assert rel_inf(r.s, u["mix2_s"]) <= TOL


def test_known_answers_exact(golden):
    u = golden("unit.npz")
    e = np.zeros(8)
    e[0] = 1.0
    r = g.rhs_total(g.KernelSet({2: g.constant_tt(1.0, 2, 8)}), st(e))
    np.testing.assert_allclose(r.s, u["ka_s2"], atol=1e-15)
    p3 = g.rhs_cp_P(g.constant_cp(1.0, 3, 8), st(e))
    np.testing.assert_allclose(p3, u["ka_p3"], atol=1e-15)
    assert np.all(p3[:2] == 0.0)
    np.testing.assert_allclose(g.rhs_cp_Q(g.constant_cp(1.0, 3, 8), st(e)), u["ka_q3"], atol=1e-15)
    n = u["conv_n"]
    np.testing.assert_allclose(g.rhs_tt_P(g.constant_tt(1.75, 3, 16), st(n)), u["conv_P"], rtol=1e-12, atol=1e-15)


def test_zero_state_is_exactly_zero():  # test_rhs.py:140-145, 188-193
    rng = np.random.default_rng(37)
    k = g.CPKernel(tuple(rng.random((16, 3)) for _ in range(3)))
    z = st(np.zeros(16))
    np.testing.assert_array_equal(g.rhs_cp_P(k, z), np.zeros(16))
    np.testing.assert_array_equal(g.rhs_cp_Q(k, z), np.zeros(16))


def test_gain_support_lower_bound_is_exact():  # test_rhs.py:308-317
    rng = np.random.default_rng(61)
    for n_classes in (32, 5000, 70000):
        n = rng.random(n_classes) + 0.5
        for d in (2, 3, 4, 5):
            k = g.CPKernel(permutation_power_cp(tuple(rng.uniform(-1, 1, d)), n_classes))
            p = g.rhs_cp_P(k, st(n))
            assert np.all(p[: d - 1] == 0.0)


@pytest.mark.parametrize("n_classes", [2, 3, 5, 17, 64, 65, 255, 1000, 4097, 12345, 70001])
def test_ragged_sizes_vs_oracle(n_classes):
    rng = np.random.default_rng(n_classes)
    n = rng.random(n_classes)
    for d in (2, 3, 4, 5, 6):
        fs = tuple(rng.random((n_classes, 3)) for _ in range(d))
        k = g.CPKernel(fs)
        assert rel_inf(g.rhs_cp_P(k, st(n)), orc.cp_gain(fs, n)) <= TOL
        assert rel_inf(g.rhs_cp_Q(k, st(n)), orc.cp_loss(fs, n)) <= TOL


@pytest.mark.parametrize("n_classes,ranks", [(64, (1, 4, 1)), (300, (1, 3, 5, 1)), (4096, (1, 4, 4, 3, 1)),
                                             (20000, (1, 7, 7, 1)), (65536, (1, 16, 16, 1))])
def test_tt_random_ranks_vs_oracle(n_classes, ranks):
    rng = np.random.default_rng(len(ranks) * 7 + n_classes)
    cores = tuple(rng.random((ranks[l], n_classes, ranks[l + 1])) for l in range(len(ranks) - 1))
    n = rng.random(n_classes)
    k = g.TTKernel(cores)
    assert rel_inf(g.rhs_tt_P(k, st(n)), orc.tt_gain(cores, n)) <= TOL
    assert rel_inf(g.rhs_tt_Q(k, st(n)), orc.tt_loss(cores, n)) <= TOL


def test_c1_vs_reference(golden):
    c = golden("c1.npz")
    cfg = CONFIGS["C1"]
    ks = g.KernelSet({d: g.CPKernel(f) for d, f in cfg.cp_factors().items()})
    r = g.rhs_total(ks, st(initial_state("mono", cfg.n_classes)))
    assert rel_inf(r.p, c["p0"]) <= TOL and rel_inf(r.q, c["q0"]) <= TOL
    r = g.rhs_total(ks, st(c["nr"]), breakdown=True)
    assert rel_inf(r.p, c["pr"]) <= TOL and rel_inf(r.q, c["qr"]) <= TOL
    for d in cfg.orders:
        assert rel_inf(r.by_order[d][0], c[f"pr_d{d}"]) <= TOL
        assert rel_inf(r.by_order[d][1], c[f"qr_d{d}"]) <= TOL
    np.testing.assert_array_equal(sum(pd for pd, _ in r.by_order.values()), r.p)


def test_c2_vs_reference(golden):
    c = golden("c2.npz")
    cfg = CONFIGS["C2"]
    ks = g.KernelSet({d: g.CPKernel(f) for d, f in cfg.cp_factors().items()})
    r = g.rhs_total(ks, st(initial_state("c2", cfg.n_classes)))
    assert rel_inf(r.p, c["p"]) <= TOL and rel_inf(r.q, c["q"]) <= TOL


def _sums(v):
    k = np.arange(1, v.size + 1, dtype=np.float64)
    return np.array([v.sum(), k @ v, (k * k) @ v, np.abs(v).sum(), np.abs(v).max()])


def test_c3_literal_state_vs_reference(golden):
    c = golden("c3.npz")
    cfg = CONFIGS["C3"]
    ks = g.KernelSet({d: g.CPKernel(f) for d, f in cfg.cp_factors().items()})
    r = g.rhs_total(ks, st(initial_state("exp256", cfg.n_classes)))
    idx = c["idx"]
    assert rel_inf(r.p[idx], c["p"]) <= TOL and rel_inf(r.q[idx], c["q"]) <= TOL
    np.testing.assert_allclose(_sums(r.p), c["p_sums"], rtol=1e-10)
    np.testing.assert_allclose(_sums(r.q), c["q_sums"], rtol=1e-10)


def test_c4_shaped_tt_vs_reference(golden):
    c = golden("c4.npz")
    for n_classes in (128, 256):
        tag = f"n{n_classes}"
        ks = g.KernelSet({2: g.TTKernel((c[f"{tag}_d2_c0"], c[f"{tag}_d2_c1"])),
                          3: g.TTKernel(tuple(c[f"{tag}_d3_c{i}"] for i in range(3)))})
        r = g.rhs_total(ks, st(c[f"{tag}_nr"]))
        assert rel_inf(r.p, c[f"{tag}_pr"]) <= TOL and rel_inf(r.q, c[f"{tag}_qr"]) <= TOL


def test_c5_full_size_vs_reference(golden):
    """N = 2^20, D = 5, ranks 2/6/24/120 at the literal initial state, against
    the reference's own rhs_total (TT route on the same tensor) — samples and
    full-vector moment checksums."""
    c = golden("c5.npz")
    cfg = CONFIGS["C5"]
    N = cfg.n_classes
    ks = g.KernelSet({d: g.CPKernel(permutation_power_cp(cfg.exponents[:d], N)) for d in cfg.orders})
    r = g.rhs_total(ks, st(initial_state("c5", N)), breakdown=True)
    idx = c["idx"]
    assert rel_inf(r.p[idx], c["p"]) <= TOL and rel_inf(r.q[idx], c["q"]) <= TOL
    for d in cfg.orders:
        assert rel_inf(r.by_order[d][0][idx], c[f"p_d{d}"]) <= TOL
        assert rel_inf(r.by_order[d][1][idx], c[f"q_d{d}"]) <= TOL
    np.testing.assert_allclose(_sums(r.p)[[0, 1, 3, 4]], c["p_sums"][[0, 1, 3, 4]], rtol=1e-10)
    np.testing.assert_allclose(_sums(r.q), c["q_sums"], rtol=1e-10)
    # the fused all-orders path agrees with the per-order path
    r2 = g.rhs_total(ks, st(initial_state("c5", N)))
    assert rel_inf(r2.s, r.s) <= 1e-14


def test_c5_full_vectors_vs_oracle_on_the_box():
    """Full-vector (not sampled) p, q and s at N = 2^20, D = 5 against the
    oracle evaluated here on the host cores: every rank term of every order
    through the reference algorithm (pow2 transform length, rhs.py:345-414),
    about 25 s on 16 threads."""
    import os

    cfg = CONFIGS["C5"]
    N = cfg.n_classes
    n = initial_state("c5", N)
    fs = {d: permutation_power_cp(cfg.exponents[:d], N) for d in cfg.orders}
    r = g.rhs_total(g.KernelSet({d: g.CPKernel(f) for d, f in fs.items()}), st(n))
    w = os.cpu_count() or 1
    p = q = 0.0
    for d in cfg.orders:
        p = p + orc.cp_gain(fs[d], n, workers=w, rank_chunk=max(1, 128 // d))
        q = q + orc.cp_loss(fs[d], n)
    assert rel_inf(r.p, p) <= TOL
    assert rel_inf(r.q, q) <= TOL
    assert rel_inf(r.s, p + q) <= TOL


def test_c5_full_size_closed_form_every_order():
    """FFT-length-independent property at full size: the permutation-power
    gain equals the collapsed d-fold convolution."""
    cfg = CONFIGS["C5"]
    N = cfg.n_classes
    n = initial_state("c5", N)
    sizes = np.arange(1, N + 1, dtype=np.float64)
    for d in cfg.orders:
        p = g.rhs_cp_P(g.CPKernel(permutation_power_cp(cfg.exponents[:d], N)), st(n))
        L = 1 << int(np.ceil(np.log2(d * N + 1)))
        spec = np.ones(L // 2 + 1, dtype=complex)
        for j in range(d):
            v = np.zeros(L)
            v[1 : N + 1] = np.exp(cfg.exponents[j] * np.log(sizes)) * n
            spec *= np.fft.rfft(v)
        conv = np.fft.irfft(spec, n=L)
        ref = np.zeros(N)
        ref[d - 1 :] = conv[d : N + 1]
        assert rel_inf(p, ref) <= TOL


def test_mass_conservation_before_boundary_contact():  # test_rhs.py:276-292
    rng = np.random.default_rng(53)
    for n_classes in (64, 1024, 1 << 16):
        n = np.zeros(n_classes)
        n[: n_classes // 4] = rng.random(n_classes // 4)
        sizes = np.arange(1, n_classes + 1, dtype=np.float64)
        for k in (g.constant_tt(1.0, 3, n_classes),
                  g.CPKernel(permutation_power_cp((1 / 3, -1 / 3, 0.0), n_classes))):
            r = g.rhs_total(g.KernelSet({3: k}) if n_classes > 64 else {3: k}, st(n))
            assert abs(sizes @ r.s) <= 1e-12 * (sizes @ r.p)


def test_order_power_scaling():  # test_rhs.py:295-305
    rng = np.random.default_rng(59)
    n = rng.random(3000)
    for d in (2, 3, 4):
        k = g.CPKernel(permutation_power_cp(tuple(rng.uniform(-1, 1, d)), 3000))
        base = g.rhs_total({d: k}, st(n))
        scaled = g.rhs_total({d: k}, st(1.7 * n))
        np.testing.assert_allclose(scaled.p, 1.7**d * base.p, rtol=1e-12, atol=1e-12 * np.abs(scaled.p).max())
        np.testing.assert_allclose(scaled.q, 1.7**d * base.q, rtol=1e-12)


def test_bitwise_determinism():  # test_rhs.py:320-327
    cfg = CONFIGS["C3"]
    ks = g.KernelSet({d: g.CPKernel(f) for d, f in cfg.cp_factors(1 << 16).items()})
    n = initial_state("exp256", 1 << 16)
    a = g.rhs_total(ks, st(n)).s
    b = g.rhs_total(ks, st(n)).s
    np.testing.assert_array_equal(a, b)


def test_rank_shards_sum_to_full_rhs():
    """Multi-GPU premise on one GPU: partial RHS over LPT rank shards (each its
    own upload and launch) sum to the unsharded RHS."""
    import torch

    cfg = CONFIGS["C5"]
    N = 1 << 14
    f = {d: permutation_power_cp(cfg.exponents[:d], N) for d in cfg.orders}
    n = initial_state("c5", N)
    ctx = _lib.get_context()
    full = g.rhs_total(g.KernelSet({d: g.CPKernel(v) for d, v in f.items()}), st(n)).s
    Np, _, _ = _lib.geometry(N)
    dev = torch.device("cuda", ctx.device)
    nt = torch.from_numpy(n).to(dev)
    nperm = torch.zeros(Np, dtype=torch.float64, device=dev)
    ctx.permute(N, nt.data_ptr(), nperm.data_ptr(), 0, None)
    for world in (2, 4, 8):
        acc = torch.zeros(Np, dtype=torch.float64, device=dev)
        for shard in g.lpt_rank_shards({d: v[0].shape[1] for d, v in f.items()}, world):
            dks = [ctx.upload_cp(f[d], rank_subset=shard[d]) for d in sorted(shard)]
            part = torch.zeros(Np, dtype=torch.float64, device=dev)
            ctx.rhs_perm(dks, nperm.data_ptr(), None, 0.0, part.data_ptr(), None)
            acc += part
        out = torch.empty(N, dtype=torch.float64, device=dev)
        ctx.permute(N, acc.data_ptr(), out.data_ptr(), 1, None)
        torch.cuda.synchronize()
        assert rel_inf(out.cpu().numpy(), full) <= 1e-13


def test_error_behaviour():
    with pytest.raises(g.KernelError):
        g.rhs_total(g.KernelSet({2: g.constant_tt(1.0, 2, 8)}), st(np.ones(9)))
    with pytest.raises(ValueError):
        g.ConcentrationState(np.array([1.0, np.nan]))
    # the C-ABI checks host inputs on the device (TTAGG_ERR_NONFINITE -> ValueError)
    ctx = _lib.get_context()
    dk = ctx.device_kernel(g.constant_tt(1.0, 2, 8))
    bad = np.ones(8)
    bad[3] = np.inf
    with pytest.raises(ValueError, match="non-finite"):
        ctx.rhs_host([dk], bad)
    np.testing.assert_allclose(ctx.rhs_host([dk], np.ones(8))["s"][:2], [-8.0, -7.5])
    with pytest.raises(_lib.TTaggError, match="exceeds"):
        g.rhs_cp_P(g.CPKernel((np.ones(((1 << 20) + 1, 1)), np.ones(((1 << 20) + 1, 1)))),
                   st(np.ones((1 << 20) + 1)))


@pytest.mark.gpu
def test_tt_rank_shards_sum_to_full_rhs():
    """TT sharding over the first internal rank (construct.tt_rank_shard): the
    partial RHS of every slice, each its own upload, sum to the unsharded RHS."""
    import torch

    from paper_1905_09071_b200.construct import tt_rank_shard

    N = 5000
    rng = np.random.default_rng(21)
    cores = (rng.random((1, N, 6)), rng.random((6, N, 5)) / 6, rng.random((5, N, 1)))
    n = rng.random(N) * np.exp(-np.arange(N) / 700.0)
    full = g.rhs_total(g.KernelSet({3: g.TTKernel(cores)}), st(n)).s
    ctx = _lib.get_context()
    Np, _, _ = _lib.geometry(N)
    dev = torch.device("cuda", ctx.device)
    nt = torch.from_numpy(n).to(dev)
    nperm = torch.zeros(Np, dtype=torch.float64, device=dev)
    ctx.permute(N, nt.data_ptr(), nperm.data_ptr(), 0, None)
    for world in (2, 3, 8):
        acc = torch.zeros(Np, dtype=torch.float64, device=dev)
        for r in range(world):
            sl = tt_rank_shard(cores, world, r)
            if sl is None:
                continue
            part = torch.zeros(Np, dtype=torch.float64, device=dev)
            ctx.rhs_perm([ctx.upload_tt(sl)], nperm.data_ptr(), None, 0.0, part.data_ptr(), None)
            acc += part
        out = torch.empty(N, dtype=torch.float64, device=dev)
        ctx.permute(N, acc.data_ptr(), out.data_ptr(), 1, None)
        torch.cuda.synchronize()
        assert rel_inf(out.cpu().numpy(), full) <= 1e-12


@pytest.mark.gpu
def test_c4_cross_kernel_vs_oracle():
    """Config C4's kernel set built by construct.c4_kernels (TT-cross d = 3,
    exact d = 2) at N = 4096: GPU RHS against the oracle on the same cores."""
    from paper_1905_09071_b200.construct import c4_kernels

    N = 4096
    (c1, c2), cores3 = c4_kernels(N, rank=16)
    n = np.exp(-np.arange(1, N + 1) / 256.0)
    ks = g.KernelSet({2: g.TTKernel((c1, c2)), 3: g.TTKernel(cores3)})
    res = g.rhs_total(ks, st(n))
    ref = orc.rhs_total({2: {"kind": "tt", "arrays": (c1, c2)}, 3: {"kind": "tt", "arrays": cores3}}, n)
    assert rel_inf(res.p, ref[0]) <= TOL
    assert rel_inf(res.q, ref[1]) <= TOL
    assert rel_inf(res.s, ref[2]) <= TOL


@pytest.mark.gpu
def test_workspace_regrowth_between_kernel_sets():
    """A kernel set with fewer column pairs sizes the per-order workspaces
    first; the next (larger) set must regrow and re-zero them before any of
    its passes run on the context's streams (regression: the zeroing once
    raced the first pass A on a non-blocking stream)."""
    cfg = CONFIGS["C5"]
    N = 1 << 16
    rng = np.random.default_rng(5)
    n = initial_state("c5", N)
    small = g.KernelSet({d: g.TTKernel(tuple(rng.random((r0, N, r1)) for r0, r1 in zip((1,) + (2,) * (d - 1), (2,) * (d - 1) + (1,))))
                         for d in cfg.orders})
    big = g.KernelSet({d: g.CPKernel(permutation_power_cp(cfg.exponents[:d], N)) for d in cfg.orders})
    g.rhs_total(small, st(n))
    got = g.rhs_total(big, st(n))
    ref = orc.rhs_total({d: {"kind": "cp", "arrays": big[d].factors} for d in big.orders}, n)
    assert rel_inf(got.p, ref[0]) <= TOL
    assert rel_inf(got.s, ref[2]) <= TOL


@pytest.mark.parametrize("n_classes", [300001, 600000])
def test_large_ragged_sizes_vs_oracle(n_classes):
    """Ragged N in the 2048- and 4096-point column-transform geometries
    (N1 = 2048 at N = 300001, N1 = 4096 at N = 600000), every order, CP and TT."""
    rng = np.random.default_rng(n_classes)
    n = rng.random(n_classes) * np.exp(-np.arange(n_classes) / (n_classes / 8))
    for d in (2, 3, 4, 5):
        fs = tuple(rng.random((n_classes, 2)) for _ in range(d))
        k = g.CPKernel(fs)
        assert rel_inf(g.rhs_cp_P(k, st(n)), orc.cp_gain(fs, n)) <= TOL
        assert rel_inf(g.rhs_cp_Q(k, st(n)), orc.cp_loss(fs, n)) <= TOL
    ranks = (1, 3, 2, 1)
    cores = tuple(rng.random((ranks[l], n_classes, ranks[l + 1])) for l in range(3))
    kt = g.TTKernel(cores)
    assert rel_inf(g.rhs_tt_P(kt, st(n)), orc.tt_gain(cores, n)) <= TOL
    assert rel_inf(g.rhs_tt_Q(kt, st(n)), orc.tt_loss(cores, n)) <= TOL


@pytest.mark.parametrize("order", [2, 3, 4])
@pytest.mark.parametrize("n_classes", [8, 16, 32])
def test_acceptance_criterion_2_small_sizes(order, n_classes):
    """test_acceptance.py:79-106: fast paths vs the dense direct sums for
    d in {2,3,4} x N in {8,16,32} x 20 states, CP and TT, P and Q, 1e-10."""
    rng = np.random.default_rng(100 * order + n_classes)
    fs = tuple(rng.random((n_classes, 3)) for _ in range(order))
    ranks = (1,) + (2,) * (order - 1) + (1,)
    cores = tuple(rng.random((ranks[l], n_classes, ranks[l + 1])) for l in range(order))
    kc, kt = g.CPKernel(fs), g.TTKernel(cores)
    dc, dt = orc.dense_from_cp(fs), orc.dense_from_tt(cores)
    for _ in range(20):
        n = rng.random(n_classes)
        assert rel_inf(g.rhs_cp_P(kc, st(n)), orc.dense_gain(dc, n)) <= TOL
        assert rel_inf(g.rhs_cp_Q(kc, st(n)), orc.dense_loss(dc, n)) <= TOL
        assert rel_inf(g.rhs_tt_P(kt, st(n)), orc.dense_gain(dt, n)) <= TOL
        assert rel_inf(g.rhs_tt_Q(kt, st(n)), orc.dense_loss(dt, n)) <= TOL


_SWITCH_SCRIPT = r"""
import sys, numpy as np
import paper_1905_09071_b200 as g
from paper_1905_09071_b200.workloads import CONFIGS, initial_state
N = 1 << 18
cfg = CONFIGS["C3"]
fac = cfg.cp_factors(N)
rng = np.random.default_rng(5)
tt = g.TTKernel((rng.random((1, N, 3)), rng.random((3, N, 2)), rng.random((2, N, 1))))
ks = g.KernelSet({2: g.CPKernel(fac[2]), 3: tt, 4: g.CPKernel(fac[4])})
n = initial_state("exp256", N)
r = g.rhs_total(ks, g.ConcentrationState(n))
np.save(sys.argv[1], np.stack([r.p, r.q, r.s]))
"""


@pytest.mark.parametrize("switch", ["TTAGG_RAWX=0", "TTAGG_PASSB_PIPE=0", "TTAGG_PASSA=0", "TTAGG_PASSB_TMA=0"])
def test_kernel_route_switches_agree(switch, tmp_path):
    """The A/B switches select other kernels for the same arithmetic (raw
    exchange off; non-pipeline CP pass B; one-CTA-per-item pass A; cp.async
    pass B): a CP + TT set at N = 2^18 through each of them (own process — the
    switches are read once) matches the default route to roundoff."""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

    def run(extra_env, out):
        env = dict(os.environ, PYTHONPATH=root + os.pathsep + os.environ.get("PYTHONPATH", ""))
        env.update(extra_env)
        subprocess.run([sys.executable, "-c", _SWITCH_SCRIPT, str(out)], check=True, env=env, cwd=root, timeout=600)
        return np.load(out)

    ref_path = tmp_path.parent / "route_default.npy"
    ref = np.load(ref_path) if ref_path.exists() else run({}, ref_path)
    key, val = switch.split("=")
    got = run({key: val}, tmp_path / "route.npy")
    for i, name in enumerate("pqs"):
        assert rel_inf(got[i], ref[i]) < 1e-12, f"{switch}: {name}"
