"""Initialisation and bounds checks that stand in for compute-sanitizer
(closed on this GPU pool):

* poisoned scratch (ttagg_debug_poison): every workspace the context uses is
  NaN-filled on the call's stream before use; a kernel that reads a value the
  call did not write first would turn the result non-finite or change it.
  Results must stay bitwise identical to an unpoisoned call, across the
  geometries (small / ragged / N1 = 4096 with the TMA-fed pass A and pass B),
  CP, TT and mixed sets, the fused RK2 graph and the rank-sharded perm path;
* guard zones: device outputs sit between NaN-filled guards that must come
  back untouched (no out-of-bounds writes past p, q, s or the perm vectors)."""

import numpy as np
import pytest
import torch

from paper_1905_09071_b200 import _lib
from paper_1905_09071_b200.workloads import CONFIGS, initial_state, permutation_power_cp

pytestmark = pytest.mark.gpu

GUARD = 4096  # doubles on each side


def _sets(ctx, N):
    """Device kernel sets (uploaded through the C-ABI; a random TT is not
    symmetric, which the Python KernelSet would reject at small N)."""
    rng = np.random.default_rng(N)
    exps = CONFIGS["C5"].exponents
    cp = {d: ctx.upload_cp(permutation_power_cp(exps[:d], N)) for d in (2, 3, 4, 5)}
    r = 5
    tt3 = ctx.upload_tt((rng.random((1, N, r)), rng.random((r, N, r)) / r, rng.random((r, N, 1))))
    return {"cp": [cp[d] for d in (2, 3, 4, 5)], "tt+cp": [cp[2], tt3, cp[4]]}


def _guarded(N, dev):
    buf = torch.full((N + 2 * GUARD,), float("nan"), dtype=torch.float64, device=dev)
    return buf, buf[GUARD:GUARD + N]


def _guards_intact(buf, N):
    head, tail = buf[:GUARD], buf[GUARD + N:]
    return bool(torch.isnan(head).all()) and bool(torch.isnan(tail).all())


def _rhs_device(ctx, dks, n_np, dev):
    N = n_np.size
    n = torch.from_numpy(n_np).to(dev)
    outs = [_guarded(N, dev) for _ in range(3)]
    ctx.rhs_device(dks, n.data_ptr(), *(o[1].data_ptr() for o in outs), None)
    torch.cuda.synchronize(dev)
    for buf, _ in outs:
        assert _guards_intact(buf, N), "write outside an output vector"
    return [o[1].cpu().numpy() for o in outs]


@pytest.mark.parametrize("N", [37, 1000, (1 << 17) + 3, 1 << 20])
def test_poisoned_scratch_changes_nothing(N):
    ctx = _lib.get_context()
    dev = torch.device("cuda", 0)
    n = initial_state("c5", N) if N >= 1024 else np.exp(-np.arange(1, N + 1) / 17.0)
    for name, dks in _sets(ctx, N).items():
        clean = _rhs_device(ctx, dks, n, dev)
        try:
            ctx.debug_poison(True)
            dirty = _rhs_device(ctx, dks, n, dev)
            dirty2 = _rhs_device(ctx, dks, n, dev)  # workspaces already sized: poisoned again in place
        finally:
            ctx.debug_poison(False)
        for a, b, c, what in zip(clean, dirty, dirty2, "pqs"):
            assert np.isfinite(b).all(), f"{name} N={N} {what}: non-finite under poisoned scratch"
            np.testing.assert_array_equal(a, b, err_msg=f"{name} N={N} {what}")
            np.testing.assert_array_equal(a, c, err_msg=f"{name} N={N} {what} (second call)")


def test_poisoned_scratch_fused_rk2():
    ctx = _lib.get_context()
    N = 1 << 16
    dks = _sets(ctx, N)["cp"]
    n0 = initial_state("c5", N, normalised=True)
    clean = ctx.rk2_host(dks, n0, 0.0, 2e-3, 5, 1)
    try:
        ctx.debug_poison(True)
        dirty = ctx.rk2_host(dks, n0, 0.0, 2e-3, 5, 1)
    finally:
        ctx.debug_poison(False)
    np.testing.assert_array_equal(clean[0], dirty[0])
    np.testing.assert_array_equal(clean[1], dirty[1])


def test_perm_path_guards_and_poison():
    """The rank-sharded path (perm layout in and out, no natural-order copy)."""
    ctx = _lib.get_context()
    dev = torch.device("cuda", 0)
    N = 1 << 20
    Np, _, _ = _lib.geometry(N)
    exps = CONFIGS["C5"].exponents
    dks = [ctx.upload_cp(permutation_power_cp(exps[:d], N), rank_subset=list(range(0, 2 * (d - 1), 2)))
           for d in (3, 4, 5)]
    n = torch.from_numpy(initial_state("c5", N)).to(dev)
    nperm = torch.zeros(Np, dtype=torch.float64, device=dev)
    ctx.permute(N, n.data_ptr(), nperm.data_ptr(), 0, None)
    results = []
    for poison in (False, True):
        buf, s = _guarded(Np, dev)
        try:
            ctx.debug_poison(poison)
            ctx.rhs_perm(dks, nperm.data_ptr(), None, 0.0, s.data_ptr(), None)
            torch.cuda.synchronize(dev)
        finally:
            ctx.debug_poison(False)
        assert _guards_intact(buf, Np)
        results.append(s.cpu().numpy())
    assert np.isfinite(results[1]).all()
    np.testing.assert_array_equal(results[0], results[1])
