"""C-ABI behaviour on the device: host-pointer staging (pageable and pinned
buffers), calls from several streams on one context, the RK2 record times
and the device-side finiteness check of the initial state."""

import ctypes

import numpy as np
import pytest
import torch

import paper_1905_09071_b200 as g
from conftest import rel_inf
from oracle import rhs_oracle as orc
from paper_1905_09071_b200 import _lib
from paper_1905_09071_b200.workloads import initial_state, permutation_power_cp

pytestmark = pytest.mark.gpu
TOL = 1e-10


def _cp_set(N, orders=(2, 3)):
    a = (0.1, -0.1, 0.05)
    return {d: permutation_power_cp(a[:d], N) for d in orders}


def _dks(ctx, fs):
    return [ctx.upload_cp(fs[d]) for d in sorted(fs)]


@pytest.mark.parametrize("pinned_out", [False, True])
def test_host_pointer_call_pageable_and_pinned(pinned_out):
    """ttagg_rhs with TTAGG_HOST_PTRS stages pageable buffers through the
    context's page-locked area and transfers pinned ones directly: both give
    the oracle's dn/dt."""
    N = 1 << 17
    fs = _cp_set(N)
    ctx = _lib.get_context()
    dks = _dks(ctx, fs)
    n = initial_state("c2", N)
    if pinned_out:
        outs = [torch.empty(N, dtype=torch.float64, pin_memory=True).numpy() for _ in range(3)]
    else:
        outs = [np.empty(N) for _ in range(3)]
    arr = (ctypes.c_void_p * len(dks))(*[k.handle for k in dks])
    rc = _lib.load().ttagg_rhs(ctx.handle, arr, len(dks), n.ctypes.data, outs[0].ctypes.data,
                               outs[1].ctypes.data, outs[2].ctypes.data, _lib.TTAGG_HOST_PTRS, None)
    assert rc == 0, _lib.lib_error()
    p, q, s = orc.rhs_total({d: {"kind": "cp", "arrays": f} for d, f in fs.items()}, n)
    assert rel_inf(outs[0], p) <= TOL and rel_inf(outs[1], q) <= TOL and rel_inf(outs[2], s) <= TOL


def test_calls_on_two_streams_share_one_context():
    """Two device-pointer calls issued back to back on different streams use
    the same context workspaces: the second waits for the first on the GPU
    (no host synchronisation between them), so both results are exact."""
    N = 1 << 18
    fs = _cp_set(N, (2, 3, 4))
    fs[4] = permutation_power_cp((0.1, -0.1, 0.05, -0.05), N)
    ctx = _lib.get_context()
    dks = _dks(ctx, fs)
    dev = torch.device("cuda", 0)
    na = torch.from_numpy(initial_state("c2", N)).to(dev)
    nb = torch.from_numpy(initial_state("exp256", N)).to(dev)
    outs = [torch.empty(N, dtype=torch.float64, device=dev) for _ in range(6)]
    torch.cuda.synchronize()
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    for _ in range(3):
        ctx.rhs_device(dks, na.data_ptr(), *[o.data_ptr() for o in outs[:3]], s1.cuda_stream)
        ctx.rhs_device(dks, nb.data_ptr(), *[o.data_ptr() for o in outs[3:]], s2.cuda_stream)
    torch.cuda.synchronize()
    ks = {d: {"kind": "cp", "arrays": f} for d, f in fs.items()}
    ref_a = orc.rhs_total(ks, na.cpu().numpy())
    ref_b = orc.rhs_total(ks, nb.cpu().numpy())
    for got, ref in zip(outs[:3], ref_a):
        assert rel_inf(got.cpu().numpy(), ref) <= TOL
    for got, ref in zip(outs[3:], ref_b):
        assert rel_inf(got.cpu().numpy(), ref) <= TOL


def test_rk2_records_carry_times_from_t0():
    """records[:, 0] = t0 accumulated by dt per step, as integrate() does
    (state.t + dt, integrator.py:179, 207), at every record_every-th step."""
    N = 4096
    fs = _cp_set(N)
    ctx = _lib.get_context()
    dks = _dks(ctx, fs)
    t0, dt = 0.5, 0.01
    _, rec, fail, _ = ctx.rk2_host(dks, initial_state("mono", N), t0, dt, 10, 5)
    assert fail == 0
    t, want = t0, [t0]
    for step in range(1, 11):
        t = t + dt
        if step % 5 == 0:
            want.append(t)
    assert rec[:, 0].tolist() == want


def test_rk2_rejects_nonfinite_initial_state():
    N = 4096
    ctx = _lib.get_context()
    dks = _dks(ctx, _cp_set(N))
    n = initial_state("mono", N)
    n[7] = np.nan
    with pytest.raises(ValueError):
        ctx.rk2_host(dks, n, 0.0, 0.01, 2, 1)
