"""Where does the time of one public-API rhs_total call go (C5)?"""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1905_09071_b200 as g
from paper_1905_09071_b200 import _lib
from paper_1905_09071_b200.workloads import CONFIGS, initial_state, permutation_power_cp
cfg = CONFIGS["C5"]; N = cfg.n_classes
ks = g.KernelSet({d: g.CPKernel(permutation_power_cp(cfg.exponents[:d], N)) for d in cfg.orders})
n0 = initial_state("c5", N)
st = g.ConcentrationState(n0)
for _ in range(3): g.rhs_total(ks, st)
def tm(f, reps=10):
    t0 = time.perf_counter()
    for _ in range(reps): f()
    return (time.perf_counter() - t0) / reps * 1e3
ctx = _lib.get_context()
dks = [ctx.device_kernel(ks[d]) for d in ks.orders]
print("ConcentrationState(n0)      %.2f ms" % tm(lambda: g.ConcentrationState(n0)))
print("np.isfinite(n0).all()       %.2f ms" % tm(lambda: np.isfinite(n0).all()))
print("ctx._pinned(N, 3)           %.2f ms" % tm(lambda: ctx._pinned(N, 3)))
print("ctx.rhs_host(dks, n)        %.2f ms" % tm(lambda: ctx.rhs_host(dks, n0)))
print("g.rhs_total(ks, st)         %.2f ms" % tm(lambda: g.rhs_total(ks, st)))
print("state+rhs_total             %.2f ms" % tm(lambda: g.rhs_total(ks, g.ConcentrationState(n0))))
# the library alone: pinned state in, pinned outputs reused (no Python allocation)
import ctypes, torch
from paper_1905_09071_b200._lib import load, _vp, TTAGG_HOST_PTRS, TTAGG_WANT_P, TTAGG_WANT_Q
lib = load()
nin = torch.from_numpy(n0.copy()).pin_memory().numpy()
outs = [torch.empty(N, dtype=torch.float64, pin_memory=True).numpy() for _ in range(3)]
arr = (_vp * len(dks))(*[k.handle for k in dks])
fl = TTAGG_HOST_PTRS | TTAGG_WANT_P | TTAGG_WANT_Q
raw = lambda: lib.ttagg_rhs(ctx.handle, arr, len(dks), nin.ctypes.data, outs[0].ctypes.data, outs[1].ctypes.data, outs[2].ctypes.data, fl, None)
print("raw ttagg_rhs pinned in/out %.2f ms" % tm(raw))
dev = torch.device("cuda", 0)
nd = torch.from_numpy(n0).to(dev); pd = torch.empty(3 * N, dtype=torch.float64, device=dev)
def devonly():
    ctx.rhs_device(dks, nd.data_ptr(), pd.data_ptr(), pd.data_ptr() + 8 * N, pd.data_ptr() + 16 * N,
                   torch.cuda.current_stream(dev).cuda_stream)
    torch.cuda.synchronize(dev)
print("device ptrs + sync          %.2f ms" % tm(devonly))
print("raw ttagg_rhs pinned in/out %.2f ms (again)" % tm(raw))
print("g.rhs_total(ks, st)         %.2f ms (again)" % tm(lambda: g.rhs_total(ks, st)))
