"""The C5 tensor through the TT route: subset-structured ("Brownian") TT cores
for the permutation-power kernel of every order (ranks C(d, lam), each core
fiber a power vector or zero), timed on the GPU and checked against the CP
route on the same state.  Benchmark tool; kernel construction is not part of
the product."""
import itertools
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1905_09071_b200 as g
from paper_1905_09071_b200 import _lib
from paper_1905_09071_b200.workloads import CONFIGS, initial_state, permutation_power_cp


def subset_tt(exponents, N):
    d = len(exponents)
    i = np.arange(1, N + 1, dtype=np.float64)
    pows = [i ** a for a in exponents]
    levels = [list(itertools.combinations(range(d), k)) for k in range(d + 1)]
    index = [{s: r for r, s in enumerate(lv)} for lv in levels]
    cores = []
    for lam in range(1, d + 1):
        core = np.zeros((len(levels[lam - 1]), N, len(levels[lam])))
        for rc, T in enumerate(levels[lam]):
            for label in T:
                S = tuple(x for x in T if x != label)
                core[index[lam - 1][S], :, rc] = pows[label]
        cores.append(core)
    return tuple(cores)


N = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 20
cfg = CONFIGS["C5"]
tt = {d: subset_tt(cfg.exponents[:d], N) for d in cfg.orders}
nz = {d: sum(int(np.any(c[p, :, q])) for c in tt[d] for p in range(c.shape[0]) for q in range(c.shape[2])) for d in tt}
tot = {d: sum(c.shape[0] * c.shape[2] for c in tt[d]) for d in tt}
print("fibers (nonzero/total):", {d: f"{nz[d]}/{tot[d]}" for d in tt})
ctx = _lib.get_context()
n0 = initial_state("c5", N)
ks_tt = g.KernelSet({d: g.TTKernel(tt[d]) for d in cfg.orders})
dks = [ctx.device_kernel(ks_tt[d]) for d in ks_tt.orders]
n = torch.from_numpy(n0).cuda()
p = torch.empty_like(n); q = torch.empty_like(n); s = torch.empty_like(n)
for _ in range(3):
    ctx.rhs_device(dks, n.data_ptr(), p.data_ptr(), q.data_ptr(), s.data_ptr(), None)
torch.cuda.synchronize()
reps = 10
ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ev0.record()
for _ in range(reps):
    ctx.rhs_device(dks, n.data_ptr(), p.data_ptr(), q.data_ptr(), s.data_ptr(), None)
ev1.record()
torch.cuda.synchronize()
ms = ev0.elapsed_time(ev1) / reps
s_tt = s.cpu().numpy()
ks_cp = g.KernelSet({d: g.CPKernel(permutation_power_cp(cfg.exponents[:d], N)) for d in cfg.orders})
s_cp = g.rhs_total(ks_cp, g.ConcentrationState(n0)).s
err = np.abs(s_tt - s_cp).max() / np.abs(s_cp).max()
print(f"C5 tensor via TT route, N={N}: {ms:.2f} ms/RHS ({1000 / ms:.1f} RHS/s); rel. diff vs CP route {err:.2e}")
