import sys, os, time
sys.path.insert(0, '/root/repo'); os.chdir(os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import numpy as np, torch
import paper_1905_09071_b200 as g
from paper_1905_09071_b200 import _lib
from paper_1905_09071_b200.workloads import CONFIGS, initial_state, permutation_power_cp
cfg = CONFIGS["C5"]; N = cfg.n_classes
factors = {d: permutation_power_cp(cfg.exponents[:d], N) for d in cfg.orders}
ctx = _lib.get_context(0)
dks = [ctx.upload_cp(factors[d]) for d in cfg.orders]
n_t = torch.from_numpy(initial_state("c5", N)).cuda(); p = torch.empty_like(n_t); q = torch.empty_like(n_t); s = torch.empty_like(n_t)
for _ in range(5): ctx.rhs_device(dks, n_t.data_ptr(), p.data_ptr(), q.data_ptr(), s.data_ptr(), torch.cuda.current_stream().cuda_stream)
torch.cuda.synchronize()
ks = g.KernelSet({d: g.CPKernel(factors[d]) for d in cfg.orders})
st = g.ConcentrationState(initial_state("c5", N))
for i in range(8):
    t0 = time.perf_counter(); r = g.rhs_total(ks, st); print(f"iter {i}: {(time.perf_counter()-t0)*1e3:.2f} ms", flush=True)
