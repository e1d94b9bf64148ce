"""Run a few C5 RHS evaluations (device pointers) for ncu captures."""
import sys, os, math
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1905_09071_b200 import _lib
from paper_1905_09071_b200.workloads import CONFIGS, initial_state, permutation_power_cp
N = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 20
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
orders = [int(x) for x in sys.argv[3].split(",")] if len(sys.argv) > 3 else [2, 3, 4, 5]
cfg = CONFIGS["C5"]
ctx = _lib.get_context(0)
dks = [ctx.upload_cp(permutation_power_cp(cfg.exponents[:d], N)) for d in orders]
n = torch.from_numpy(initial_state("c5", N)).cuda()
p = torch.empty_like(n); q = torch.empty_like(n); s = torch.empty_like(n)
for _ in range(reps):
    ctx.rhs_device(dks, n.data_ptr(), p.data_ptr(), q.data_ptr(), s.data_ptr(), None)
torch.cuda.synchronize()
print("done", float(s.abs().max()))
