"""Small RHS + RK2 workload for compute-sanitizer runs (memcheck / racecheck / synccheck)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_1905_09071_b200 as g
from oracle import rhs_oracle as orc
from paper_1905_09071_b200.workloads import permutation_power_cp

N = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
rng = np.random.default_rng(0)
exps = (0.1, -0.1, 0.05, -0.05, 0.0)
cp = {d: permutation_power_cp(exps[:d], N) for d in (2, 3, 4, 5)}
i = np.arange(1, N + 1, dtype=np.float64)
tt2 = (np.stack([i ** (2 / 3), 2 * i ** (1 / 3), np.ones(N)], axis=1)[None], np.stack([np.ones(N), i ** (1 / 3), i ** (2 / 3)], axis=0)[:, :, None])
n = np.exp(-i / 50.0) * (1 + 0.1 * rng.random(N))
ks = g.KernelSet({d: g.CPKernel(cp[d]) for d in (3, 4, 5)} | {2: g.TTKernel(tt2)})
res = g.rhs_total(ks, g.ConcentrationState(n))
ref = orc.rhs_total({**{d: {"kind": "cp", "arrays": cp[d]} for d in (3, 4, 5)}, 2: {"kind": "tt", "arrays": tt2}}, n)
err = np.abs(res.s - ref[2]).max() / np.abs(ref[2]).max()
print("rhs rel err", err)
from paper_1905_09071_b200 import _lib
ctx = _lib.get_context()
dks = [ctx.device_kernel(ks[d]) for d in ks.orders]
out = ctx.rk2_host(dks, n / n.sum(), 0.0, 1e-4, 3, 1)
print("rk2 ok", np.isfinite(out[0]).all())
assert err < 1e-10
