"""Time the TT path at C4 scale (N = 2^20, d=3 ranks (1,r,r,1) + d=2 ranks (1,3,1))."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1905_09071_b200 as g
from paper_1905_09071_b200 import _lib
N = 1 << 20
r = int(sys.argv[1]) if len(sys.argv) > 1 else 16
rng = np.random.default_rng(0)
i = np.arange(1, N + 1, dtype=np.float64)
c1 = np.zeros((1, N, 3)); c1[0, :, 0], c1[0, :, 1], c1[0, :, 2] = i ** (2 / 3), 2 * i ** (1 / 3), 1.0
c2 = np.zeros((3, N, 1)); c2[0, :, 0], c2[1, :, 0], c2[2, :, 0] = 1.0, i ** (1 / 3), i ** (2 / 3)
d3 = (rng.random((1, N, r)), rng.random((r, N, r)) / r, rng.random((r, N, 1)))
ks = g.KernelSet({2: g.TTKernel((c1, c2)), 3: g.TTKernel(d3)})
ctx = _lib.get_context()
dks = [ctx.device_kernel(ks[d]) for d in ks.orders]
n = torch.from_numpy(np.exp(-i / 1024)).cuda()
p = torch.empty_like(n); q = torch.empty_like(n); s = torch.empty_like(n)
for _ in range(2):
    ctx.rhs_device(dks, n.data_ptr(), p.data_ptr(), q.data_ptr(), s.data_ptr(), None)
torch.cuda.synchronize()
ctx.profile_read(); ctx.profile(True)
t0 = time.perf_counter()
reps = 5
for _ in range(reps):
    ctx.rhs_device(dks, n.data_ptr(), p.data_ptr(), q.data_ptr(), s.data_ptr(), None)
torch.cuda.synchronize()
dt = (time.perf_counter() - t0) / reps
ctx.profile(False)
prof = ctx.profile_read()
print(f"TT C4-shape r={r}: {dt*1e3:.2f} ms/RHS ({1/dt:.1f} RHS/s)", {f"{'ABCO'[c]}{d}": round(v[0]/reps, 3) for (c, d), v in sorted(prof.items())})
