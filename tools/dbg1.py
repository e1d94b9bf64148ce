import sys, os, time
print("start", flush=True)
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1905_09071_b200 import _lib
print("lib loaded", _lib.load().ttagg_version(), flush=True)
ctx = _lib.Context(0)
print("ctx ok", flush=True)
rng = np.random.default_rng(0)
N, d = 64, 2
fs = [rng.random((N, 2)) for _ in range(d)]
dk = ctx.upload_cp(fs)
print("upload ok", dk.info(), flush=True)
n = rng.random(N)
out = ctx.rhs_host([dk], n, want_p=False, want_q=True, outputs=("q",))
print("Q ok", out["q"][:4], flush=True)
out = ctx.rhs_host([dk], n, want_p=True, want_q=False, outputs=("p",))
print("P ok", out["p"][:4], flush=True)
from oracle import rhs_oracle as orc
print(np.abs(out["p"] - orc.cp_gain(fs, n)).max(), np.abs(orc.cp_gain(fs, n)).max())
