"""Fused RK2 (ttagg_rk2) timing on config C5: per-step time by differencing
runs of different lengths (removes capture and transfer costs).
Usage: python tools/rk2_timing.py [steps...]"""
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_1905_09071_b200 import _lib  # noqa: E402
from paper_1905_09071_b200.workloads import CONFIGS, initial_state, permutation_power_cp  # noqa: E402

cfg = CONFIGS["C5"]
N = 1 << 20
ctx = _lib.get_context(0)
dks = [ctx.upload_cp(permutation_power_cp(cfg.exponents[:d], N)) for d in cfg.orders]
nn = initial_state("c5", N, normalised=True)
ctx.rk2_host(dks, nn, 0.0, cfg.dt, 2, 2)
for graphs in (True, False):
    ctx.profile(not graphs)  # profiling mode runs the steps eagerly (no CUDA graphs)
    for steps in [int(x) for x in sys.argv[1:]] or [10, 50]:
        torch.cuda.synchronize()
        t = time.perf_counter()
        ctx.rk2_host(dks, nn, 0.0, cfg.dt, steps, steps)
        print("graphs" if graphs else "eager", steps, round((time.perf_counter() - t) * 1e3, 1), "ms", flush=True)
    ctx.profile_read()
ctx.profile(False)
