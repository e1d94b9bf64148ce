import time, os, sys, math
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from oracle import rhs_oracle as orc
from paper_1905_09071_b200.workloads import CONFIGS, initial_state, permutation_power_cp
cfg = CONFIGS["C5"]; N = 1 << 20
n0 = initial_state("c5", N)
f = {d: permutation_power_cp(cfg.exponents[:d], N) for d in cfg.orders}
W = os.cpu_count()
chunk = int(sys.argv[1]) if len(sys.argv) > 1 else 8
for d in sorted(f):
    t0 = time.perf_counter(); orc.cp_gain(f[d], n0, workers=W, rank_chunk=chunk); tg = time.perf_counter() - t0
    t0 = time.perf_counter(); orc.cp_loss(f[d], n0); tl = time.perf_counter() - t0
    print(d, f"gain {tg:.2f}s loss {tl:.3f}s", flush=True)
