"""Projected rank-sharded scaling of config C5 on ONE GPU.

For W = 1, 2, 4, 8 every rank's shard (LPT over the (d, r) rank terms,
`lpt_rank_shards`, the assignment bench.py uses under torchrun) is uploaded
and its partial RHS (`ttagg_rhs_perm`, perm layout, exactly the per-GPU work
of the sharded path) is timed with CUDA events; the per-step time at W GPUs
is the slowest shard.  The all-reduce of the length-N partial (8 MB over
NVLink, tens of microseconds) is not included.  Prints one JSON line.
"""
import json
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1905_09071_b200 as g  # noqa: E402
from paper_1905_09071_b200 import _lib  # noqa: E402
from paper_1905_09071_b200.workloads import CONFIGS, initial_state, permutation_power_cp  # noqa: E402

N = 1 << 20
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
cfg = CONFIGS["C5"]
ctx = _lib.get_context(0)
factors = {d: permutation_power_cp(cfg.exponents[:d], N) for d in cfg.orders}
Np, _, _ = _lib.geometry(N)
n = torch.from_numpy(initial_state("c5", N)).cuda()
nperm = torch.zeros(Np, dtype=torch.float64, device="cuda")
sperm = torch.zeros_like(nperm)
stream = torch.cuda.current_stream()
ctx.permute(N, n.data_ptr(), nperm.data_ptr(), 0, stream.cuda_stream)


def time_shard(shard):
    dks = [ctx.upload_cp(factors[d], rank_subset=shard[d]) for d in cfg.orders if shard.get(d)]
    for _ in range(2):
        ctx.rhs_perm(dks, nperm.data_ptr(), None, 0.0, sperm.data_ptr(), stream.cuda_stream)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for _ in range(reps):
        ctx.rhs_perm(dks, nperm.data_ptr(), None, 0.0, sperm.data_ptr(), stream.cuda_stream)
    b.record(stream)
    torch.cuda.synchronize()
    del dks
    return a.elapsed_time(b) / reps


out = {}
t1 = None
for W in (1, 2, 4, 8):
    shards = g.lpt_rank_shards({d: math.factorial(d) for d in cfg.orders}, W)
    times = [time_shard(sh) for sh in shards]
    tmax = max(times)
    t1 = t1 or tmax
    out[W] = {"ms_per_step": tmax, "rhs_per_s": 1000.0 / tmax, "shard_ms": [round(x, 3) for x in times],
              "efficiency_vs_1": t1 / (W * tmax)}
    print(W, json.dumps(out[W]), flush=True)
print(json.dumps({"projection": "C5 rank shards timed one after another on one B200 (no all-reduce)", "by_gpus": out}))
