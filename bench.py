#!/usr/bin/env python
"""Benchmark of the RHS evaluator (BASELINE.json metric: RHS evals/sec and RK2
steps/sec at N = 2^20; achieved HBM GB/s vs peak).

Workload (``config.workload``): BASELINE config 5 — D = 5 (orders 2..5),
N = 2^20, permutation-power CP kernel, ranks 2/6/24/120, fp64, initial
state n_k = exp(-k/1024)(1 +/- 5% seeded noise).  One "step" = one full RHS
evaluation dn/dt = sum_d P^(d) + Q^(d).  Inputs (6 GB of factors, 25 GB of
exchange) are far larger than the 126 MB L2, so no flush is needed.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Under torchrun (N > 1) the CP rank terms are sharded over the GPUs (LPT,
SURVEY.md §8(e)) and one NCCL all-reduce of the length-N partial dn/dt runs
per RHS; rank 0 prints one JSON line.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "RHS evals/sec"
UNIT = "RHS/s"
WORKLOAD = "C5: D=5 (d=2..5), N=2^20, permutation-power CP ranks 2/6/24/120, fp64"


def _peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


# --------------------------------------------------------------------------
# clocks during the timed region
# --------------------------------------------------------------------------
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
            time.sleep(0.3)
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for name, val in zip(names, parts[2:6]):
                if val.lower().startswith("active"):
                    reasons.add(name)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# --------------------------------------------------------------------------
# algorithmic bytes (SURVEY.md §8(d) model)
# --------------------------------------------------------------------------
def model_bytes(N: int, cols: dict, tails: dict) -> dict:
    """Per-RHS byte model with L_d = d*N: B_RHS and per-kernel terms."""
    out = {"B_min": 16 * N, "B_RHS": 16 * N, "passA": {}, "passB": {}}
    for d, X in cols.items():
        L = d * N
        T = tails[d]
        out["B_min"] += 8 * N * (X + T)
        out["B_RHS"] += 8 * N * (X + T) + 16 * L * (X + 2)
        out["passA"][d] = X * (8 * N + 8 * L)   # read each column, write its half spectrum
        out["passB"][d] = X * 8 * L + 8 * L       # read every half spectrum, write the inverse rows
    return out


def fp64_flops(N: int, cols: dict) -> float:
    return sum((X + 1) * 2.5 * (d * N) * math.log2(d * N) for d, X in cols.items())


# --------------------------------------------------------------------------
# CPU arm (the reference algorithm, restated in oracle/; checker + baseline only)
# --------------------------------------------------------------------------
def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform

    return platform.processor() or "unknown"


def cpu_whole_rhs(factors_by_order, n0, workers):
    """Seconds for ONE whole RHS of the workload on the host cores, through the
    port of the reference algorithm (oracle/rhs_oracle.py restates
    rhs.py:345-414 on scipy.fft, the reference's default pow2 transform length
    L = 2^23 at d = 5): every rank term of every order, p, q and s = p + q.
    ``rank_chunk`` only bounds the memory (about 125 spectra at a time)."""
    from oracle import rhs_oracle as orc

    t0 = time.perf_counter()
    p = q = None
    for d, fs in sorted(factors_by_order.items()):
        R = fs[0].shape[1]
        pd = orc.cp_gain(fs, n0, workers=workers, rank_chunk=max(1, min(R, 128 // d)))
        qd = orc.cp_loss(fs, n0)
        p = pd if p is None else p + pd
        q = qd if q is None else q + qd
    s = p + q
    del s
    return time.perf_counter() - t0


def cpu_sample_desc(factors_by_order, workers):
    ranks = "/".join(str(fs[0].shape[1]) for _, fs in sorted(factors_by_order.items()))
    return (f"whole C5 RHS (all {ranks} rank terms, p, q and s; nothing sampled or scaled) on {workers} "
            f"host threads of a {cpu_model()}; oracle/rhs_oracle.py restates rhs.py:345-414 on "
            "scipy.fft with the reference's pow2 transform length")


def run_reference(args, N, factors_by_order, n0):
    """The reference arm: whole C5 RHS evaluations on the host cores.  One
    whole RHS (≈23 s on the box's 16 cores) warms scipy's plan cache and the
    page-ins; more warm-up would only lengthen the run (the line reports the
    warm-up actually run)."""
    workers = os.cpu_count() or 1
    args.warmup = min(args.warmup, 1)
    for _ in range(args.warmup):
        cpu_whole_rhs(factors_by_order, n0, workers)
    times = [cpu_whole_rhs(factors_by_order, n0, workers) for _ in range(args.steps)]
    total = sum(times)
    value = args.steps / total
    line = {
        "impl": "reference",
        "metric": METRIC,
        "value": value,
        "unit": UNIT,
        "n_gpus": args.gpus,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": total / args.steps * 1e3,
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": WORKLOAD, "l2": "inputs larger than L2"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": workers, "kind": "port",
                         "sample": cpu_sample_desc(factors_by_order, workers),
                         "median_s": statistics.median(times), "min_s": min(times), "max_s": max(times)},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def c4_tt_timing(ctx, N, dev, stream, steps):
    """RHS/s of config C4: the d = 3 TT-cross kernel (ranks 16; rebuilt in
    seconds from the cross skeleton stored with the C4 trajectory golden, or
    seeded cores of the same shape when that file is absent — the cost
    depends on the ranks only) and the exact rank-3 TT of
    (i^(1/3) + j^(1/3))^2 for d = 2, monodisperse state."""
    import numpy as np
    import torch

    import paper_1905_09071_b200 as g

    from paper_1905_09071_b200 import construct

    skel = os.path.join(ROOT, "tests", "golden", "c4traj.npz")
    if os.path.exists(skel):  # the config's own TT-cross kernel, rebuilt from its stored skeleton
        c = np.load(skel)
        d3 = construct.c4_d3_from_skeleton(N, [c["I0"], c["I1"], c["I2"]], [None, c["J1"], c["J2"], c["J3"]])
        source = "TT-cross kernel of config C4 (ranks 16), rebuilt from its stored cross skeleton"
    else:  # same shape, seeded cores (the cost depends on the ranks only)
        rng = np.random.default_rng(0)
        r = 16
        d3 = (rng.random((1, N, r)), rng.random((r, N, r)) / r, rng.random((r, N, 1)))
        source = "TT d=3 ranks (1,16,16,1) seeded cores (config C4's shape)"
    ks = g.KernelSet({2: g.TTKernel(construct.c4_d2_cores(N)), 3: g.TTKernel(d3)})
    del d3
    dks = [ctx.device_kernel(ks[d]) for d in ks.orders]
    n = torch.zeros(N, dtype=torch.float64, device=dev)
    n[0] = 1.0
    p = torch.empty_like(n)
    q = torch.empty_like(n)
    s = torch.empty_like(n)
    sp = stream.cuda_stream
    for _ in range(3):
        ctx.rhs_device(dks, n.data_ptr(), p.data_ptr(), q.data_ptr(), s.data_ptr(), sp)
    torch.cuda.synchronize(dev)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for _ in range(steps):
        ctx.rhs_device(dks, n.data_ptr(), p.data_ptr(), q.data_ptr(), s.data_ptr(), sp)
    b.record(stream)
    torch.cuda.synchronize(dev)
    ms = a.elapsed_time(b) / steps
    return {"ms_per_rhs": ms, "rhs_per_s": 1000.0 / ms, "unit": UNIT,
            "workload": f"config C4: D=3, N=2^20, monodisperse; d=3: {source}; d=2: exact rank-3 TT; fp64",
            "note": "CUDA events on the launching stream, inputs resident"}


# --------------------------------------------------------------------------
# more of the metric: the other configs and D at N = 2^20 (single GPU)
# --------------------------------------------------------------------------
def _timed_rhs(ctx, dks, n_np, dev, stream, calls, warm=3):
    import torch

    N = n_np.size
    n = torch.from_numpy(n_np).to(dev)
    p, q, s = (torch.empty_like(n) for _ in range(3))
    sp = stream.cuda_stream
    for _ in range(warm):
        ctx.rhs_device(dks, n.data_ptr(), p.data_ptr(), q.data_ptr(), s.data_ptr(), sp)
    torch.cuda.synchronize(dev)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for _ in range(calls):
        ctx.rhs_device(dks, n.data_ptr(), p.data_ptr(), q.data_ptr(), s.data_ptr(), sp)
    b.record(stream)
    torch.cuda.synchronize(dev)
    del N
    return a.elapsed_time(b) / calls


def _rk2_rate(ctx, dks, n_np, dt, steps):
    """Fused device RK2 (ttagg_rk2, one CUDA graph per step): steps/s over the
    whole call (H2D, capture, final D2H included) and per step by differencing
    a 1-step call (fixed costs removed)."""
    import torch

    ctx.rk2_host(dks, n_np, 0.0, dt, 2, 1)  # warm-up
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ctx.rk2_host(dks, n_np, 0.0, dt, 1, 1)
    t1 = time.perf_counter() - t0
    t0 = time.perf_counter()
    _, _, fail, _ = ctx.rk2_host(dks, n_np, 0.0, dt, steps, steps)
    tn = time.perf_counter() - t0
    per = (tn - t1) / max(steps - 1, 1)
    return {"steps_per_s": steps / tn, "steps_per_s_marginal": 1.0 / per if per > 0 else None,
            "steps": steps, "fail_step": fail}


def extras(ctx, dev, stream, peak, steps):
    """RHS/s and RK2 steps/s over the rest of BASELINE.json's configs and D =
    3..5 at N = 2^20, each with its model-byte fraction of the HBM peak."""
    import paper_1905_09071_b200 as g
    from paper_1905_09071_b200.workloads import CONFIGS, initial_state, permutation_power_cp

    out = {}

    def cp_set(exps, orders, N):
        ks = g.KernelSet({d: g.CPKernel(permutation_power_cp(exps[:d], N)) for d in orders})
        dks = [ctx.device_kernel(ks[d]) for d in ks.orders]
        cols = {d: d * math.factorial(d) for d in orders}
        tails = {d: math.factorial(d) for d in orders}
        return ks, dks, model_bytes(N, cols, tails)["B_RHS"]

    def frac(bytes_, ms):
        return bytes_ / (ms * 1e-3) / 1e9 / peak

    c5 = CONFIGS["C5"]
    N = 1 << 20
    # opt-in deduplication (ttagg_cp_upload_dedup) on the C5 tensor itself: the
    # permutation-power factors hold d distinct vectors per order, so pass A
    # transforms <= d^2 distinct column pairs instead of d R / 2; same results
    # (bitwise), reported apart from the headline (which evaluates every rank term)
    dks = [ctx.upload_cp(permutation_power_cp(c5.exponents[:d], N), dedup=True) for d in c5.orders]
    ms = _timed_rhs(ctx, dks, initial_state("c5", N), dev, stream, steps)
    out["c5_dedup"] = {"rhs_per_s": 1e3 / ms, "ms_per_rhs": ms,
                       "workload": "C5 tensor (D=5, N=2^20, CP ranks 2/6/24/120) with identical factor columns "
                                   "stored and transformed once (opt-in; same RHS bitwise)"}
    del dks
    # D = 4 at N = 2^20 (orders 2..4, CP ranks 2/6/24, the C5 exponents / state)
    ks, dks, B = cp_set(c5.exponents, (2, 3, 4), N)
    ms = _timed_rhs(ctx, dks, initial_state("c5", N), dev, stream, steps)
    # RK2 at the same size (mass-normalised state, the C5 step size; 20 steps)
    r4 = _rk2_rate(ctx, dks, initial_state("c5", N, normalised=True), c5.dt, 20)
    r4["model_frac_marginal"] = (frac(2 * B, 1e3 / r4["steps_per_s_marginal"])
                                 if r4["steps_per_s_marginal"] else None)
    out["d4_n2p20"] = {"rhs_per_s": 1e3 / ms, "ms_per_rhs": ms, "model_frac": frac(B, ms), "rk2": r4,
                       "workload": "D=4 (d=2..4), N=2^20, CP ranks 2/6/24 (C5 exponents and state); "
                                   "RK2 dt=0.002, 20 steps (normalised state)"}
    del ks, dks
    # C2: 1000 back-to-back RHS calls at N = 65536, D = 3
    c2 = CONFIGS["C2"]
    ks, dks, B = cp_set(c2.exponents, c2.orders, c2.n_classes)
    ms = _timed_rhs(ctx, dks, initial_state("c2", c2.n_classes), dev, stream, 1000)
    out["c2"] = {"rhs_per_s": 1e3 / ms, "ms_per_rhs": ms, "calls": 1000, "model_frac": frac(B, ms),
                 "workload": "C2: D=3, N=65536, CP ranks 2/6, 1000 calls (L2-resident: absolute rate only)"}
    # C1: RK2, 100 steps at N = 4096, monodisperse
    c1 = CONFIGS["C1"]
    ks, dks, B = cp_set(c1.exponents, c1.orders, c1.n_classes)
    out["c1_rk2"] = dict(_rk2_rate(ctx, dks, initial_state("mono", c1.n_classes), c1.dt, c1.steps),
                         workload="C1: D=3, N=4096, dt=0.01, 100 steps (launch-bound)")
    # C3: RHS/s and RK2 200 steps at N = 2^18, D = 4 (mass-normalised state: the
    # literal one diverges in the reference at step 2)
    c3 = CONFIGS["C3"]
    ks, dks, B = cp_set(c3.exponents, c3.orders, c3.n_classes)
    ms = _timed_rhs(ctx, dks, initial_state("exp256", c3.n_classes), dev, stream, steps)
    r = _rk2_rate(ctx, dks, initial_state("exp256", c3.n_classes, normalised=True), c3.dt, c3.steps)
    r["model_frac_marginal"] = (frac(2 * B, 1e3 / r["steps_per_s_marginal"])
                                if r["steps_per_s_marginal"] else None)
    out["c3"] = {"rhs_per_s": 1e3 / ms, "ms_per_rhs": ms, "model_frac": frac(B, ms), "rk2": r,
                 "workload": "C3: D=4, N=2^18, CP ranks 2/6/24; RK2 dt=0.005, 200 steps (normalised state)"}
    return out


def free_port():
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def launch_ranks(args) -> int:
    """`--gpus N` outside a torchrun environment: start N ranks (one process
    per GPU, NCCL) with torchrun on this node and relay the exit code."""
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    env.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={free_port()}", os.path.abspath(__file__), *sys.argv[1:]]
    print(f"[bench] launching {args.gpus} ranks: {' '.join(cmd)}", file=sys.stderr, flush=True)
    return subprocess.call(cmd, env=env)


# --------------------------------------------------------------------------
# GPU arm
# --------------------------------------------------------------------------
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=("ours", "reference"))
    ap.add_argument("--n-classes", type=int, default=1 << 20)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-c4", action="store_true", help="skip the D=3 TT (config C4 shape) RHS timing")
    ap.add_argument("--no-extras", action="store_true", help="skip the other configs' timings")
    ap.add_argument("--rk2-steps", type=int, default=50)  # config C5: dt = 0.002, 50 steps
    ap.add_argument("--launcher-selftest", action="store_true", help=argparse.SUPPRESS)
    ap.add_argument("--sharded", action="store_true",
                    help="use the rank-sharded multi-GPU code path (perm layout + all-reduce) even at 1 GPU")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    if args.gpus < 1:
        ap.error("--gpus must be >= 1")
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        sys.exit(launch_ranks(args))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        print(f"[bench] --gpus {args.gpus} but WORLD_SIZE={world}: refusing to report a mismatched n_gpus",
              file=sys.stderr)
        sys.exit(2)
    if args.launcher_selftest:  # the launch plumbing alone (gloo, no GPU): tests/test_host.py
        import torch
        import torch.distributed as dist

        dist.init_process_group("gloo")
        t = torch.tensor([float(rank), float(local), float(world)])
        got = [torch.zeros(3) for _ in range(world)]
        dist.all_gather(got, t)
        ms = torch.tensor([1.0 + rank])
        dist.all_reduce(ms, op=dist.ReduceOp.MAX)  # the max-over-ranks timing reduction
        if rank == 0:
            print(json.dumps({"launcher_selftest": True, "n_gpus": world,
                              "ranks": [[int(x) for x in v.tolist()] for v in got], "max_ms": float(ms)}), flush=True)
        dist.destroy_process_group()
        return

    from paper_1905_09071_b200.workloads import CONFIGS, initial_state, permutation_power_cp

    cfg = CONFIGS["C5"]
    N = args.n_classes
    n0 = initial_state("c5", N)

    if args.impl == "reference":
        if rank != 0:
            return
        factors = {d: permutation_power_cp(cfg.exponents[:d], N) for d in cfg.orders}
        run_reference(args, N, factors, n0)
        return

    import torch

    if torch.cuda.device_count() < world:
        print(f"[bench] {world} ranks but {torch.cuda.device_count()} visible GPUs", file=sys.stderr)
        sys.exit(2)
    torch.cuda.set_device(local)
    sharded = world > 1 or args.sharded
    if sharded and "RANK" in os.environ:
        import torch.distributed as dist

        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    os.environ["TTAGG_DEVICE"] = str(local)

    import paper_1905_09071_b200 as g
    from paper_1905_09071_b200 import _lib
    from paper_1905_09071_b200.dist import CudaEngine, DistRHS

    ctx = _lib.get_context(local)
    shards = g.lpt_rank_shards({d: math.factorial(d) for d in cfg.orders}, world)[rank]
    factors = {d: permutation_power_cp(cfg.exponents[:d], N) for d in cfg.orders}
    dks, cols, tails = [], {}, {}
    for d in cfg.orders:
        sub = shards.get(d, [])
        if not sub:
            continue
        dk = ctx.upload_cp(factors[d], rank_subset=sub if sharded else None)
        dks.append(dk)
        cols[d] = d * len(sub)
        tails[d] = len(sub)
    Np, N1, N2 = _lib.geometry(N)
    dev = torch.device("cuda", local)
    stream = torch.cuda.current_stream(dev)
    sp = stream.cuda_stream
    n_t = torch.from_numpy(n0).to(dev)
    p_t = torch.empty(N, dtype=torch.float64, device=dev)
    q_t = torch.empty_like(p_t)
    s_t = torch.empty_like(p_t)
    nperm = torch.zeros(Np, dtype=torch.float64, device=dev)
    sperm = torch.zeros(Np, dtype=torch.float64, device=dev)
    if sharded:
        ctx.permute(N, n_t.data_ptr(), nperm.data_ptr(), 0, sp)
    dist_on = sharded and torch.distributed.is_available() and torch.distributed.is_initialized()

    def step():
        if not sharded:
            ctx.rhs_device(dks, n_t.data_ptr(), p_t.data_ptr(), q_t.data_ptr(), s_t.data_ptr(), sp)
        else:
            ctx.rhs_perm(dks, nperm.data_ptr(), None, 0.0, sperm.data_ptr(), sp)
            if dist_on:
                torch.distributed.all_reduce(sperm)

    def barrier():
        if dist_on:
            torch.distributed.barrier()

    def max_over_ranks(x: float) -> float:
        if not dist_on:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        return float(t.item())

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize(dev)
    ctx.profile_read()  # drop warm-up records
    launches0 = ctx.launch_count()
    ctx.profile(True)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clocks:
        barrier()
        torch.cuda.synchronize(dev)
        ev0.record(stream)
        for _ in range(args.steps):
            step()
        ev1.record(stream)
        torch.cuda.synchronize(dev)
        barrier()
    ctx.profile(False)
    launches = ctx.launch_count() - launches0
    ms = max_over_ranks(ev0.elapsed_time(ev1))
    prof = ctx.profile_read()
    ms_step = ms / args.steps
    value = 1000.0 / ms_step

    # ---- end to end through the public API (host buffers, copies inside)
    e2e = None
    if not args.no_e2e:
        if not sharded:
            ks = g.KernelSet({d: g.CPKernel(factors[d]) for d in cfg.orders})
            st = g.ConcentrationState(n0)
            for _ in range(max(4, args.warmup)):
                g.rhs_total(ks, st)
            n_e2e = max(args.steps, 20)  # host-side timing: more calls than the device loop
            t0 = time.perf_counter()
            for _ in range(n_e2e):
                r = g.rhs_total(ks, st)
            te = (time.perf_counter() - t0) / n_e2e
            del r
            # where the time goes: the library call alone, and the two PCIe copies
            dkc = [ctx.device_kernel(ks[d]) for d in ks.orders]
            t0 = time.perf_counter()
            for _ in range(5):
                ctx.rhs_host(dkc, n0)
            th = (time.perf_counter() - t0) / 5
            hb = torch.empty(3 * N, dtype=torch.float64).pin_memory()
            db = torch.empty(3 * N, dtype=torch.float64, device=dev)
            a, b, c = (torch.cuda.Event(enable_timing=True) for _ in range(3))
            for _ in range(2):  # first-touch of the page-locked buffer out of the timing
                db[:N].copy_(hb[:N], non_blocking=True)
                hb.copy_(db, non_blocking=True)
            torch.cuda.synchronize(dev)
            a.record(stream)
            db[:N].copy_(hb[:N], non_blocking=True)
            b.record(stream)
            hb.copy_(db, non_blocking=True)
            c.record(stream)
            torch.cuda.synchronize(dev)
            h2d, d2h = a.elapsed_time(b), b.elapsed_time(c)
            e2e = {"value": 1.0 / te, "unit": UNIT, "h2d_bytes_per_step": 8 * N,
                   "d2h_bytes_per_step": 24 * N, "api": "paper_1905_09071_b200.rhs_total (numpy in, p/q/s out)",
                   "breakdown_ms": {"rhs_total_call": te * 1e3, "library_call": th * 1e3,
                                    "device_rhs": ms_step, "h2d_8MB": h2d, "d2h_24MB": d2h,
                                    "host_rest": te * 1e3 - ms_step - h2d - d2h}}
        else:
            host_n = torch.from_numpy(n0).pin_memory()
            host_s = torch.empty(N, dtype=torch.float64).pin_memory()
            for _ in range(2):
                n_t.copy_(host_n, non_blocking=True)
                ctx.permute(N, n_t.data_ptr(), nperm.data_ptr(), 0, sp)
                step()
                ctx.permute(N, sperm.data_ptr(), s_t.data_ptr(), 1, sp)
                host_s.copy_(s_t, non_blocking=True)
            torch.cuda.synchronize(dev)
            barrier()
            t0 = time.perf_counter()
            for _ in range(args.steps):
                n_t.copy_(host_n, non_blocking=True)
                ctx.permute(N, n_t.data_ptr(), nperm.data_ptr(), 0, sp)
                step()
                ctx.permute(N, sperm.data_ptr(), s_t.data_ptr(), 1, sp)
                host_s.copy_(s_t, non_blocking=True)
                torch.cuda.synchronize(dev)
            te = max_over_ranks((time.perf_counter() - t0) / args.steps)
            e2e = {"value": 1.0 / te, "unit": UNIT, "h2d_bytes_per_step": 8 * N,
                   "d2h_bytes_per_step": 8 * N, "api": "ttagg_rhs_perm + NCCL all-reduce (pinned host buffers)"}

    # ---- D = 3 at N = 2^20 through the TT route (config C4 shape), single GPU
    c4 = None
    if not sharded and not args.no_c4 and N == 1 << 20:
        c4 = c4_tt_timing(ctx, N, dev, stream, args.steps)

    # ---- RK2 steps/s over the C5 trajectory (mass-normalised state)
    rk2 = None
    if args.rk2_steps > 0:
        nn = initial_state("c5", N, normalised=True)
        if not sharded:
            rk2 = _rk2_rate(ctx, dks, nn, cfg.dt, args.rk2_steps)
            rk2["note"] = ("ttagg_rk2 over the C5 trajectory length (mass-normalised C5 state, CUDA graph "
                           "per step); steps_per_s includes H2D, capture and the final D2H")
        else:
            eng = CudaEngine({d: factors[d] for d in cfg.orders}, shards, N, local)
            drhs = DistRHS(eng)
            drhs.rk2(nn, 0.0, cfg.dt, 1)  # warm-up
            torch.cuda.synchronize(dev)
            barrier()
            t0 = time.perf_counter()
            res = drhs.rk2(nn, 0.0, cfg.dt, args.rk2_steps, args.rk2_steps)
            torch.cuda.synchronize(dev)
            trk = max_over_ranks(time.perf_counter() - t0)
            rk2 = {"steps_per_s": args.rk2_steps / trk, "steps": args.rk2_steps, "fail_step": res.fail_step,
                   "note": f"rank-sharded RK2 over {world} GPUs (dist.DistRHS: one NCCL all-reduce per RHS, "
                           "replicated stage updates; H2D and final D2H included); max over ranks"}
            del eng

    if rank != 0:
        if dist_on:
            torch.distributed.destroy_process_group()
        return

    # ---- roofline of the dominant kernel (CUDA events over the timed region)
    peak, peak_kind = _peaks()
    model = model_bytes(N, cols, tails)
    # dominant kernel = most algorithmic bytes (the costliest order's pass A); its
    # events sit on the high-priority stream, so its intervals are its own runtime
    cands = [((model["passA"] if k[0] == 0 else model["passB"])[k[1]], k) for k in prof if k[0] in (0, 1)]
    roof = None
    if cands:
        cls, d = max(cands)[1]
        tot_ms, cnt = prof[(cls, d)]
        per_ms = tot_ms / cnt
        bytes_launch = (model["passA"] if cls == 0 else model["passB"])[d]
        achieved = bytes_launch / (per_ms * 1e-3) / 1e9
        kname = f"pass{'AB'[cls]} d={d}"
        traffic = None
        tsrc = None
        for fname in ("r02_roofline_traffic.json", "r01_roofline_traffic.json"):
            try:  # DRAM bytes of the same kernel from the committed ncu --set full capture
                with open(os.path.join(ROOT, "profiles", fname)) as fh:
                    tk = json.load(fh)["kernels"].get(kname)
                if tk and N == 1 << 20 and world == 1:
                    traffic, tsrc = tk["dram_bytes"], f"profiles/{fname} (ncu dram__bytes_read+write per launch)"
                    break
            except Exception:
                pass
        roof = {"bound": "hbm", "kernel": kname, "achieved": achieved, "peak": peak,
                "unit": "GB/s", "frac": achieved / peak, "traffic": traffic, "peak_kind": peak_kind,
                "launch_ms": per_ms, "bytes_per_launch": bytes_launch, "traffic_source": tsrc}
    rhs_gbs = model["B_RHS"] / (ms_step * 1e-3) / 1e9
    breakdown = {f"{'ABCO'[c]}{d}": round(v[0] / args.steps, 4) for (c, d), v in sorted(prof.items())}

    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        n_cpu = os.cpu_count() or 1
        t_cpu = cpu_whole_rhs(factors, n0, n_cpu)
        cpu = {"value": 1.0 / t_cpu, "unit": UNIT, "cores": n_cpu, "kind": "port",
               "sample": cpu_sample_desc(factors, n_cpu), "seconds": t_cpu}

    more = None
    if world == 1 and not sharded and not args.no_extras and N == 1 << 20:
        more = extras(ctx, dev, stream, peak, args.steps)

    line = {
        "metric": METRIC,
        "value": value * 1.0,
        "unit": UNIT,
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms_step,
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": WORKLOAD,
                   "l2": "inputs larger than L2 (6 GB factors, 25 GB exchange)",
                   "parallelism": f"rank-sharded x{world} (NCCL all-reduce per RHS)" if sharded else "1 GPU",
                   "geometry": {"Np": Np, "N1": N1, "N2": N2}},
        "roofline": roof,
        "rhs_model": {"B_RHS_GB": model["B_RHS"] / 1e9, "B_min_GB": model["B_min"] / 1e9,
                      "achieved_GBs": rhs_gbs, "frac_of_peak": rhs_gbs / peak,
                      "fp64_TFLOPs": fp64_flops(N, cols) / (ms_step * 1e-3) / 1e12,
                      "note": "model bytes of rank 0's shard" if sharded and world > 1 else "whole RHS"},
        "kernel_ms_per_step": breakdown,
        "kernel_ms_note": "CUDA-event intervals on each launch stream (A/B/C = pass, O = qcoef/combine); the cheaper orders' pass B/C sit on a least-priority stream that only gets SMs the costliest order leaves idle, so their intervals span that wait",
        "cpu_baseline": cpu,
        "e2e": e2e,
        "rk2": rk2,
        "c4_tt": c4,
        "extras": more,
        "gpu_launches": launches,
        "clocks": clocks.summary(),
    }
    print(json.dumps(line), flush=True)
    if dist_on:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
