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
def cpu_sample(N, factors_by_order, n0, frac=0.05, workers=None):
    """Time a bounded sample of one RHS on the host cores: a `frac` share of the
    rank terms of every order (>= 1) through the reference algorithm, losses in
    full; returns (extrapolated seconds per RHS, description)."""
    from oracle import rhs_oracle as orc

    workers = workers or os.cpu_count() or 1
    total = 0.0
    parts = []
    for d, fs in sorted(factors_by_order.items()):
        R = fs[0].shape[1]
        rs = max(1, int(math.ceil(R * frac)))
        t0 = time.perf_counter()
        orc.cp_gain(fs, n0, workers=workers, ranks=np.arange(rs))
        tg = time.perf_counter() - t0
        t0 = time.perf_counter()
        orc.cp_loss(fs, n0)
        tl = time.perf_counter() - t0
        total += tg * R / rs + tl
        parts.append(f"d={d}:{rs}/{R} ranks")
    return total, "gain over " + ", ".join(parts) + " (scaled to all ranks) + full losses"


def run_reference(args, N, factors_by_order, n0):
    workers = os.cpu_count() or 1
    for _ in range(args.warmup):
        cpu_sample(N, factors_by_order, n0, workers=workers)
    times = []
    desc = ""
    for _ in range(args.steps):
        t, desc = cpu_sample(N, factors_by_order, n0, workers=workers)
        times.append(t)
    t_rhs = statistics.median(times)
    value = 1.0 / t_rhs
    line = {
        "impl": "reference",
        "metric": METRIC,
        "value": value,
        "unit": UNIT,
        "n_gpus": args.gpus,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": t_rhs * 1e3,
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": "C5: D=5 (d=2..5), N=2^20, permutation-power CP ranks 2/6/24/120, fp64",
                   "l2": "inputs larger than L2"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": workers, "kind": "port",
                         "sample": desc + "; oracle/rhs_oracle.py restates rhs.py:345-414 on scipy.fft"},
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
    ap.add_argument("--rk2-steps", type=int, default=50)  # config C5: dt = 0.002, 50 steps
    ap.add_argument("--sharded", action="store_true",
                    help="use the rank-sharded multi-GPU code path (perm layout + all-reduce) even at 1 GPU")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

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

    torch.cuda.set_device(local)
    sharded = world > 1 or args.sharded
    if sharded and "RANK" in os.environ:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    os.environ["TTAGG_DEVICE"] = str(local)

    import paper_1905_09071_b200 as g
    from paper_1905_09071_b200 import _lib

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
    ms = ev0.elapsed_time(ev1)
    if dist_on:
        t = torch.tensor([ms], dtype=torch.float64, device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t.item())
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
            e2e = {"value": 1.0 / te, "unit": UNIT, "h2d_bytes_per_step": 8 * N,
                   "d2h_bytes_per_step": 24 * N, "api": "paper_1905_09071_b200.rhs_total (numpy in, p/q/s out)"}
            del r
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
            te = (time.perf_counter() - t0) / args.steps
            if dist_on:
                tt = torch.tensor([te], dtype=torch.float64, device=dev)
                torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
                te = float(tt.item())
            e2e = {"value": 1.0 / te, "unit": UNIT, "h2d_bytes_per_step": 8 * N,
                   "d2h_bytes_per_step": 8 * N, "api": "ttagg_rhs_perm + NCCL all-reduce (pinned host buffers)"}

    # ---- RK2 steps/s (fused device-resident integrator), single GPU
    # ---- D = 3 at N = 2^20 through the TT route (config C4 shape), single GPU
    c4 = None
    if not sharded and not args.no_c4 and N == 1 << 20:
        c4 = c4_tt_timing(ctx, N, dev, stream, args.steps)

    rk2 = None
    if not sharded and args.rk2_steps > 0:
        nn = initial_state("c5", N, normalised=True)
        ctx.rk2_host(dks, nn, 0.0, cfg.dt, 1, 1)  # warm-up / graph shapes
        torch.cuda.synchronize(dev)
        t0 = time.perf_counter()
        _, _, fail, _ = ctx.rk2_host(dks, nn, 0.0, cfg.dt, args.rk2_steps, args.rk2_steps)
        trk = time.perf_counter() - t0
        rk2 = {"steps_per_s": args.rk2_steps / trk, "steps": args.rk2_steps, "fail_step": fail,
               "note": "ttagg_rk2 over the C5 trajectory length (mass-normalised C5 state, CUDA graph per step, incl. capture, H2D and final D2H)"}

    if rank != 0:
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
        try:  # DRAM bytes of the same kernel from the committed ncu --set full capture
            with open(os.path.join(ROOT, "profiles", "r01_roofline_traffic.json")) as fh:
                tk = json.load(fh)["kernels"].get(kname)
            if tk and N == 1 << 20:
                traffic = tk["dram_bytes"]
        except Exception:
            pass
        roof = {"bound": "hbm", "kernel": kname, "achieved": achieved, "peak": peak,
                "unit": "GB/s", "frac": achieved / peak, "traffic": traffic, "peak_kind": peak_kind,
                "launch_ms": per_ms, "bytes_per_launch": bytes_launch,
                "traffic_source": "profiles/r01_roofline_traffic.json (ncu dram__bytes_read+write per launch)"}
    rhs_gbs = model["B_RHS"] / (ms_step * 1e-3) / 1e9
    breakdown = {f"{'ABCO'[c]}{d}": round(v[0] / args.steps, 4) for (c, d), v in sorted(prof.items())}

    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        n_cpu = os.cpu_count() or 1
        t_cpu, desc = cpu_sample(N, factors, n0, workers=n_cpu)
        cpu = {"value": 1.0 / t_cpu, "unit": UNIT, "cores": n_cpu, "kind": "port",
               "sample": desc + "; oracle/rhs_oracle.py restates rhs.py:345-414 on scipy.fft"}

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
        "config": {"workload": "C5: D=5 (d=2..5), N=2^20, permutation-power CP ranks 2/6/24/120, fp64",
                   "l2": "inputs larger than L2 (6 GB factors, 25 GB exchange)",
                   "parallelism": f"rank-sharded x{world} (NCCL all-reduce per RHS)" if sharded else "1 GPU",
                   "geometry": {"Np": Np, "N1": N1, "N2": N2}},
        "roofline": roof,
        "rhs_model": {"B_RHS_GB": model["B_RHS"] / 1e9, "B_min_GB": model["B_min"] / 1e9,
                      "achieved_GBs": rhs_gbs, "frac_of_peak": rhs_gbs / peak,
                      "fp64_TFLOPs": fp64_flops(N, cols) / (ms_step * 1e-3) / 1e12},
        "kernel_ms_per_step": breakdown,
        "kernel_ms_note": "CUDA-event intervals on each launch stream (A/B/C = pass, O = qcoef/combine); the cheaper orders' pass B/C sit on a least-priority stream that only gets SMs the costliest order leaves idle, so their intervals span that wait",
        "cpu_baseline": cpu,
        "e2e": e2e,
        "rk2": rk2,
        "c4_tt": c4,
        "gpu_launches": launches,
        "clocks": clocks.summary(),
    }
    print(json.dumps(line), flush=True)
    if dist_on:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
