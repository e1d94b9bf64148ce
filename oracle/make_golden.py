"""Generate golden fixtures by running the REFERENCE package itself.

Run in the build container only (it needs the read-only reference tree):

    PYTHONPATH=/root/reference/pkg/src PYTHONDONTWRITEBYTECODE=1 \
        python oracle/make_golden.py

Every array written here is an output of ``ttagg`` v0.1.0's own operators
(``rhs_cp_P/Q``, ``rhs_tt_P/Q``, ``rhs_total``, ``integrate``), evaluated on
inputs built by ``paper_1905_09071_b200.workloads`` (seeded) or by the
reference's own builders.  The fixtures pin both the oracle restatement
(``oracle/rhs_oracle.py``) and, on the GPU box, the CUDA path.

Large vectors (N >= 2^18) are stored as index samples plus full-vector
moment checksums, keeping the committed fixtures small.
"""

from __future__ import annotations

import math
import os
import sys
import time
import warnings

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, "/root/reference/pkg/src")

import ttagg  # noqa: E402  (the reference, read-only)
from ttagg import (  # noqa: E402
    BrownianSpec,
    ConcentrationState,
    CPKernel,
    ExecutionPlan,
    InitialCondition,
    KernelSet,
    SimulationConfig,
    StepFailureError,
    TimeGrid,
    TTKernel,
    build_brownian_tt,
    constant_cp,
    constant_tt,
    integrate,
    rhs_cp_P,
    rhs_cp_Q,
    rhs_total,
    rhs_tt_P,
    rhs_tt_Q,
)

from oracle.tt_svd import tt_svd  # noqa: E402
from paper_1905_09071_b200.workloads import (  # noqa: E402
    CONFIGS,
    initial_state,
    permutation_power_cp,
)

OUT = os.path.join(ROOT, "tests", "golden")
WORKERS = min(8, os.cpu_count() or 1)
PLAN = ExecutionPlan(workers=WORKERS)


def sample_indices(n_classes: int) -> np.ndarray:
    """First 1024 sizes, then a geometric-ish sweep, plus the last sizes."""
    head = np.arange(min(1024, n_classes))
    sweep = np.unique(np.round(np.geomspace(1024, n_classes - 1, 1500)).astype(np.int64))
    tail = np.arange(max(0, n_classes - 64), n_classes)
    return np.unique(np.concatenate([head, sweep, tail]))


def checksums(v: np.ndarray) -> np.ndarray:
    k = np.arange(1, v.size + 1, dtype=np.float64)
    return np.array([v.sum(), k @ v, (k * k) @ v, np.abs(v).sum(), np.abs(v).max()])


def cp_set(factors_by_order):
    return KernelSet({d: CPKernel(f) for d, f in factors_by_order.items()})


def save(name, **arrays):
    path = os.path.join(OUT, name)
    np.savez_compressed(path, **arrays)
    print(f"wrote {path} ({os.path.getsize(path) / 1024:.0f} KiB)", flush=True)


# ---------------------------------------------------------------------------
# unit cases: mirror the reference test suite's oracle tests
# ---------------------------------------------------------------------------

def unit_case():
    out = {}
    # CP with random factors (test_rhs.py:210-219 shape), d = 2, 3, 4, 5, N = 32
    for order in (2, 3, 4, 5):
        rng = np.random.default_rng(order * 43)
        n_classes = 32
        factors = tuple(rng.random((n_classes, 4)) for _ in range(order))
        cp = CPKernel(factors)
        for f_i, f in enumerate(factors):
            out[f"cp{order}_f{f_i}"] = f
        for s in range(3):
            state = ConcentrationState(rng.random(n_classes))
            out[f"cp{order}_n{s}"] = state.n
            out[f"cp{order}_P{s}"] = rhs_cp_P(cp, state)
            out[f"cp{order}_Q{s}"] = rhs_cp_Q(cp, state)
    # odd CP ranks and odd N (ragged): d = 3, R = 5, N = 37 and d = 2, R = 1, N = 2
    for tag, order, n_classes, rank, seed in (("cpodd", 3, 37, 5, 7), ("cptiny", 2, 2, 1, 8)):
        rng = np.random.default_rng(seed)
        factors = tuple(rng.random((n_classes, rank)) for _ in range(order))
        state = ConcentrationState(rng.random(n_classes))
        for f_i, f in enumerate(factors):
            out[f"{tag}_f{f_i}"] = f
        out[f"{tag}_n"] = state.n
        out[f"{tag}_P"] = rhs_cp_P(CPKernel(factors), state)
        out[f"{tag}_Q"] = rhs_cp_Q(CPKernel(factors), state)
    # TT Brownian (test_rhs.py:171-181 shape), d = 2, 3, 4, N = 32
    for order in (2, 3, 4):
        rng = np.random.default_rng(order * 31)
        n_classes = 32
        spec = BrownianSpec(tuple(rng.uniform(-1, 1, size=order)))
        tt = build_brownian_tt(spec, n_classes)
        out[f"tt{order}_mu"] = np.array(spec.exponents)
        for c_i, c in enumerate(tt.cores):
            out[f"tt{order}_c{c_i}"] = c
        for s in range(3):
            state = ConcentrationState(rng.random(n_classes))
            out[f"tt{order}_n{s}"] = state.n
            out[f"tt{order}_P{s}"] = rhs_tt_P(tt, state)
            out[f"tt{order}_Q{s}"] = rhs_tt_Q(tt, state)
    # mixed orders TT (test_rhs.py:240-263)
    rng = np.random.default_rng(47)
    n_classes = 32
    ks = KernelSet(
        {
            2: build_brownian_tt(BrownianSpec((0.25, -0.25)), n_classes),
            3: build_brownian_tt(BrownianSpec((1 / 3, -1 / 3, 0.0)), n_classes),
        }
    )
    state = ConcentrationState(rng.random(n_classes))
    res = rhs_total(ks, state, breakdown=True)
    out["mixed_n"] = state.n
    out["mixed_p"], out["mixed_q"], out["mixed_s"] = res.p, res.q, res.s
    # mixed CP + TT in one set (d=2 CP, d=3 TT), N = 48
    rng = np.random.default_rng(91)
    n_classes = 48
    cpf = permutation_power_cp((0.2, -0.3), n_classes)
    tt3 = build_brownian_tt(BrownianSpec((0.3, -0.2, 0.1)), n_classes)
    state = ConcentrationState(rng.random(n_classes))
    res = rhs_total(KernelSet({2: CPKernel(cpf), 3: tt3}), state)
    out["mix2_n"] = state.n
    out["mix2_p"], out["mix2_q"], out["mix2_s"] = res.p, res.q, res.s
    # known answers (test_rhs.py:87-110, 226-232)
    n = np.zeros(8)
    n[0] = 1.0
    out["ka_s2"] = rhs_total(KernelSet({2: constant_tt(1.0, 2, 8)}), ConcentrationState(n)).s
    out["ka_p3"] = rhs_cp_P(constant_cp(1.0, 3, 8), ConcentrationState(n))
    out["ka_q3"] = rhs_cp_Q(constant_cp(1.0, 3, 8), ConcentrationState(n))
    # constant-kernel self convolution (test_rhs.py:147-157)
    rng = np.random.default_rng(23)
    n = rng.random(16)
    out["conv_n"] = n
    out["conv_P"] = rhs_tt_P(constant_tt(1.75, 3, 16), ConcentrationState(n))
    save("unit.npz", **out)


# ---------------------------------------------------------------------------
# configuration-shaped cases (BASELINE.json configs)
# ---------------------------------------------------------------------------

def _cfg(n_classes, D, dt, steps, record_every, n0):
    return SimulationConfig(
        n_classes=n_classes,
        dimension=D,
        kernel_specs={D: BrownianSpec(tuple([0.0] * D))},  # placeholder; kernels= overrides
        initial=InitialCondition.from_vector(n0),
        time=TimeGrid(0.0, dt, steps),
        record_every=record_every,
    )


def _run_traj(ks, n0, dt, steps, record_every):
    config = _cfg(n0.size, max(ks.orders), dt, steps, record_every, n0)
    with warnings.catch_warnings(record=True) as caught:
        warnings.simplefilter("always")
        try:
            final, series = integrate(config, kernels=ks, plan=PLAN)
            fail = 0
            rows = np.array(series.rows())
            nfinal = final.n
            neg = series.negativity_flagged
        except StepFailureError as exc:
            fail = exc.step_index
            rows = np.array(exc.series.rows())
            nfinal = np.zeros(0)
            neg = exc.series.negativity_flagged
    warned = any(issubclass(w.category, ttagg.StepSizeWarning) for w in caught)
    return dict(rows=rows, n_final=nfinal, fail_step=np.int64(fail),
                negativity=np.bool_(neg), warned=np.bool_(warned))


def c1_case():
    cfg = CONFIGS["C1"]
    ks = cp_set(cfg.cp_factors())
    n0 = initial_state("mono", cfg.n_classes)
    out = {}
    r = rhs_total(ks, ConcentrationState(n0), PLAN)
    out["p0"], out["q0"] = r.p, r.q
    rng = np.random.default_rng(5)
    nr = rng.random(cfg.n_classes) * np.exp(-np.arange(cfg.n_classes) / 300.0)
    r = rhs_total(ks, ConcentrationState(nr), PLAN, breakdown=True)
    out["nr"], out["pr"], out["qr"] = nr, r.p, r.q
    for d, (pd, qd) in r.by_order.items():
        out[f"pr_d{d}"], out[f"qr_d{d}"] = pd, qd
    t0 = time.perf_counter()
    traj = _run_traj(ks, n0, cfg.dt, cfg.steps, 10)
    print(f"C1 trajectory {time.perf_counter() - t0:.1f}s", flush=True)
    for k, v in traj.items():
        out["traj_" + k] = v
    save("c1.npz", **out)


def c2_case():
    cfg = CONFIGS["C2"]
    ks = cp_set(cfg.cp_factors())
    n0 = initial_state("c2", cfg.n_classes)
    t0 = time.perf_counter()
    r = rhs_total(ks, ConcentrationState(n0), PLAN)
    print(f"C2 RHS {time.perf_counter() - t0:.2f}s", flush=True)
    save("c2.npz", p=r.p, q=r.q)


def c3_case():
    cfg = CONFIGS["C3"]
    ks = cp_set(cfg.cp_factors())
    n0 = initial_state("exp256", cfg.n_classes)
    t0 = time.perf_counter()
    r = rhs_total(ks, ConcentrationState(n0), PLAN)
    print(f"C3 RHS {time.perf_counter() - t0:.2f}s", flush=True)
    idx = sample_indices(cfg.n_classes)
    out = dict(idx=idx, p=r.p[idx], q=r.q[idx], p_sums=checksums(r.p), q_sums=checksums(r.q))
    # literal trajectory: reference failure semantics
    t0 = time.perf_counter()
    traj = _run_traj(ks, n0, cfg.dt, 3, 1)
    print(f"C3 literal trajectory {time.perf_counter() - t0:.1f}s fail_step={traj['fail_step']}", flush=True)
    for k, v in traj.items():
        if k != "n_final":
            out["lit_" + k] = v
    # mass-normalised variant at reduced N, full 200 steps
    n_small = 1 << 12
    ks_s = cp_set(cfg.cp_factors(n_small))
    n0s = initial_state("exp256", n_small, normalised=True)
    traj = _run_traj(ks_s, n0s, cfg.dt, cfg.steps, 20)
    for k, v in traj.items():
        out["norm4096_" + k] = v
    save("c3.npz", **out)


def c5_case():
    cfg = CONFIGS["C5"]
    out = {}
    # cross-route check at N = 2^14: reference CP route on the permutation-power factors
    n_mid = 1 << 14
    ks_cp = cp_set(cfg.cp_factors(n_mid))
    n0m = initial_state("c5", n_mid)
    r = rhs_total(ks_cp, ConcentrationState(n0m), PLAN, breakdown=True)
    out["n16k_p"], out["n16k_q"] = r.p, r.q
    for d, (pd, qd) in r.by_order.items():
        out[f"n16k_p_d{d}"], out[f"n16k_q_d{d}"] = pd, qd
    # full N = 2^20, literal initial state: reference TT route on the same tensor
    # (build_brownian_tt(BrownianSpec(a[:d])) == permutation-power CP)
    n_classes = cfg.n_classes
    n0 = initial_state("c5", n_classes)
    idx = sample_indices(n_classes)
    out["idx"] = idx
    t0 = time.perf_counter()
    ks_tt = KernelSet(
        {d: build_brownian_tt(BrownianSpec(cfg.exponents[:d]), n_classes) for d in cfg.orders}
    )
    r = rhs_total(ks_tt, ConcentrationState(n0), PLAN, breakdown=True)
    print(f"C5 full-N TT-route RHS {time.perf_counter() - t0:.1f}s", flush=True)
    out["p"], out["q"] = r.p[idx], r.q[idx]
    out["p_sums"], out["q_sums"] = checksums(r.p), checksums(r.q)
    for d, (pd, qd) in r.by_order.items():
        out[f"p_d{d}"], out[f"q_d{d}"] = pd[idx], qd[idx]
    del ks_tt, r
    # literal failure semantics and normalised trajectory at reduced N = 2^12
    n_small = 1 << 12
    ks_s = cp_set(cfg.cp_factors(n_small))
    traj = _run_traj(ks_s, initial_state("c5", n_small), cfg.dt, 3, 1)
    for k, v in traj.items():
        if k != "n_final":
            out["lit4096_" + k] = v
    traj = _run_traj(ks_s, initial_state("c5", n_small, normalised=True), cfg.dt, cfg.steps, 5)
    for k, v in traj.items():
        out["norm4096_" + k] = v
    save("c5.npz", **out)


def c5traj_case():
    """The C5 trajectory at full size: N = 2^20, D = 5, dt = 0.002, 50 steps,
    on the mass-normalised state (the literal one diverges at step 2, SURVEY.md
    §8(d)), through the reference's own integrate() on its Brownian TT route
    (the same tensor as the permutation-power CP kernels; the CP route needs
    more memory than this container has).  Stored: sample indices of the
    final state, full-vector checksums and the moment rows (every 10 steps)."""
    cfg = CONFIGS["C5"]
    n_classes = cfg.n_classes
    ks_tt = KernelSet(
        {d: build_brownian_tt(BrownianSpec(cfg.exponents[:d]), n_classes) for d in cfg.orders}
    )
    n0 = initial_state("c5", n_classes, normalised=True)
    t0 = time.perf_counter()
    traj = _run_traj(ks_tt, n0, cfg.dt, cfg.steps, 10)
    print(f"C5 full-N trajectory {time.perf_counter() - t0:.1f}s", flush=True)
    idx = sample_indices(n_classes)
    save("c5traj.npz", idx=idx, n_final=traj["n_final"][idx], n_sums=checksums(traj["n_final"]),
         rows=traj["rows"], fail_step=traj["fail_step"], negativity=traj["negativity"], warned=traj["warned"])


def c3traj_case():
    """The C3 trajectory at full size: N = 2^18, D = 4, dt = 0.005, 200 steps,
    mass-normalised state (the literal one diverges at step 2), through the
    reference's own integrate() on its CP route.  Stored: sample indices of
    the final state, full-vector checksums and the moment rows (every 20)."""
    cfg = CONFIGS["C3"]
    n_classes = cfg.n_classes
    ks = cp_set(cfg.cp_factors())
    n0 = initial_state("exp256", n_classes, normalised=True)
    t0 = time.perf_counter()
    traj = _run_traj(ks, n0, cfg.dt, cfg.steps, 20)
    print(f"C3 full-N trajectory {time.perf_counter() - t0:.1f}s", flush=True)
    idx = sample_indices(n_classes)
    save("c3traj.npz", idx=idx, n_final=traj["n_final"][idx], n_sums=checksums(traj["n_final"]),
         rows=traj["rows"], fail_step=traj["fail_step"], negativity=traj["negativity"], warned=traj["warned"])


def c4traj_case():
    """Config C4 at full size: N = 2^20, D = 3, TT kernels (exact rank-3 d = 2,
    TT-cross d = 3 with ranks 16 from paper_1905_09071_b200.construct, the
    compressor the reference lacks), monodisperse state, dt = 0.01, through
    the reference's own integrate() on its TT route.  As literally specified
    (100 steps) it diverges: StepSizeWarning, then StepFailureError at step 9
    (explicit RK2 is unstable for the large sizes, whose loss rates reach
    dt * 4 k^(2/3) >> 1; FFT roundoff there grows every step).  Stored: the
    literal failure semantics, and a 2-step trajectory (record every step)
    whose final state is compared at sampled sizes plus checksums.  The d = 3
    cores are 2 GB, so the fixture stores the cross skeleton (I, J) that
    rebuilds them (construct.c4_d3_from_skeleton)."""
    from paper_1905_09071_b200 import construct

    n_classes = 1 << 20
    path = os.path.join(OUT, "c4traj.npz")
    t0 = time.perf_counter()
    if os.path.exists(path):  # reuse the skeleton of an earlier run (the cross takes minutes)
        old = np.load(path)
        I = [old["I0"], old["I1"], old["I2"]]
        J = [None, old["J1"], old["J2"], old["J3"]]
        cores3 = construct.c4_d3_from_skeleton(n_classes, I, J)
    else:
        _, cores3, (I, J) = construct.c4_kernels(n_classes, rank=16, return_skeleton=True)
    c1, c2 = construct.c4_d2_cores(n_classes)
    print(f"C4 cores {time.perf_counter() - t0:.1f}s ranks {[c.shape[2] for c in cores3]}", flush=True)
    ks = KernelSet({2: TTKernel((c1, c2)), 3: TTKernel(tuple(cores3))})
    n0 = np.zeros(n_classes)
    n0[0] = 1.0
    lit = _run_traj(ks, n0, 0.01, 100, 10)
    short = _run_traj(ks, n0, 0.01, 2, 1)
    print(f"C4 literal: fail_step {int(lit['fail_step'])} warned {bool(lit['warned'])}; "
          f"2-step rows\n{short['rows']}", flush=True)
    idx = sample_indices(n_classes)
    nf = short["n_final"]
    out = dict(idx=idx, lit_fail_step=lit["fail_step"], lit_rows=lit["rows"], lit_warned=lit["warned"],
               n2_final=nf[idx], n2_sums=checksums(nf), n2_rows=short["rows"])
    for k in range(3):  # I[0..d-1] and J[1..d] define the d = 3 cores
        out[f"I{k}"] = I[k]
        out[f"J{k + 1}"] = J[k + 1]
    save("c4traj.npz", **out)


def c4_case():
    """C4-shaped TT case at a size where the dense TT-SVD is cheap.

    d=2: exact rank-3 cores of (i^(1/3)+j^(1/3))^2; d=3: TT-SVD of
    (i+j+l)^(1/2)(ijl)^(-1/6) to tolerance 1e-6, ranks capped at 16.  The
    cores are stored and fed identically to every implementation, so parity
    does not depend on the compression.
    """
    out = {}
    for n_classes in (128, 256):
        i = np.arange(1, n_classes + 1, dtype=np.float64)
        c1 = np.zeros((1, n_classes, 3))
        c1[0, :, 0], c1[0, :, 1], c1[0, :, 2] = i ** (2 / 3), 2 * i ** (1 / 3), 1.0
        c2 = np.zeros((3, n_classes, 1))
        c2[0, :, 0], c2[1, :, 0], c2[2, :, 0] = 1.0, i ** (1 / 3), i ** (2 / 3)
        s = i[:, None, None] + i[None, :, None] + i[None, None, :]
        dense3 = np.sqrt(s) * (i[:, None, None] * i[None, :, None] * i[None, None, :]) ** (-1 / 6)
        cores3 = tt_svd(dense3, eps=1e-6, rmax=16)
        tag = f"n{n_classes}"
        out[f"{tag}_d2_c0"], out[f"{tag}_d2_c1"] = c1, c2
        for c_i, c in enumerate(cores3):
            out[f"{tag}_d3_c{c_i}"] = c
        ks = KernelSet({2: TTKernel((c1, c2)), 3: TTKernel(tuple(cores3))})
        n0 = np.zeros(n_classes)
        n0[0] = 1.0
        rng = np.random.default_rng(13)
        nr = rng.random(n_classes)
        r = rhs_total(ks, ConcentrationState(nr), PLAN)
        out[f"{tag}_nr"], out[f"{tag}_pr"], out[f"{tag}_qr"] = nr, r.p, r.q
        traj = _run_traj(ks, n0, 0.01, 100, 10)
        for k, v in traj.items():
            out[f"{tag}_traj_" + k] = v
        print(f"C4 n={n_classes} ranks {[c.shape for c in cores3]}", flush=True)
    save("c4.npz", **out)


def ternary_case():
    """The reference's recorded M0(t) trajectory (demos/out_ternary) re-run."""
    config = SimulationConfig(
        n_classes=1 << 10,
        dimension=3,
        kernel_specs={3: ttagg.ConstantSpec(1.0, 3)},
        initial=InitialCondition.monodisperse(1.0),
        time=TimeGrid(0.0, 1e-3, 1000),
        record_every=50,
    )
    final, series = integrate(config)
    save("ternary.npz", rows=np.array(series.rows()), n_final=final.n)


def dense_case():
    """Direct-summation operators rhs_dense_P / rhs_dense_Q (rhs.py:202-227) on
    dense kernels the reference builds itself: a TableSpec read back from a
    binary file (its dense input format), a Brownian spec materialized by
    dense_from_spec, and a mixed KernelSet through rhs_total."""
    import tempfile

    from ttagg import DenseKernel, TableSpec, dense_from_spec, rhs_dense_P, rhs_dense_Q

    rng = np.random.default_rng(7)
    out = {}
    cases = [("d2", 2, 200), ("d3", 3, 40), ("d4", 4, 14), ("d5", 5, 8)]
    with tempfile.TemporaryDirectory() as tmp:
        for tag, d, N in cases:
            a = rng.random((N,) * d)
            sym = sum(np.transpose(a, perm) for perm in __import__("itertools").permutations(range(d)))
            path = os.path.join(tmp, f"{tag}.bin")
            sym.astype("<f8").tofile(path)
            k = dense_from_spec(TableSpec(path=path, dimension=d), N)
            n = rng.random(N) * np.exp(-np.arange(N) / (N / 4))
            out[f"{tag}_values"] = k.values
            out[f"{tag}_n"] = n
            out[f"{tag}_P"] = rhs_dense_P(k, ConcentrationState(n))
            out[f"{tag}_Q"] = rhs_dense_Q(k, ConcentrationState(n))
    N = 40
    kb = dense_from_spec(BrownianSpec((0.2, -0.2, 0.1)), N)
    n = np.exp(-np.arange(N) / 10.0)
    out["brown3_values"] = kb.values
    out["brown3_n"] = n
    out["brown3_P"] = rhs_dense_P(kb, ConcentrationState(n))
    out["brown3_Q"] = rhs_dense_Q(kb, ConcentrationState(n))
    ks = KernelSet({2: DenseKernel(out["d2_values"][:N, :N].copy()), 3: kb})
    r = rhs_total(ks, ConcentrationState(n), breakdown=True)
    out["mix_p"], out["mix_q"], out["mix_s"] = r.p, r.q, r.s
    save("dense.npz", **out)


CLI_CONFIG = {
    "N": 4096,
    "D": 3,
    "kernels": {"2": {"type": "brownian", "mu": [0.3, -0.3]},
                "3": {"type": "brownian", "mu": [0.2, -0.1, -0.1]}},
    "initial": {"kind": "monodisperse", "c0": 1.0},
    "time": {"t0": 0.0, "dt": 0.01, "steps": 40},
    "record_every": 10,
}


def cli_case():
    """The reference's own CLI (``ttagg simulate``, cli.py:80-110) on a
    Brownian D = 3 config: its moments.csv rows and the final snapshot
    n_40.csv.  The kernels are the reference's default ones for Brownian
    specs (exact TT, config.py:231-242)."""
    import json
    import tempfile

    from ttagg import cli

    with tempfile.TemporaryDirectory() as tmp:
        path = os.path.join(tmp, "run.json")
        with open(path, "w") as fh:
            json.dump(CLI_CONFIG, fh)
        out = os.path.join(tmp, "out")
        assert cli.main(["simulate", "--config", path, "--output", out]) == 0
        rows = np.loadtxt(os.path.join(out, "moments.csv"), delimiter=",", skiprows=1)
        snap = np.loadtxt(os.path.join(out, "n_40.csv"), delimiter=",", skiprows=1)
    save("cli.npz", config=np.array(json.dumps(CLI_CONFIG)), rows=rows, n_final=snap[:, 1])


if __name__ == "__main__":
    os.makedirs(OUT, exist_ok=True)
    which = sys.argv[1:] or ["unit", "ternary", "c1", "c2", "c3", "c4", "c5", "dense"]
    for name in which:
        t0 = time.perf_counter()
        globals()[f"{name}_case" if not name.endswith("_case") else name]()
        print(f"[{name}] {time.perf_counter() - t0:.1f}s", flush=True)
