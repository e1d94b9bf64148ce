"""GPU RK2 trajectories vs the reference's own (golden) trajectories.
Tolerance: relative max-norm error <= 1e-8 after the full integration."""

import warnings

import numpy as np
import pytest

import paper_1905_09071_b200 as g
from conftest import assert_rows, rel_inf
from oracle import rhs_oracle as orc
from paper_1905_09071_b200.workloads import CONFIGS, initial_state

pytestmark = pytest.mark.gpu
TRAJ_TOL = 1e-8


class Cfg:
    def __init__(self, n0, dt, steps, record_every, t0=0.0):
        self.n_classes = n0.size
        self.initial = g.InitialCondition.from_vector(n0) if n0.min() >= 0 else None
        self.time = g.TimeGrid(t0, dt, steps)
        self.record_every = record_every


def test_c1_trajectory_vs_reference(golden):
    c = golden("c1.npz")
    cfg = CONFIGS["C1"]
    ks = g.KernelSet({d: g.CPKernel(f) for d, f in cfg.cp_factors().items()})
    final, series = g.integrate(Cfg(initial_state("mono", cfg.n_classes), cfg.dt, cfg.steps, 10), kernels=ks)
    assert rel_inf(final.n, c["traj_n_final"]) <= TRAJ_TOL
    assert_rows(series.rows(), c["traj_rows"], TRAJ_TOL)
    assert not series.negativity_flagged


def test_ternary_constant_kernel_vs_reference(golden):
    t = golden("ternary.npz")
    ks = g.KernelSet({3: g.constant_tt(1.0, 3, 1024)})
    final, series = g.integrate(Cfg(initial_state("mono", 1024), 1e-3, 1000, 50), kernels=ks)
    assert_rows(series.rows(), t["rows"], TRAJ_TOL)
    assert rel_inf(final.n, t["n_final"]) <= TRAJ_TOL
    assert abs(series.m0[-1] - (1 + 2 / 3) ** -0.5) < 1e-3


def test_c4_shaped_tt_trajectories_vs_reference(golden):
    c = golden("c4.npz")
    for n_classes in (128, 256):
        tag = f"n{n_classes}"
        ks = g.KernelSet({2: g.TTKernel((c[f"{tag}_d2_c0"], c[f"{tag}_d2_c1"])),
                          3: g.TTKernel(tuple(c[f"{tag}_d3_c{i}"] for i in range(3)))})
        final, series = g.integrate(Cfg(initial_state("mono", n_classes), 0.01, 100, 10), kernels=ks)
        assert rel_inf(final.n, c[f"{tag}_traj_n_final"]) <= TRAJ_TOL
        assert_rows(series.rows(), c[f"{tag}_traj_rows"], TRAJ_TOL)


def test_c3_literal_failure_semantics(golden):
    """Reference: StepSizeWarning then StepFailureError(step_index=2) with 2 rows."""
    c = golden("c3.npz")
    cfg = CONFIGS["C3"]
    ks = g.KernelSet({d: g.CPKernel(f) for d, f in cfg.cp_factors().items()})
    with warnings.catch_warnings(record=True) as caught:
        warnings.simplefilter("always")
        with pytest.raises(g.StepFailureError) as exc:
            g.integrate(Cfg(initial_state("exp256", cfg.n_classes), cfg.dt, 3, 1), kernels=ks)
    assert exc.value.step_index == int(c["lit_fail_step"]) == 2
    assert len(exc.value.series) == len(c["lit_rows"])
    assert_rows(exc.value.series.rows()[:1], c["lit_rows"][:1], 1e-12)
    assert_rows(exc.value.series.rows(), c["lit_rows"], 1e-6)  # diverged step-1 row
    assert any(issubclass(w.category, g.StepSizeWarning) for w in caught) == bool(c["lit_warned"])


def test_c3_normalised_trajectory_vs_reference(golden):
    c = golden("c3.npz")
    cfg = CONFIGS["C3"]
    ks = g.KernelSet({d: g.CPKernel(f) for d, f in cfg.cp_factors(1 << 12).items()})
    final, series = g.integrate(Cfg(initial_state("exp256", 1 << 12, normalised=True), cfg.dt, cfg.steps, 20),
                                kernels=ks)
    assert rel_inf(final.n, c["norm4096_n_final"]) <= TRAJ_TOL
    assert_rows(series.rows(), c["norm4096_rows"], TRAJ_TOL)


def test_c5_literal_failure_and_normalised_trajectory(golden):
    c = golden("c5.npz")
    cfg = CONFIGS["C5"]
    ks = g.KernelSet({d: g.CPKernel(f) for d, f in cfg.cp_factors(1 << 12).items()})
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        with pytest.raises(g.StepFailureError) as exc:
            g.integrate(Cfg(initial_state("c5", 1 << 12), cfg.dt, 3, 1), kernels=ks)
    assert exc.value.step_index == int(c["lit4096_fail_step"]) == 2
    assert len(exc.value.series) == len(c["lit4096_rows"])
    final, series = g.integrate(Cfg(initial_state("c5", 1 << 12, normalised=True), cfg.dt, cfg.steps, 5),
                                kernels=ks)
    assert rel_inf(final.n, c["norm4096_n_final"]) <= TRAJ_TOL
    assert_rows(series.rows(), c["norm4096_rows"], TRAJ_TOL)


def test_fused_integrate_matches_stepwise_and_rk2_step(monkeypatch):
    """The device-resident fused loop (ttagg_rk2), its per-record-interval form
    (on_record) and the host-orchestrated rk2_step loop (taken when the
    rhs_total seam is replaced) agree."""
    import paper_1905_09071_b200.integrator as integrator_mod

    cfg = CONFIGS["C5"]
    N = 1 << 13
    ks = g.KernelSet({d: g.CPKernel(f) for d, f in cfg.cp_factors(N).items()})
    n0 = initial_state("c5", N, normalised=True)
    fused_final, fused = g.integrate(Cfg(n0, cfg.dt, 7, 2), kernels=ks)
    seen, states = [], []
    chunk_final, chunked = g.integrate(Cfg(n0, cfg.dt, 7, 2), kernels=ks,
                                       on_record=lambda s, x: (seen.append(s), states.append(x.n.copy())))
    assert seen == [0, 2, 4, 6]
    assert rel_inf(fused_final.n, chunk_final.n) <= 1e-13
    assert_rows(fused.rows(), chunked.rows(), 1e-13)
    orig = integrator_mod.rhs_total
    monkeypatch.setattr(integrator_mod, "rhs_total", lambda *a, **k: orig(*a, **k))
    seen2 = []
    step_final, stepped = g.integrate(Cfg(n0, cfg.dt, 7, 2), kernels=ks, on_record=lambda s, x: seen2.append(x.n.copy()))
    assert len(seen2) == 4
    for a, b in zip(states, seen2):
        assert rel_inf(a, b) <= 1e-13
    assert rel_inf(fused_final.n, step_final.n) <= 1e-13
    assert_rows(fused.rows(), stepped.rows(), 1e-12)
    s = g.ConcentrationState(n0)
    for _ in range(7):
        s = g.rk2_step(s, cfg.dt, ks)
    assert rel_inf(s.n, fused_final.n) <= 1e-13
    ref_n, _, _ = orc.integrate({d: {"kind": "cp", "arrays": ks[d].factors} for d in ks.orders}, n0,
                                dt=cfg.dt, steps=7)
    assert rel_inf(fused_final.n, ref_n) <= 1e-10


def test_negativity_flag():
    """min(n) < -1e-9 max|n| after a step sets the flag and warns once (integrator.py:216-223)."""
    ks = g.KernelSet({2: g.constant_tt(1.0, 2, 64)})
    n0 = np.full(64, 1.0)
    with warnings.catch_warnings(record=True) as caught:
        warnings.simplefilter("always")
        _, series = g.integrate(Cfg(n0, 0.9, 3, 1), kernels=ks)
    ref_n, _, ref = orc.integrate({2: {"kind": "tt", "arrays": ks[2].cores}}, n0, dt=0.9, steps=3)
    assert series.negativity_flagged == ref.negativity_flagged
    if ref.negativity_flagged:
        assert sum(issubclass(w.category, g.StepSizeWarning) for w in caught) == 1


def test_dist_engine_rk2_matches_fused_integrate():
    """The multi-GPU orchestration (dist.DistRHS + CudaEngine: perm-layout
    partial RHS, all-reduce, ttagg_stage updates) on one GPU == ttagg_rk2."""
    from paper_1905_09071_b200.dist import CudaEngine, DistRHS, shard_for_rank
    from paper_1905_09071_b200 import _lib

    cfg = CONFIGS["C5"]
    N = 1 << 13
    f = cfg.cp_factors(N)
    n0 = initial_state("c5", N, normalised=True)
    eng = CudaEngine(f, shard_for_rank({d: v[0].shape[1] for d, v in f.items()}, 1, 0), N, _lib.get_context().device)
    res = DistRHS(eng).rk2(n0, 0.0, cfg.dt, 6, record_every=2)
    ks = g.KernelSet({d: g.CPKernel(v) for d, v in f.items()})
    final, series = g.integrate(Cfg(n0, cfg.dt, 6, 2), kernels=ks)
    assert res.fail_step == 0
    assert rel_inf(res.n, final.n) <= 1e-13
    assert_rows(res.rows, series.rows(), 1e-12)


def test_dt_halving_ratio_is_second_order():
    """test_integrator.py:105-110 / test_acceptance.py:157-165: halving dt cuts
    the RK2 error by ~4 (reference solution at dt/8)."""
    N = 256
    ks = g.KernelSet({3: g.constant_tt(1.0, 3, N)})
    n0 = initial_state("mono", N)
    T = 0.4

    def final(dt):
        return g.integrate(Cfg(n0, dt, int(round(T / dt)), int(round(T / dt))), kernels=ks)[0].n

    ref = final(0.0125)
    e1 = np.abs(final(0.1) - ref).max()
    e2 = np.abs(final(0.05) - ref).max()
    assert 3.2 <= e1 / e2 <= 4.8


def test_brownian_tt_mass_drift():
    """test_integrator.py:130-141: the exact Brownian TT kernel conserves mass
    to <= 1e-6 over 100 steps at N = 1024 before boundary contact (here through
    the live-fiber TT upload)."""
    from test_gpu_tt_sparse import subset_tt

    N = 1024
    ks = g.KernelSet({3: g.TTKernel(subset_tt((0.1, -0.1, 0.0), N))})
    n0 = initial_state("mono", N)
    final, series = g.integrate(Cfg(n0, 1e-3, 100, 100), kernels=ks)
    m1 = np.array([r[2] for r in series.rows()])
    assert abs(m1[-1] - m1[0]) / m1[0] <= 1e-6


def test_execution_plan_does_not_change_results():
    """test_rhs.py:330-366 (worker-count and FFT-length-policy independence):
    the GPU path accepts any plan; results are bitwise identical."""
    cfg = CONFIGS["C1"]
    ks = g.KernelSet({d: g.CPKernel(f) for d, f in cfg.cp_factors().items()})
    st = g.ConcentrationState(initial_state("exp256", cfg.n_classes))
    base = g.rhs_total(ks, st).s
    for plan in (g.ExecutionPlan(workers=8), g.ExecutionPlan(fft_length_policy="min"), g.SERIAL_PLAN):
        assert np.array_equal(g.rhs_total(ks, st, plan).s, base)


def test_c5_full_size_trajectory_vs_reference(golden):
    """North star: the RK2 trajectory at N = 2^20, D = 5 (config C5: dt = 0.002,
    50 steps; mass-normalised state since the literal one diverges at step 2)
    against the reference's own integrate() on the same tensor (its Brownian
    TT route) — sampled final state, full-vector checksums, moment rows —
    to the north star's 1e-8."""
    c = golden("c5traj.npz")
    cfg = CONFIGS["C5"]
    ks = g.KernelSet({d: g.CPKernel(f) for d, f in cfg.cp_factors().items()})
    n0 = initial_state("c5", cfg.n_classes, normalised=True)
    final, series = g.integrate(Cfg(n0, cfg.dt, cfg.steps, 10), kernels=ks)
    assert int(c["fail_step"]) == 0
    assert rel_inf(final.n[c["idx"]], c["n_final"]) <= TRAJ_TOL
    k = np.arange(1, cfg.n_classes + 1, dtype=np.float64)
    v = final.n
    sums = np.array([v.sum(), k @ v, (k * k) @ v, np.abs(v).sum(), np.abs(v).max()])
    assert np.all(np.abs(sums - c["n_sums"]) <= TRAJ_TOL * np.abs(c["n_sums"]))
    assert_rows(series.rows(), c["rows"], TRAJ_TOL)


def test_c3_full_size_trajectory_vs_reference(golden):
    """Config C3 at full size (N = 2^18, D = 4, dt = 0.005, 200 steps,
    mass-normalised state) against the reference's own integrate() (CP route)."""
    c = golden("c3traj.npz")
    cfg = CONFIGS["C3"]
    ks = g.KernelSet({d: g.CPKernel(f) for d, f in cfg.cp_factors().items()})
    n0 = initial_state("exp256", cfg.n_classes, normalised=True)
    final, series = g.integrate(Cfg(n0, cfg.dt, cfg.steps, 20), kernels=ks)
    assert int(c["fail_step"]) == 0
    assert rel_inf(final.n[c["idx"]], c["n_final"]) <= TRAJ_TOL
    k = np.arange(1, cfg.n_classes + 1, dtype=np.float64)
    v = final.n
    sums = np.array([v.sum(), k @ v, (k * k) @ v, np.abs(v).sum(), np.abs(v).max()])
    assert np.all(np.abs(sums - c["n_sums"]) <= TRAJ_TOL * np.abs(c["n_sums"]))
    assert_rows(series.rows(), c["rows"], TRAJ_TOL)


def test_c4_full_size_vs_reference(golden):
    """Config C4 at full size (N = 2^20, D = 3, TT kernels: exact rank-3 d = 2,
    TT-cross d = 3 with ranks 16, rebuilt from the stored cross skeleton;
    monodisperse, dt = 0.01) against the reference's own integrate() on the
    same cores: as literally specified it diverges (StepSizeWarning, then
    StepFailureError at step 9, one recorded row) and so must the GPU run;
    the first two steps (before the instability of the large sizes reaches
    the roundoff floor) are compared state for state."""
    from paper_1905_09071_b200 import construct

    c = golden("c4traj.npz")
    N = 1 << 20
    c1, c2 = construct.c4_d2_cores(N)
    cores3 = construct.c4_d3_from_skeleton(N, [c["I0"], c["I1"], c["I2"]], [None, c["J1"], c["J2"], c["J3"]])
    ks = g.KernelSet({2: g.TTKernel((c1, c2)), 3: g.TTKernel(cores3)})
    n0 = initial_state("mono", N)
    with warnings.catch_warnings(record=True) as caught:
        warnings.simplefilter("always")
        with pytest.raises(g.StepFailureError) as exc:
            g.integrate(Cfg(n0, 0.01, 100, 10), kernels=ks)
    assert exc.value.step_index == int(c["lit_fail_step"]) == 9
    assert any(issubclass(w.category, g.StepSizeWarning) for w in caught) == bool(c["lit_warned"])
    assert_rows(exc.value.series.rows(), c["lit_rows"], TRAJ_TOL)
    final, series = g.integrate(Cfg(n0, 0.01, 2, 1), kernels=ks)
    assert rel_inf(final.n[c["idx"]], c["n2_final"]) <= TRAJ_TOL
    # M0, M1 and the state's own sums; the k^2-weighted M2 of a monodisperse
    # start is dominated by the roundoff floor of the ~10^6 empty sizes
    # (k^2 up to 10^12 times ~1e-17 noise, different in any two correct FFT
    # implementations: 1.0577 vs 1.0578 after one step), so it is not compared
    k = np.arange(1, N + 1, dtype=np.float64)
    v = final.n
    sums = np.array([v.sum(), k @ v, (k * k) @ v, np.abs(v).sum(), np.abs(v).max()])
    for i in (0, 1, 4):
        assert abs(sums[i] - c["n2_sums"][i]) <= TRAJ_TOL * abs(c["n2_sums"][i])
    rows = np.array(series.rows())
    assert np.allclose(rows[:, :3], c["n2_rows"][:, :3], rtol=TRAJ_TOL, atol=0.0)


def test_config_kernels_match_reference_cli(golden):
    """integrate(config) with kernels=None builds the reference's default
    kernels from the config's specs in-repo (construct.kernel_set_from_config,
    config.py:231-242: Brownian -> exact TT) and matches the reference's own
    `ttagg simulate` run (moments.csv rows and the final snapshot n_40.csv,
    oracle/make_golden.py cli)."""
    import json
    from types import SimpleNamespace

    ref = golden("cli.npz")
    c = json.loads(str(ref["config"]))
    specs = {int(d): SimpleNamespace(exponents=tuple(k["mu"]), dimension=len(k["mu"]))
             for d, k in c["kernels"].items()}
    cfg = SimpleNamespace(n_classes=c["N"], kernel_specs=specs,
                          initial=g.InitialCondition.monodisperse(c["initial"]["c0"]),
                          time=g.TimeGrid(c["time"]["t0"], c["time"]["dt"], c["time"]["steps"]),
                          record_every=c["record_every"])
    final, series = g.integrate(cfg)
    assert rel_inf(final.n, ref["n_final"]) <= TRAJ_TOL
    assert_rows(series.rows(), ref["rows"], TRAJ_TOL)
    assert final.t == ref["rows"][-1, 0]
